# A/B: upper-triangle atomics + mirror pass (default) vs both halves by atomics (nomir) for wide-model interactions
mkdir -p gpurun_out/r01q
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r01q/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r01q/gpu_tests.log
TAG=r01q LIBS="libgts.so libgts_nomir.so" WLS="fashion_mnist-med:interactions:10000 covtype-large:interactions:8192" STEPS=3 bash scripts/gpu_ab.sh
