OUT=gpurun_out/r01t; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
