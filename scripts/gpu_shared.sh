#!/bin/bash
# Shared-row interaction blocks: the new GPU parity test, then fashion_mnist /
# covtype interactions with the mode on (auto) and off (GTS_INTER_SHARED_ROWS=0),
# and the identity-map interaction kernels against the previous build (var_prev).
set -u
OUT=gpurun_out/${TAG:-r02_sh}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "shared_row or configs_interactions or fused or mirror" > $OUT/gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests.log
Q="--steps 3 --warmup 1 --no-e2e --no-ablation --no-cpu-baseline --extras none"
for env in auto 0; do
  GTS_INTER_SHARED_ROWS=$([ $env = auto ] && echo 1 || echo 0) timeout 900 python bench.py --workload fashion_mnist-med \
    --mode interactions --rows-per-gpu 1024 --rows-per-step 0 $Q > $OUT/fashion_inter_$env.json 2> $OUT/fashion_inter_$env.err
  echo "fashion inter $env rc=$?"
  GTS_INTER_SHARED_ROWS=$([ $env = auto ] && echo 1 || echo 2) timeout 900 python bench.py --workload covtype-large \
    --mode interactions --rows-per-gpu 4096 --rows-per-step 0 $Q > $OUT/covtype_inter_$env.json 2> $OUT/covtype_inter_$env.err
  echo "covtype inter $env rc=$?"
done
TAG=${TAG:-r02_sh}/ab LIBS="libgts.so var_prev.so" STEPS=3 WLS="cal_housing-med:both:1048576 adult-large:both:65536" bash scripts/gpu_ab.sh
python scripts/ab_table.py $OUT $OUT/ab
