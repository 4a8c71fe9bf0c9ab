#!/bin/bash
# Persistent grid sized with the max-carveout occupancy (+ L2 batches for single-group
# models) vs the one-block-per-item build (var_prev); interaction register variants.
set -u
OUT=gpurun_out/${TAG:-r02k}; mkdir -p $OUT
GTS_DEBUG_LAUNCH=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; grep per_sm $OUT/smoke.log | sort | uniq | head
GTS_DEBUG_LAUNCH=1 timeout 300 python bench.py --workload covtype-large --mode shap --rows-per-gpu 4096 --rows-per-step 0 --steps 1 --warmup 1 \
  --no-e2e --no-ablation --no-cpu-baseline --extras none 2>&1 | grep per_sm | sort | uniq
TAG=${TAG:-r02k}/ab LIBS="libgts.so var_prev.so" STEPS=3 \
  WLS="covtype-large:shap:65536 cal_housing-med:both:1048576 fashion_mnist-med:shap:65536 fashion_mnist-med:interactions:1024 adult-large:both:65536 covtype-large:interactions:4096" bash scripts/gpu_ab.sh
TAG=${TAG:-r02k}/inter LIBS="var_ra5.so var_cu5.so" STEPS=3 WLS="adult-large:both:65536 covtype-large:interactions:4096" bash scripts/gpu_ab.sh
GTS_LIB=$PWD/paper_2010_13972_b200/_lib/libgts.so timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.per_cycle_active \
  --clock-control none -k regex:nodal_kernel -s 1 -c 1 --csv python bench.py --workload covtype-large --mode shap \
  --rows-per-gpu 65536 --rows-per-step 0 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ablation --extras none \
  > $OUT/traffic_libgts.csv 2> $OUT/traffic_libgts.err
grep -E "dram__bytes|duration|warps_active" $OUT/traffic_libgts.csv | sed 's/"//g' | awk -F, '{print $(NF-2), $(NF-1), $NF}'
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests.log
python scripts/ab_table.py $OUT/ab $OUT/inter
