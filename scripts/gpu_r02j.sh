#!/bin/bash
# Persistent blocks with a staggered chunk start (GTS_STAGGER 4 / 16 / 1) vs the
# one-block-per-item build (var_prev); TMEM X by slot for the 32-slot kernel is in
# every persistent build; GPU tests; DRAM traffic; ncu --set full of covtype SHAP.
set -u
OUT=gpurun_out/${TAG:-r02j}; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests.log
TAG=${TAG:-r02j}/ab LIBS="libgts.so var_st16.so var_st1.so var_prev.so" STEPS=3 \
  WLS="covtype-large:shap:65536 cal_housing-med:both:1048576 fashion_mnist-med:shap:65536 fashion_mnist-med:interactions:1024 adult-large:both:65536" bash scripts/gpu_ab.sh
for lib in libgts.so var_st16.so; do
  GTS_LIB=$PWD/paper_2010_13972_b200/_lib/$lib timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:nodal_kernel -s 1 -c 1 --csv python bench.py --workload covtype-large --mode shap \
    --rows-per-gpu 65536 --rows-per-step 0 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ablation --extras none \
    > $OUT/traffic_${lib%.so}.csv 2> $OUT/traffic_${lib%.so}.err
  echo "traffic $lib rc=$?"; grep -E "dram__bytes|duration" $OUT/traffic_${lib%.so}.csv | sed 's/"//g' | awk -F, '{print $(NF-2), $(NF-1), $NF}'
done
KEEP=0 OUT=$OUT NAME=ncu_covtype-large_shap WL=covtype-large ROWS=16384 MODE=shap BARGS="--rows-per-step 0 --extras none" bash scripts/ncu_one.sh
grep -E "Duration|duration|warps_active|issue|pipe_fma|Registers|dram__bytes|stalls" $OUT/ncu_covtype-large_shap.summary.txt | head -20
python scripts/ab_table.py $OUT/ab
