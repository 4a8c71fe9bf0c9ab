#!/bin/bash
# Persistent stream-ordered blocks: GPU tests + smoke of the main build, A/B
# against the one-block-per-item build (var_prev), DRAM traffic of the covtype launch.
set -u
OUT=gpurun_out/${TAG:-r02_p}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpuinfo.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests.log
fi
TAG=${TAG:-r02_p}/ab LIBS="${LIBS:-libgts.so var_prev.so}" STEPS=3 \
  WLS="${WLS:-covtype-large:shap:65536 fashion_mnist-med:shap:65536 adult-large:shap:65536 cal_housing-med:both:1048576 adult-large:both:65536 covtype-large:interactions:4096 fashion_mnist-med:interactions:1024}" bash scripts/gpu_ab.sh
for lib in ${TRAFFIC_LIBS:-libgts.so}; do
  GTS_LIB=$PWD/paper_2010_13972_b200/_lib/$lib timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:nodal_kernel -s 1 -c 1 --csv python bench.py --workload covtype-large --mode shap \
    --rows-per-gpu 65536 --rows-per-step 0 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ablation --extras none \
    > $OUT/traffic_${lib%.so}.csv 2> $OUT/traffic_${lib%.so}.err
  echo "traffic $lib rc=$?"; grep -E "dram__bytes|duration" $OUT/traffic_${lib%.so}.csv | sed 's/"//g' | awk -F, '{print $(NF-2), $(NF-1), $NF}'
done
python scripts/ab_table.py $OUT/ab
