#!/bin/bash
# Persistent grid sized by computed occupancy (libgts) vs one block per item with the
# same item order (var_np) vs the earlier one-block-per-item build (var_prev).
set -u
OUT=gpurun_out/${TAG:-r02l}; mkdir -p $OUT
GTS_DEBUG_LAUNCH=1 timeout 300 python bench.py --workload covtype-large --mode shap --rows-per-gpu 4096 --rows-per-step 0 --steps 1 --warmup 1 \
  --no-e2e --no-ablation --no-cpu-baseline --extras none 2>&1 | grep per_sm | sort | uniq
GTS_DEBUG_LAUNCH=1 timeout 300 python bench.py --workload fashion_mnist-med --mode shap --rows-per-gpu 4096 --rows-per-step 0 --steps 1 --warmup 1 \
  --no-e2e --no-ablation --no-cpu-baseline --extras none 2>&1 | grep per_sm | sort | uniq
TAG=${TAG:-r02l}/ab LIBS="libgts.so var_np.so var_prev.so" STEPS=4 \
  WLS="covtype-large:shap:65536 cal_housing-med:both:1048576 fashion_mnist-med:shap:65536 fashion_mnist-med:interactions:1024 adult-large:both:65536 covtype-large:interactions:4096" bash scripts/gpu_ab.sh
for f in $OUT/ab/*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["config"]["rows_per_step"]
print("%-55s min %.1f ms -> %.4g rows/s" % (sys.argv[1].split("/")[-1], d["ms_per_step_min"], r / d["ms_per_step_min"] * 1e3))
PY
done
GTS_LIB=$PWD/paper_2010_13972_b200/_lib/libgts.so timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.per_cycle_active \
  --clock-control none -k regex:nodal_kernel -s 1 -c 1 --csv python bench.py --workload covtype-large --mode shap \
  --rows-per-gpu 65536 --rows-per-step 0 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ablation --extras none \
  > $OUT/traffic_libgts.csv 2> $OUT/traffic_libgts.err
grep -E "dram__bytes|duration|warps_active" $OUT/traffic_libgts.csv | sed 's/"//g' | awk -F, '{print $(NF-2), $(NF-1), $NF}'
