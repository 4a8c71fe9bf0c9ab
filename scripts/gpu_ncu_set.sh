#!/bin/bash
# ncu --set full captures of the nodal kernel on several workloads (one launch each).
# usage: TAG=x SPECS="fashion_mnist-med:shap:65536 covtype-large:shap:32768" bash scripts/gpu_ncu_set.sh
set -u
OUT=gpurun_out/${TAG:-ncuset}
mkdir -p $OUT
for spec in ${SPECS}; do
  IFS=: read wl mode rows <<< "$spec"
  OUT=$OUT NAME=ncu_${wl}_${mode} WL=$wl ROWS=$rows MODE=$mode KEEP=${KEEP:-0} bash scripts/ncu_one.sh
  head -24 $OUT/ncu_${wl}_${mode}.summary.txt | grep -E "Kernel Name|duration|issue_active|warps_active.avg.per|pipe_fma_cycles|registers_per|dram__bytes|stalls"
done
