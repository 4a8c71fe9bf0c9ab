#!/bin/bash
# One short bench line per (kernel-variant library, workload/mode) on one B200.
# usage: OUT=dir VARS="main gm0 gm2" CASES="covtype fashion fashion_int" bash scripts/gpu_variants.sh
set -u
OUT=${OUT:-gpurun_out/var}; mkdir -p $OUT
Q="--steps 3 --warmup 1 --no-e2e --no-ablation --no-cpu-baseline --extras none"
for v in ${VARS:-main}; do
  lib=paper_2010_13972_b200/_lib/libgts.so
  [ $v != main ] && lib=paper_2010_13972_b200/_lib/var_$v.so
  [ -f $lib ] || { echo "no $lib"; continue; }
  for c in ${CASES:-covtype}; do
    case $c in
      covtype) A="--workload covtype-large --mode shap --rows-per-step 65536";;
      fashion) A="--workload fashion_mnist-med --mode shap --rows-per-gpu 65536 --rows-per-step 0";;
      fashion_int) A="--workload fashion_mnist-med --mode interactions --rows-per-gpu 2048 --rows-per-step 0";;
      covtype_int) A="--workload covtype-large --mode interactions --rows-per-gpu 8192 --rows-per-step 0";;
      adult) A="--workload adult-large --mode both --rows-per-gpu 65536 --rows-per-step 0";;
      adult_shap) A="--workload adult-large --mode shap --rows-per-gpu 65536 --rows-per-step 0";;
      calmed) A="--workload cal_housing-med --mode both --rows-per-step 0";;
      calmed_shap) A="--workload cal_housing-med --mode shap --rows-per-step 0";;
    esac
    GTS_LIB=$lib timeout 900 python bench.py $A $Q > $OUT/${c}_$v.json 2> $OUT/${c}_$v.err
  done
done
for f in $OUT/*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d["roofline"]; print(sys.argv[1].split("/")[-1], round(d["value"],1), "rows/s frac", round(r["frac"],3), "ms", round(d["ms_per_step"],1))
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
