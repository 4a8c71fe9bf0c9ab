#!/bin/bash
# Kernel-shape variants (built with _build.build(out=..., defines=...)) on one
# B200: one short bench line per (variant lib, workload).
out=${1:-gpurun_out/r02_var}; shift
vars=${@:-main}
mkdir -p $out
Q="--steps 3 --warmup 1 --no-e2e --no-ablation --no-cpu-baseline --extras none"
for v in $vars; do
  lib=paper_2010_13972_b200/_lib/libgts.so
  [ $v != main ] && lib=paper_2010_13972_b200/_lib/var_$v.so
  [ -f $lib ] || continue
  GTS_LIB=$lib timeout 600 python bench.py --workload covtype-large --mode shap --rows-per-step 65536 $Q > $out/covtype_$v.json 2> $out/covtype_$v.err
  case $v in main|rmw1)
    GTS_LIB=$lib timeout 600 python bench.py --workload fashion_mnist-med --mode shap --rows-per-gpu 65536 --rows-per-step 65536 $Q > $out/fashion_$v.json 2> $out/fashion_$v.err
    GTS_LIB=$lib timeout 600 python bench.py --workload cal_housing-med --mode shap --rows-per-step 0 $Q > $out/calmed_shap_$v.json 2> $out/calmed_shap_$v.err
    GTS_LIB=$lib timeout 600 python bench.py --workload adult-large --mode shap --rows-per-gpu 65536 --rows-per-step 0 $Q > $out/adult_shap_$v.json 2> $out/adult_shap_$v.err;;
  esac
done
for f in $out/*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d["roofline"]; print(sys.argv[1].split("/")[-1], round(d["value"],1), "rows/s frac", round(r["frac"],3), "ms", round(d["ms_per_step"],1))
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
