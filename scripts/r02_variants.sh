#!/bin/bash
# Kernel-shape variants of the wide SHAP kernels (covtype-large S=64 identity,
# fashion_mnist-med S=32 slot maps) on one B200: bench lines per variant lib.
out=${1:-gpurun_out/r02_var}
mkdir -p $out
Q="--steps 3 --warmup 1 --no-e2e --no-ablation --no-cpu-baseline --extras none"
for v in default c8 w6 r1w8; do
  lib=paper_2010_13972_b200/_lib/libgts.so
  [ $v != default ] && lib=paper_2010_13972_b200/_lib/var_$v.so
  [ -f $lib ] || continue
  GTS_LIB=$lib timeout 600 python bench.py --workload covtype-large --mode shap --rows-per-step 65536 $Q > $out/covtype_$v.json 2> $out/covtype_$v.err
  GTS_LIB=$lib timeout 600 python bench.py --workload fashion_mnist-med --mode shap --rows-per-gpu 65536 --rows-per-step 65536 $Q > $out/fashion_$v.json 2> $out/fashion_$v.err
done
GTS_LIB=paper_2010_13972_b200/_lib/libgts.so timeout 600 python bench.py --workload fashion_mnist-med --mode shap --max-slots 64 --rows-per-gpu 65536 --rows-per-step 65536 $Q > $out/fashion_s64.json 2> $out/fashion_s64.err
timeout 600 python bench.py --workload cal_housing-med --mode both --rows-per-step 0 $Q > $out/calmed_both.json 2> $out/calmed_both.err
timeout 600 python bench.py --workload cal_housing-med --mode shap --rows-per-step 0 $Q > $out/calmed_shap.json 2> $out/calmed_shap.err
timeout 900 python bench.py --workload adult-large --mode both --rows-per-gpu 65536 --rows-per-step 0 $Q > $out/adult_both.json 2> $out/adult_both.err
for f in $out/*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d["roofline"]; print(sys.argv[1].split("/")[-1], round(d["value"],1), "rows/s frac", round(r["frac"],3), "ms", round(d["ms_per_step"],1))
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
