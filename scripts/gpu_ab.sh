#!/bin/bash
# A/B kernel variants: the same bench lines through each in-tree library build.
# usage: TAG=ab LIBS="libgts.so libgts_r4.so" WLS="cal_housing-med:shap:1048576 adult-large:both:65536" bash scripts/gpu_ab.sh
set -u
OUT=gpurun_out/${TAG:-ab}
mkdir -p $OUT
for lib in ${LIBS:-libgts.so}; do
  for spec in ${WLS:-cal_housing-med:both:1048576}; do
    IFS=: read wl mode rows slots <<< "$spec"
    slots=${slots:-0}
    GTS_LIB=$PWD/paper_2010_13972_b200/_lib/$lib timeout 900 python bench.py --workload $wl --mode $mode \
      --rows-per-gpu $rows --max-slots $slots --steps ${STEPS:-5} --no-cpu-baseline --no-e2e --no-ablation ${EXTRA:-} > $OUT/${lib%.so}_${wl}_${mode}_s$slots.json 2> $OUT/${lib%.so}_${wl}_${mode}_s$slots.err
    echo "$lib $wl $mode slots=$slots rc=$?"
    python - $OUT/${lib%.so}_${wl}_${mode}_s$slots.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print("  ERR", e); sys.exit()
for m in ("shap", "interactions"):
    x = d.get(m)
    if x:
        print(f"  {m:13s} {x['rows_per_s']:.4g} rows/s  {x['ms']:.3f} ms  frac {x['roofline']['frac']:.3f}")
PY
  done
done
