#!/bin/bash
# Per-launch device times (ncu, one metric, no replay cost) of one bench configuration.
# usage: OUT=dir NAME=tag BARGS="--workload ... --mode ... --rows-per-gpu ..." bash scripts/launch_list.sh
set -u
OUT=${OUT:-gpurun_out/ll}; mkdir -p $OUT
timeout ${LL_TIMEOUT:-900} ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${NAME:-ll}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ablation --extras none ${BARGS:-} > $OUT/${NAME:-ll}.log 2>&1
echo "launch list ${NAME:-ll} rc=$?"
python - "$OUT/${NAME:-ll}.csv" <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]; ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    agg.setdefault(r[ki][:90], []).append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"  {k:90s} n={len(v):4d} total {sum(v)/1e6:9.3f} ms  share {sum(v)/tot:.3f}")
PY
