#!/bin/bash
# ncu --set full capture of the nodal kernel(s) for one workload; summaries are
# written on the box (text), the .ncu-rep is deleted unless KEEP=1.
# usage: OUT=dir NAME=tag WL=workload ROWS=n MODE=shap|interactions|both [KEEP=1] bash scripts/ncu_one.sh
set -u
OUT=${OUT:-gpurun_out/ncu}
mkdir -p $OUT
N=1; [ "${MODE:-both}" = "both" ] && N=2
# mode both, warm-up 1: nodal launches are SHAP, interactions, fused (warm-up) then the same three timed;
# SKIP=5 COUNT=1 captures the timed fused call
timeout ${NCU_TIMEOUT:-900} ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-nodal_kernel} -s ${SKIP:-$N} -c ${COUNT:-$N} \
  -o $OUT/${NAME:-prof} python bench.py --workload ${WL:-cal_housing-med} --mode ${MODE:-both} --steps 1 --warmup 1 \
  --rows-per-gpu ${ROWS:-262144} --no-cpu-baseline --no-e2e --no-ablation ${BARGS:-} > $OUT/${NAME:-prof}.log 2>&1
echo "ncu ${NAME:-prof} rc=$?"
python scripts/ncu_summary.py $OUT/${NAME:-prof}.ncu-rep > $OUT/${NAME:-prof}.summary.txt 2>&1
python scripts/ncu_sass_mix.py $OUT/${NAME:-prof}.ncu-rep 30 > $OUT/${NAME:-prof}.mix.txt 2>&1
ncu -i $OUT/${NAME:-prof}.ncu-rep --page raw --csv > $OUT/${NAME:-prof}.raw.csv 2>/dev/null
[ "${KEEP:-0}" = "1" ] || rm -f $OUT/${NAME:-prof}.ncu-rep
