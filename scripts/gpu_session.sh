#!/bin/bash
# One full GPU session: parity tests, smoke, the default bench line, the ncu
# launch list of that bench command, and one `ncu --set full` capture of each
# nodal kernel (SHAP + interactions) with text summaries.
# usage: TAG=r01 bash scripts/gpu_session.sh
set -u
OUT=gpurun_out/${TAG:-run}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpuinfo.txt 2>&1
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests/ -m gpu -q -x --timeout 600 -p no:cacheprovider ${TEST_ARGS:-} > $OUT/gpu_tests.log 2>&1
  echo "tests rc=$?"; tail -3 $OUT/gpu_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
  echo "smoke rc=$?"; tail -2 $OUT/smoke.log
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
  echo "bench rc=$?"; tail -c 3000 $OUT/bench.json; tail -3 $OUT/bench.err
fi
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
     python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation ${BENCH_ARGS:-} > $OUT/ncu_launch.log 2>&1
  echo "ncu launches rc=$?"
  # one capture per kernel (a long second kernel in the same process came back as nan twice)
  for m in shap interactions; do
    OUT=$OUT NAME=nodal_$m WL=${WL:-cal_housing-med} ROWS=${NCU_ROWS:-1048576} MODE=$m KEEP=${KEEP:-0} bash scripts/ncu_one.sh
    head -24 $OUT/nodal_$m.summary.txt
  done
  OUT=$OUT NAME=nodal_fused WL=${WL:-cal_housing-med} ROWS=${NCU_ROWS:-1048576} MODE=both SKIP=5 COUNT=1 KEEP=${KEEP:-0} \
    bash scripts/ncu_one.sh
  head -24 $OUT/nodal_fused.summary.txt
fi
