#!/bin/bash
# GPU session: parity tests, then the bench line, then optional ncu captures.
set -u
OUT=gpurun_out/${TAG:-run}
mkdir -p $OUT
timeout ${TEST_TIMEOUT:-900} python -m pytest tests/ -m gpu -q -x --timeout 600 -p no:cacheprovider ${TEST_ARGS:-} > $OUT/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -5 $OUT/gpu_tests.log
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
  echo "bench rc=$?"; tail -c 2500 $OUT/bench.json; tail -3 $OUT/bench.err
fi
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:nodal_kernel -s 2 -c 2 \
     -o $OUT/prof python bench.py --steps 1 --warmup 1 --rows-per-gpu ${NCU_ROWS:-262144} --no-cpu-baseline --no-e2e --no-ablation ${NCU_ARGS:-} > $OUT/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
