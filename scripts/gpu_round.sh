#!/bin/bash
# One GPU session: bench line, launch list (ncu), full capture of the nodal kernels.
set -u
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-run}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpuinfo.txt 2>&1
timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"
tail -c 3000 $OUT/bench.json
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
     python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-ablation ${NCU_ARGS:-} > $OUT/ncu_launch.log 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:nodal_kernel -s 2 -c 2 \
     -o $OUT/prof python bench.py --steps 1 --warmup 1 --rows-per-gpu ${NCU_ROWS:-262144} --no-cpu-baseline --no-e2e --no-ablation ${NCU_ARGS:-} > $OUT/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
