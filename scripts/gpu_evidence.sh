#!/bin/bash
# Evidence for HEAD on one B200: smoke, GPU tests, compute-sanitizer (memcheck,
# racecheck, synccheck) on the small cases, the default bench line + launch
# list, ncu --set full of the covtype-large and fashion_mnist-med SHAP kernels.
# usage: TAG=r02c [SAN=0] [TESTS=0] [BENCH=0] [NCU=0] bash scripts/gpu_evidence.sh
set -u
OUT=gpurun_out/${TAG:-ev}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpuinfo.txt 2>&1
nproc > $OUT/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests.log
fi
if [ "${SAN:-1}" = "1" ]; then
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > $OUT/sanitizer_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -3 $OUT/sanitizer_$tool.log
done
fi
if [ "${BENCH:-1}" = "1" ]; then
  t0=$(date +%s)
  timeout 1500 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
  tail -c 1500 $OUT/bench.json
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --extras none > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
fi
if [ "${TRAFFIC:-1}" = "1" ]; then
  # DRAM bytes of the bench's own launch (default config, 2^18 rows): one metrics pass, not --set full
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:nodal_kernel -s 1 -c 1 -o $OUT/traffic_bench python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    --no-e2e --no-ablation --extras none > $OUT/traffic_bench.log 2>&1; echo "traffic pass rc=$?"
  ncu -i $OUT/traffic_bench.ncu-rep --page raw --csv > $OUT/traffic_bench.raw.csv 2>/dev/null; rm -f $OUT/traffic_bench.ncu-rep
fi
if [ "${NCU:-1}" = "1" ]; then
  KEEP=1 OUT=$OUT NAME=ncu_covtype-large_shap WL=covtype-large ROWS=${CT_ROWS:-2048} MODE=shap BARGS="--rows-per-step 0 --extras none" bash scripts/ncu_one.sh
  OUT=$OUT NAME=ncu_fashion_mnist-med_shap WL=fashion_mnist-med ROWS=65536 MODE=shap BARGS="--rows-per-step 0 --extras none" bash scripts/ncu_one.sh
  grep -E "dram__bytes|Duration|warps_active|issue|pipe_fma|Registers" $OUT/*.summary.txt | head -40
fi
