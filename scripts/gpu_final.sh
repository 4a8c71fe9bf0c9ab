# Final evidence for HEAD: smoke, default bench line + launch list, every config, ncu of the wide-model interaction kernels
OUT=gpurun_out/r01r; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpuinfo.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
OUT=$OUT NAME=ncu_fashion_mnist-med_interactions WL=fashion_mnist-med ROWS=1000 MODE=interactions bash scripts/ncu_one.sh
OUT=$OUT NAME=ncu_covtype-large_interactions WL=covtype-large ROWS=512 MODE=interactions bash scripts/ncu_one.sh
TAG=r01r_all bash scripts/bench_all.sh
