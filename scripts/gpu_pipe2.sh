OUT=gpurun_out/r01s; mkdir -p $OUT
for c in 2 3 4; do
timeout 900 python bench.py --e2e-chunks $c --no-cpu-baseline --no-ablation > $OUT/bench_e2e_c$c.json 2> $OUT/bench_e2e_c$c.err; echo "c$c rc=$?"
done
