OUT=gpurun_out/r01s; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "pipelined or mirror or fused" > $OUT/gpu_tests_new.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/gpu_tests_new.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --e2e-serial --no-cpu-baseline --no-ablation > $OUT/bench_e2e_serial.json 2> $OUT/bench_e2e_serial.err; echo "bench serial rc=$?"
