set -x
mkdir -p gpurun_out/r01m
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r01m/gpuinfo.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01m/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "fused" > gpurun_out/r01m/gpu_tests_fused.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r01m/bench.json 2> gpurun_out/r01m/bench.err
timeout 600 python bench.py --steps 10 --warmup 3 --separate --no-cpu-baseline --no-ablation > gpurun_out/r01m/bench_separate.json 2> gpurun_out/r01m/bench_separate.err
timeout 900 python bench.py --workload adult-large --rows-per-gpu 65536 --steps 5 --warmup 3 --no-cpu-baseline --no-ablation --no-e2e > gpurun_out/r01m/adult-large.json 2> gpurun_out/r01m/adult-large.err
tail -3 gpurun_out/r01m/*.log; cat gpurun_out/r01m/*.json | cut -c1-600
