#!/bin/bash
# Second-tier GPU evidence: latency sweeps, packer ablation
# (§8(f)-1), an ncu capture of the interaction kernel at the bench config.
set -u
OUT=gpurun_out/${TAG:-extras}
mkdir -p $OUT
for wl in cal_housing-small cal_housing-med; do
  timeout 600 python bench.py --latency-sweep --workload $wl --rows-per-gpu 1048576 > $OUT/sweep_$wl.json 2> $OUT/sweep_$wl.err
  echo "sweep $wl rc=$?"
done
for wl in cal_housing-med adult-large fashion_mnist-med; do
  timeout 900 python bench.py --workload $wl --mode shap --rows-per-gpu 65536 --steps 3 --pack-ablation \
     --ablation-rows 16384 --no-cpu-baseline --no-e2e > $OUT/packs_$wl.json 2> $OUT/packs_$wl.err
  echo "packs $wl rc=$?"
done
if [ "${NCU:-1}" = "1" ]; then
  OUT=$OUT NAME=inter_full WL=cal_housing-med ROWS=${NCU_ROWS:-1048576} MODE=interactions bash scripts/ncu_one.sh
  head -30 $OUT/inter_full.summary.txt
fi
