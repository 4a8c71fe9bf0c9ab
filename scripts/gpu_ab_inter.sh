# A/B of paired-node interaction runs per Q (GTS_INTER_PAIRED bitmask) + parity of each variant
mkdir -p gpurun_out/r01n
for v in p24 p34 p234; do
  GTS_LIB=$PWD/paper_2010_13972_b200/_lib/libgts_$v.so timeout 600 python -m pytest tests -m gpu -x -q \
    -k "(configs_interactions or fused) and nodal and f32" > gpurun_out/r01n/parity_$v.log 2>&1
  echo "$v parity rc=$?"
done
TAG=r01n LIBS="libgts_base.so libgts_p24.so libgts_p34.so libgts_p234.so" \
  WLS="cal_housing-med:interactions:1048576 adult-large:interactions:65536 cal_housing-small:interactions:1048576" \
  bash scripts/gpu_ab.sh
TAG=r01n LIBS="libgts_base.so libgts_p34.so libgts_p234.so" WLS="cal_housing-med:interactions:1048576" bash scripts/gpu_ab.sh
