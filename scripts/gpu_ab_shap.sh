# A/B: rows per lane of the wide-slot SHAP kernel (rw2) and recomputed o-bits in scalar SHAP runs (reo)
mkdir -p gpurun_out/r01p
for v in rw2 reo; do
  GTS_LIB=$PWD/paper_2010_13972_b200/_lib/libgts_$v.so timeout 600 python -m pytest tests -m gpu -x -q \
    -k "(configs_shap and nodal and f32) or slot_widths" > gpurun_out/r01p/parity_$v.log 2>&1
  echo "$v parity rc=$?"; tail -1 gpurun_out/r01p/parity_$v.log
done
TAG=r01p LIBS="libgts_base.so libgts_rw2.so" WLS="covtype-large:shap:32768 fashion_mnist-med:shap:65536" bash scripts/gpu_ab.sh
TAG=r01p LIBS="libgts_base.so libgts_reo.so" WLS="cal_housing-med:shap:1048576 adult-large:shap:65536" bash scripts/gpu_ab.sh
