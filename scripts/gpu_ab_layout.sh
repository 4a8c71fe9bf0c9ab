#!/bin/bash
# r02 A/B: bounds-in-rho-row table layout (main) vs the previous HEAD build (var_head),
# plus register-shape variants; GPU tests of the main build first.
set -u
OUT=gpurun_out/${TAG:-r02_ab}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpuinfo.txt 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests.log
fi
TAG=${TAG:-r02_ab}/shap LIBS="${SHAP_LIBS:-var_head.so libgts.so var_r2q5.so}" STEPS=3 \
  WLS="covtype-large:shap:65536 fashion_mnist-med:shap:65536 adult-large:shap:65536 cal_housing-med:shap:1048576" bash scripts/gpu_ab.sh
TAG=${TAG:-r02_ab}/inter LIBS="${INTER_LIBS:-var_head.so libgts.so var_i8w6.so var_i8w4b3.so}" STEPS=3 \
  WLS="cal_housing-med:both:1048576 adult-large:both:65536" bash scripts/gpu_ab.sh
