#!/bin/bash
# full GPU tests on the product build, then same-box A/B against a baseline build
#   CONFIGS="c2 c5" tools/gpu_ab_quick.sh <baseline.so>
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
CONFIGS="${CONFIGS:-c2 c5}" ROUNDS=${ROUNDS:-2} bash tools/ab.sh "$1" paper_1603_08081_b200/_lib/libfourierbf_b200.so
