#!/bin/bash
# one experiment call: optional gpu tests, phase split, same-box A/B of two library builds
# usage: TESTS=1 PHASE="c2" CONFIGS="c2 c4" tools/gpu_ab_run.sh <libA> <libB>
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
fi
[ -n "$PHASE" ] && timeout 300 python tools/phase_probe.py $PHASE
CONFIGS="${CONFIGS:-c2 c5}" ROUNDS=${ROUNDS:-2} bash tools/ab.sh "$@"
