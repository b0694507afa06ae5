#!/bin/bash
# ncu --set full of the fused kernel for two library builds (same config):
#   CONFIG=c2 tools/gpu_ncu_ab.sh <libA> <libB>
mkdir -p gpurun_out/ncu_ab
c=${CONFIG:-c2}
i=0
for lib in "$@"; do
  i=$((i+1))
  FBF_LIBRARY=$(realpath $lib) python bench.py --profile-once --config $c > gpurun_out/ncu_ab/plain_$i.log 2>&1 && \
  FBF_LIBRARY=$(realpath $lib) ncu --set full --clock-control none --import-source on -k regex:fused_kernel -c 1 -f \
     -o gpurun_out/ncu_ab/prof_${c}_$i python bench.py --profile-once --config $c > gpurun_out/ncu_ab/ncu_$i.log 2>&1
  echo "ncu $i ($lib) rc=$?"
done
