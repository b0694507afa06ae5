#!/bin/bash
# ncu --set full of the fused kernel under two environment settings of one build:
#   LIB=<lib> CONFIG=c2 tools/gpu_ncu_env.sh "FBF_X=0" "FBF_X=1"
mkdir -p gpurun_out/ncu_env
c=${CONFIG:-c2}; i=0
for e in "$@"; do
  i=$((i+1))
  env $e FBF_LIBRARY=$(realpath $LIB) python bench.py --profile-once --config $c > /dev/null 2>&1 && \
  env $e FBF_LIBRARY=$(realpath $LIB) ncu --set full --clock-control none --import-source on -k regex:fused_kernel -c 1 -f \
     -o gpurun_out/ncu_env/prof_${c}_$i python bench.py --profile-once --config $c > gpurun_out/ncu_env/ncu_$i.log 2>&1
  echo "ncu $i ($e) rc=$?"
done
