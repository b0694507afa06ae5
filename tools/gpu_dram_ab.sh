#!/bin/bash
# DRAM bytes (ncu) and bench speed of the fused kernel for several library builds
#   CONFIGS="c5 c4" tools/gpu_dram_ab.sh <lib1> <lib2> ...
mkdir -p gpurun_out/dram
for c in ${CONFIGS:-c5}; do for lib in "$@"; do
  n=$(basename $lib .so)
  FBF_LIBRARY=$(realpath $lib) python bench.py --profile-once --config $c > /dev/null 2>&1 && \
  FBF_LIBRARY=$(realpath $lib) ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fused_kernel -c 1 --csv python bench.py --profile-once --config $c > gpurun_out/dram/${c}_$n.csv 2>/dev/null
  echo "$c $n $(grep -E 'dram__bytes|gpu__time' gpurun_out/dram/${c}_$n.csv | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')"
done; done
CONFIGS="${CONFIGS:-c5}" ROUNDS=1 bash tools/ab.sh "$@"
