#!/bin/bash
# A/B two builds of the library on the same box, interleaved:
#   tools/ab.sh <libA.so> <libB.so>   (CONFIGS="c2 c5" ROUNDS=2)
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-2}); do
for c in ${CONFIGS:-c2 c5}; do
for lib in "$@"; do
  FBF_LIBRARY=$(realpath $lib) timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').readline()); r=d['roofline']
print('$r', '$c', '$(basename $lib)', round(d['value'],1), round(r['frac'],3), d['clocks']['sm_mhz'])"
done; done; done
