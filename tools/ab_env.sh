#!/bin/bash
# same-box A/B of environment settings on one (experiment) build:
#   LIB=<lib.so> CONFIGS="c2" tools/ab_env.sh "FBF_X=1" "FBF_X=2" ...
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-1}); do
for c in ${CONFIGS:-c2}; do
for env in "$@"; do
  env $env FBF_LIBRARY=$(realpath ${LIB}) timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/abe.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/abe.json').readline()); r=d['roofline']
print('$r', '$c', '$(basename ${LIB})', '$env', round(d['value'],1), round(r['frac'],4), round(r['kernel_ms'],4), round(r['prep_ms'],4), d['clocks']['sm_mhz'])"
done; done; done
