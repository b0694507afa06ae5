#!/bin/bash
# Same-box A/B of an experiment switch: tools/ab_env.sh VAR "v1 v2 ..."
# (value "-" = unset), CONFIGS="c2 c5" ROUNDS=2; one bench line per run.
mkdir -p gpurun_out
var=$1; vals=$2
for r in $(seq 1 ${ROUNDS:-2}); do
for c in ${CONFIGS:-c2 c5}; do
for v in $vals; do
  if [ "$v" = - ]; then unset $var; else export $var=$v; fi
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').readline()); r=d['roofline']
print('$r', '$c', '$var=$v', round(d['value'],1), round(r['frac'],3), d['clocks']['sm_mhz'])"
done; done; done
unset $var
