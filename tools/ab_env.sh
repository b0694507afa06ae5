#!/bin/bash
# A/B the default fused config against FBF_FUSED_CFG=$1 on the same box
mkdir -p gpurun_out
for r in 1 2; do
for c in ${CONFIGS:-c2 c5}; do
for cfg in default "$1"; do
  if [ "$cfg" = default ]; then unset FBF_FUSED_CFG; else export FBF_FUSED_CFG=$cfg; fi
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').readline()); r=d['roofline']
print('$r', '$c', '$cfg', round(d['value'],1), round(r['frac'],3), d['clocks']['sm_mhz'])"
done; done; done
unset FBF_FUSED_CFG
