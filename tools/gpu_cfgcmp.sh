#!/bin/bash
# A/B the fused-kernel configurations (FBF_FUSED_CFG) on the bench configs
mkdir -p gpurun_out
for cfgname in ${CFGS:-small big Small Big}; do for c in ${CONFIGS:-c1 c2 c5}; do
FBF_FUSED_CFG=$cfgname timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/cmp_${cfgname}_$c.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/cmp_${cfgname}_$c.json').readline()); r=d['roofline']; print('$cfgname $c', round(d['value'],1), round(r['frac'],3), round(r['kernel_ms'],3))"
done; done
