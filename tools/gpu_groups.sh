#!/bin/bash
mkdir -p gpurun_out
for gr in 1 2 4 8; do for c in c1 c2 c4 c5 c3; do
FBF_GROUPS=$gr timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/grp_${gr}_$c.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/grp_${gr}_$c.json').readline()); r=d['roofline']; print('groups $gr $c', round(d['value'],1), round(r['frac'],3), round(r['kernel_ms'],3))"
done; done
