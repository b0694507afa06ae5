#!/bin/bash
# quick GPU check: -m gpu tests + bench of the headline and the other configs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c2}; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c2}; do python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['value'],1), 'e2e', round(d.get('e2e',{}).get('value',0),1), 'frac', round(d['roofline']['frac'],4), 'kernel_ms', round(d['roofline']['kernel_ms'],4), d['clocks'])
" 2>&1 | tail -1; done
