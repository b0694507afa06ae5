#!/bin/bash
# tests + bench lines of every config on the product build (+ optional A/B against $OLD)
cd "$(dirname "$0")/.."
A=gpurun_out/r2c; mkdir -p $A
timeout 1200 python -m pytest tests -m gpu -q -x > $A/pytest_gpu3.log 2>&1; echo "pytest rc=$?" | tee -a $A/pytest_gpu3.log; tail -3 $A/pytest_gpu3.log
for c in ${CONFIGS:-c2 c1 c3 c5 c4}; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_EXTRA} > $A/bench_$c.json 2> $A/bench_$c.err; echo "bench $c rc=$?"
  python - <<PY
import json; d=json.loads(open('$A/bench_$c.json').readline()); r=d['roofline']
e=d.get('e2e',{}).get('value'); e6=d.get('e2e_f64',{}).get('value')
print('$c', round(d['value'],1), round(r['frac'],4), round(r['kernel_ms'],4), round(r['prep_ms'],4), 'e2e', e and round(e), 'e2e_f64', e6 and round(e6), 'launches', d['gpu_launches']//d['steps'])
PY
done
