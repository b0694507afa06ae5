#!/bin/bash
# gpurun_out/r02 (tools/gpu_round2.sh) -> profiles/: bench lines, logs, launch list, ncu summaries and
# the per-launch DRAM traffic files bench.py reads (profiles/ncu_fused_<cfg>.json)
cd "$(dirname "$0")/.."
A=gpurun_out/r02; P=profiles
for c in c1 c3 c4 c5; do cp $A/bench_$c.json $P/r02_bench_$c.json; done
cp $A/bench_default.json $P/r02_bench_default.json
cp $A/bench_reference.json $P/r02_bench_reference.json
cp $A/bench_c2_naive.json $P/r02_bench_c2_naive.json
cp $A/launches_c2.csv $P/r02_launches_c2.csv
for c in c1 c3 c5; do [ -f $A/launches_$c.csv ] && cp $A/launches_$c.csv $P/r02_launches_$c.csv; done
cp $A/pytest_gpu.log $P/r02_pytest_gpu.log
cp $A/shake.log $P/r02_shake.txt
cp $A/gpu.txt $P/r02_gpu.txt
for c in c1 c2 c3 c4 c5; do
  python tools/ncu_summary.py $A/prof_fused_$c.ncu-rep 25 > $P/r02_ncu_fused_${c}_summary.txt
  python tools/ncu_json.py $A/prof_fused_$c.ncu-rep $c > /dev/null
done
python tools/ncu_summary.py $A/prof_n0_c2.ncu-rep 10 > $P/r02_ncu_n0_c2_summary.txt
python tools/ncu_lines.py $A/prof_fused_c2.ncu-rep > $P/r02_ncu_fused_c2_lines.txt 2>/dev/null
for c in default c1 c3 c4 c5; do python - $P/r02_bench_$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).readline()); r=d['roofline']
print(d['config']['workload'], round(d['value'],1), 'Mpx/s frac', round(r['frac'],4), 'kernel_ms', round(r['kernel_ms'],4), 'prep', round(r['prep_ms'],4), 'e2e', round(d['e2e']['value']), 'e2e_f64', round(d['e2e_f64']['value']), 'traffic', r['traffic'], 'clocks', d['clocks']['sm_mhz'], d['clocks']['reasons'])
PY
done
