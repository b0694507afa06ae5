#!/bin/bash
# session check: GPU tests, c2 / c5 bench lines, harmonic-group A/B on the experiment build,
# and one compute-sanitizer attempt (racecheck, quick cases)
cd "$(dirname "$0")/.."
A=gpurun_out/r2c; mkdir -p $A
timeout 1200 python -m pytest tests -m gpu -q > $A/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $A/pytest_gpu.log; tail -3 $A/pytest_gpu.log
for c in c2 c5; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $A/bench_$c.json 2> $A/bench_$c.err; echo "bench $c rc=$?"
  python - <<PY
import json; d=json.loads(open('$A/bench_$c.json').readline()); r=d['roofline']
print('$c', round(d['value'],1), round(r['frac'],4), r['kernel_ms'], r['prep_ms'], d['e2e']['value'], d['e2e_f64']['value'])
PY
done
LIB=paper_1603_08081_b200/_lib/libfourierbf_b200_exp.so CONFIGS="c2" ROUNDS=2 bash tools/ab_env.sh "FBF_GROUPS=1" "FBF_GROUPS=2" "FBF_GROUPS=3" 2>&1 | tee $A/groups_ab.txt
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
FBF_GROUPS=2 FBF_LIBRARY=$(realpath paper_1603_08081_b200/_lib/libfourierbf_b200_exp.so) ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_c2_g2.csv $CMD > $A/ncu_launch_g2.log 2>&1
echo "ncu g2 rc=$?"
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_cases.py --quick > $A/racecheck_quick.log 2>&1; echo "racecheck rc=$?"; tail -5 $A/racecheck_quick.log
