#!/bin/bash
# Round-2 artifacts: GPU tests, race-shake check, bench lines of every config,
# the reference arm, the ncu launch list of the default bench command and one
# ncu --set full capture of the fused kernel per config (+ the n = 0 kernel).
cd "$(dirname "$0")/.."
A=gpurun_out/r02; mkdir -p $A
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $A/gpu.txt
lscpu > $A/lscpu.txt
timeout 1200 python -m pytest tests -m gpu -q > $A/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $A/pytest_gpu.log
timeout 900 python tools/shake_check.py > $A/shake.log 2>&1; echo "shake rc=$?"
python bench.py > $A/bench_default.json 2> $A/bench_default.err; echo "bench default rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > $A/bench_reference.json 2> $A/bench_reference.err; echo "reference rc=$?"
for c in c1 c3 c4 c5; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $A/bench_$c.json 2> $A/bench_$c.err; echo "bench $c rc=$?"
done
python bench.py --variant naive --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $A/bench_c2_naive.json 2>&1; echo "naive rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $A/plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_c2.csv $CMD > $A/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
for c in c1 c3 c5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
for c in c2 c1 c3 c4 c5; do
  python bench.py --profile-once --config $c > $A/plain_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fused_kernel -c 1 -f -o $A/prof_fused_$c python bench.py --profile-once --config $c > $A/ncu_full_$c.log 2>&1
  echo "ncu full $c rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:n0_plane -c 1 -f -o $A/prof_n0_c2 python bench.py --profile-once --config c2 > $A/ncu_n0.log 2>&1
echo "ncu n0 rc=$?"
