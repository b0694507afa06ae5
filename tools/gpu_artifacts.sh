#!/bin/bash
# Round artifacts: default bench line (c2), reference arm, other configs, the
# ncu launch list of the bench command and one --set full capture of the fused kernel.
mkdir -p gpurun_out/art
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/art/gpu.txt
lscpu > gpurun_out/art/lscpu.txt
python bench.py > gpurun_out/art/bench_default.json 2> gpurun_out/art/bench_default.err; echo "bench default rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/art/bench_reference.json 2> gpurun_out/art/bench_reference.err; echo "reference rc=$?"
for c in c1 c3 c4 c5; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/art/bench_$c.json 2> gpurun_out/art/bench_$c.err; echo "bench $c rc=$?"
done
python bench.py --variant naive --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/art/bench_c2_naive.json 2>&1; echo "naive rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/art/plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/art/launches_c2.csv $CMD > gpurun_out/art/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
for c in c2 c4; do
python bench.py --profile-once --config $c > gpurun_out/art/plain_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fused_kernel -c 1 -f -o gpurun_out/art/prof_fused_$c python bench.py --profile-once --config $c > gpurun_out/art/ncu_full_$c.log 2>&1
echo "ncu full $c rc=$?"
done
