#!/bin/bash
# one gpurun session: smoke, gpu tests, bench lines for every config, ncu launch list + full capture (c2)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for c in c2 c1 c3 c4 c5; do
  extra=""; [ $c != c2 ] && extra="--no-cpu-baseline"
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 $extra > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
timeout 300 python bench.py --config c2 --variant naive --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_naive.json 2>&1
python bench.py --profile-once > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --profile-once > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
python bench.py --profile-once > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fused_kernel -c 1 -o gpurun_out/prof_fused_c2 python bench.py --profile-once > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
