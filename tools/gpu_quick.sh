#!/bin/bash
# quick iteration: smoke + gpu tests + c2 bench + one ncu --set full capture of the fused kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c2}; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_EXTRA} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; cut -c1-400 gpurun_out/bench_$c.json
done
if [ -n "$NCU" ]; then
python bench.py --profile-once --config ${NCU} > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fused_kernel -c 1 -o gpurun_out/prof_fused_${NCU} -f python bench.py --profile-once --config ${NCU} > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
fi
