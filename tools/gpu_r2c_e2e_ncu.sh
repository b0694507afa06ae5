#!/bin/bash
cd "$(dirname "$0")/.."
L=$(realpath paper_1603_08081_b200/_lib); A=gpurun_out/r2c; mkdir -p $A
for lib in old ""; do
  n=libfourierbf_b200${lib:+_$lib}.so
  FBF_LIBRARY=$L/$n ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/e2e_launches_${lib:-new}.csv python tools/e2e_probe.py c2 > /dev/null 2>&1
  echo "ncu $n rc=$?"
done
