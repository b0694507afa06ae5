#!/bin/bash
cd "$(dirname "$0")/.."
A=gpurun_out/r2c; mkdir -p $A; L=paper_1603_08081_b200/_lib
timeout 1200 python -m pytest tests -m gpu -q -x > $A/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -2 $A/pytest_gpu4.log
CONFIGS="c2 c5 c1 c3" ROUNDS=1 bash tools/ab.sh $L/libfourierbf_b200_old.so $L/libfourierbf_b200.so
CMD="python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
for lib in libfourierbf_b200_old.so libfourierbf_b200.so; do
FBF_LIBRARY=$(realpath $L/$lib) ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_c5_$lib.csv $CMD > /dev/null 2>&1
grep -E "n0_plane|prep_padded" $A/launches_c5_$lib.csv | tail -2 | awk -F'","' '{print $5, $NF}' | cut -c1-40,100-
done
