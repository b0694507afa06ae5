#!/bin/bash
# group sweeps on the experiment build + launch list with 2 groups (finish_groups time)
cd "$(dirname "$0")/.."
A=gpurun_out/r2c; mkdir -p $A
L=paper_1603_08081_b200/_lib
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c2" ROUNDS=2 bash tools/ab_env.sh "FBF_GROUPS=1" "FBF_GROUPS=2" "FBF_GROUPS=4" 2>&1 | tee $A/groups_c2.txt
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c1" bash tools/ab_env.sh "FBF_GROUPS=3" "FBF_GROUPS=4" "FBF_GROUPS=5" "FBF_GROUPS=6" "FBF_GROUPS=7" "FBF_GROUPS=8" 2>&1 | tee $A/groups_c1.txt
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c3" bash tools/ab_env.sh "FBF_GROUPS=2" "FBF_GROUPS=3" "FBF_GROUPS=4" "FBF_GROUPS=5" "FBF_GROUPS=6" "FBF_GROUPS=8" 2>&1 | tee $A/groups_c3.txt
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c5" bash tools/ab_env.sh "FBF_GROUPS=1" "FBF_GROUPS=2" 2>&1 | tee $A/groups_c5.txt
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for c in c2 c1 c3; do
FBF_GROUPS=$([ $c = c2 ] && echo 2 || echo 6) FBF_LIBRARY=$(realpath $L/libfourierbf_b200_exp.so) ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_${c}_g.csv $CMD --config $c > $A/ncu_launch_g.log 2>&1
echo "ncu $c rc=$?"
done
