#!/bin/bash
cd "$(dirname "$0")/.."
A=gpurun_out/r2c; mkdir -p $A
L=paper_1603_08081_b200/_lib
CONFIGS="c1 c3" BENCH_EXTRA=--no-e2e bash tools/gpu_r2c_check.sh
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c1" bash tools/ab_env.sh "FBF_GROUPS=6" "FBF_GROUPS=12" "FBF_GROUPS=6 FBF_FUSED_CFG=big" "FBF_GROUPS=4 FBF_FUSED_CFG=big" "FBF_GROUPS=3 FBF_FUSED_CFG=big" "FBF_GROUPS=12 FBF_FUSED_CFG=big" 2>&1 | tee $A/c1_cfg.txt
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c3" bash tools/ab_env.sh "FBF_GROUPS=5" "FBF_GROUPS=10" "FBF_GROUPS=15" "FBF_GROUPS=5 FBF_FUSED_CFG=big" "FBF_GROUPS=3 FBF_FUSED_CFG=big" "FBF_GROUPS=2 FBF_FUSED_CFG=big" 2>&1 | tee $A/c3_cfg.txt
