#!/bin/bash
# CS-aligned ring + finish_groups rewrite + replayed-partition group model: tests, old/new A/B, group sweeps
cd "$(dirname "$0")/.."
A=gpurun_out/r2c; mkdir -p $A
L=paper_1603_08081_b200/_lib
timeout 1200 python -m pytest tests -m gpu -q -x > $A/pytest_gpu2.log 2>&1; echo "pytest rc=$?" | tee -a $A/pytest_gpu2.log; tail -3 $A/pytest_gpu2.log
python - <<'PY'
import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, spatial_of, approx_of
for n,c in CONFIGS.items():
    g=fb.whole_geometry(c.width,c.height,c.batch)
    print(n,'model groups (gaussian query):',fb.harmonic_groups(g,spatial_of(c).radius,c.N),'launches',fb.launches_per_call(g,spatial_of(c),approx_of(c)))
PY
CONFIGS="c2 c5 c1 c3 c4" ROUNDS=1 bash tools/ab.sh $L/libfourierbf_b200_old.so $L/libfourierbf_b200.so 2>&1 | tee $A/ab_old_new.txt
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c2" bash tools/ab_env.sh "FBF_GROUPS=1" "FBF_GROUPS=2" "FBF_GROUPS=4" 2>&1 | tee $A/groups_c2.txt
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c1" bash tools/ab_env.sh "FBF_GROUPS=3" "FBF_GROUPS=4" "FBF_GROUPS=5" "FBF_GROUPS=6" "FBF_GROUPS=7" "FBF_GROUPS=8" 2>&1 | tee $A/groups_c1.txt
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c3" bash tools/ab_env.sh "FBF_GROUPS=2" "FBF_GROUPS=3" "FBF_GROUPS=4" "FBF_GROUPS=5" "FBF_GROUPS=6" "FBF_GROUPS=8" 2>&1 | tee $A/groups_c3.txt
LIB=$L/libfourierbf_b200_exp.so CONFIGS="c5" bash tools/ab_env.sh "FBF_GROUPS=1" "FBF_GROUPS=2" 2>&1 | tee $A/groups_c5.txt
