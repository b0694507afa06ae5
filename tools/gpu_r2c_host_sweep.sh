#!/bin/bash
cd "$(dirname "$0")/.."
export FBF_LIBRARY=$(realpath paper_1603_08081_b200/_lib/libfourierbf_b200_exp.so)
python tools/e2e_probe.py c2
for k in 3 4 5 6; do for e in 25 35 50; do FBF_HOST_CHUNKS=$k FBF_HOST_EDGE=$e python tools/e2e_probe.py c2; done; done
python tools/e2e_probe.py c3
for k in 1 2 3; do FBF_HOST_CHUNKS=$k python tools/e2e_probe.py c3; done
