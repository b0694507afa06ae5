#!/bin/bash
cd "$(dirname "$0")/.."
L=$(realpath paper_1603_08081_b200/_lib)
for c in c2 c3 c4; do
for lib in libfourierbf_b200_old.so libfourierbf_b200.so; do echo $lib; FBF_LIBRARY=$L/$lib python tools/e2e_probe.py $c; done
done
