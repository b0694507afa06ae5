#!/bin/bash
# FIR visiting order variants: |fast - exact| on c4/c2 and same-box speed
L=paper_1603_08081_b200/_lib
for lib in ab_r0c0 ab_r0c1 ab_r1c0 libfourierbf_b200; do
  echo "== $lib"; FBF_LIBRARY=$PWD/$L/$lib.so python tools/bound_report.py --no-oracle c2 c4 2>&1 | tail -2
done
CONFIGS="c2 c4 c5" ROUNDS=1 bash tools/ab.sh $L/ab_r0c0.so $L/ab_r0c1.so $L/ab_r1c0.so $L/libfourierbf_b200.so
