#!/bin/bash
# e2e of ~1 Mpixel calls: single CUDA-graph launch vs the two-stream strip pipeline
for cfg in c3 c1; do
  python tools/e2e_probe.py $cfg
  FBF_HOST_MIN_MPX=0.2 python tools/e2e_probe.py $cfg
  FBF_HOST_MIN_MPX=0.2 FBF_HOST_CHUNKS=3 python tools/e2e_probe.py $cfg
done
