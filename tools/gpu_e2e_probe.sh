#!/bin/bash
# c4 (8192^2) strip pipeline: strip count x edge weight
python tools/e2e_probe.py c4
for k in 6 8; do for e in 10 20; do FBF_HOST_CHUNKS=$k FBF_HOST_EDGE=$e python tools/e2e_probe.py c4; done; done
FBF_HOST_CHUNKS=4 FBF_HOST_EDGE=10 python tools/e2e_probe.py c4
