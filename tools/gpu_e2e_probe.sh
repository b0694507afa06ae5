#!/bin/bash
# host-entry e2e after the per-chunk grouping change: default vs inherited groups, c2 / c4 / c5
for cfg in c2 c4; do
  FBF_HOST_INHERIT_GROUPS=1 python tools/e2e_probe.py $cfg
  python tools/e2e_probe.py $cfg
done
