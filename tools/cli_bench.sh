#!/bin/bash
# The reference CLI's --bench sweeps (cli.hpp:72-100: sigma_s 1..12, sigma_r
# 10..100) on a 512^2 synthetic PGM: this build's fourierbf tool (GPU) and the
# reference run() (oracle/_ref, one CPU thread, as the reference is written).
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
python - <<'PY'
import numpy as np
import paper_1603_08081_b200 as fb
img = fb.synth_image(0, 512, 512, 6, 10.0)
q = np.clip(np.floor(img + 0.5), 0, 255).astype(np.uint8)
open("gpurun_out/bench512.pgm", "wb").write(b"P5\n512 512\n255\n" + q.tobytes())
PY
echo "# GPU (paper_1603_08081_b200/_lib/fourierbf --bench, host buffers in/out per call)"
paper_1603_08081_b200/_lib/fourierbf --input gpurun_out/bench512.pgm --sigma-s 5 --sigma-r 20 --bench
echo "# reference run() --bench (CPU, fp64, 1 thread)"
python - <<'PY'
from oracle.pyoracle import Reference
rc, out, err = Reference().cli_run("gpurun_out/bench512.pgm", "", 5.0, 20.0, bench=True)
print(out, end="")
PY
