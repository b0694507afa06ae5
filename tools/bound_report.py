#!/usr/bin/env python
"""Measured |fast - exact| (GPU fp64 brute force) vs the paper's bound, and
max-abs vs the fp64 oracle, per BASELINE config -> stdout (profiles/)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_08081_b200 as fb  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402
from paper_1603_08081_b200.configs import CONFIGS, T_FIXED, approx_of, image_of, spatial_of  # noqa: E402

O = Oracle()
print("config | max-abs vs fp64 oracle (rows checked) | max |fast-exact| (rows) | paper bound")
for name, c in CONFIGS.items():
    s, a = spatial_of(c), approx_of(c)
    img = image_of(c)
    fast = fb.bilateral_fast(img, s, a, check_epsilon=c.check_epsilon)
    rows = (0, c.height) if c.height * c.width <= 2048 * 2048 // 4 else (c.height // 2 - 32, c.height // 2 + 32)
    ref, rc, _ = O.bilateral_fast(img, s.profile, s.radius, s.w0, a.d, a.omega, a.max_pointwise_error,
                                  c.check_epsilon, rows[0], rows[1], os.cpu_count() or 8)
    par = float(np.abs(fast[rows[0]:rows[1]] - ref).max())
    er = (0, c.height) if c.width * c.height <= 4096 * 4096 else (c.height // 2 - 64, c.height // 2 + 64)
    ex = fb.bilateral_exact_gpu(img, s, c.range_family, c.sigma_r, er[0], er[1] - er[0])
    err = float(np.abs(fast[er[0]:er[1]] - ex).max())
    try:
        bound = fb.error_bound(T_FIXED, a.max_pointwise_error, s.w0)
    except ValueError:
        bound = float("nan")
    print(f"{name} | {par:.3e} (rows {rows[0]}-{rows[1]}) | {err:.3e} (rows {er[0]}-{er[1]}) | {bound:.4e}")
