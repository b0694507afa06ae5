#!/usr/bin/env python
"""Measured |fast - exact| (GPU fp64 brute force) vs the paper's bound, and
max-abs vs the fp64 oracle, per BASELINE config -> stdout (profiles/).
Whole images everywhere (c5: its first four images)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_08081_b200 as fb  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402
from paper_1603_08081_b200.configs import CONFIGS, T_FIXED, approx_of, image_of, spatial_of  # noqa: E402

O = Oracle()
NO_ORACLE = "--no-oracle" in sys.argv  # |fast - exact| only (the fp64 oracle on c4 takes minutes)
ONLY = [a for a in sys.argv[1:] if not a.startswith("--")]
threads = os.cpu_count() or 8
print("config | image | max-abs vs fp64 oracle | max |fast-exact| | paper bound | oracle s | exact s")
for name, c in CONFIGS.items():
    if ONLY and name not in ONLY:
        continue
    s, a = spatial_of(c), approx_of(c)
    try:
        bound = fb.error_bound(T_FIXED, a.max_pointwise_error, s.w0)
    except ValueError:
        bound = float("nan")
    for index in range(4 if c.batch > 1 else 1):
        img = image_of(c, index)
        fast = fb.bilateral_fast(img, s, a, check_epsilon=c.check_epsilon)
        t = time.perf_counter()
        par = float("nan")
        if not NO_ORACLE:
            ref, rc, _ = O.bilateral_fast(img, s.profile, s.radius, s.w0, a.d, a.omega, a.max_pointwise_error,
                                          c.check_epsilon, 0, c.height, threads)
            assert rc == 0
            par = float(np.abs(fast - ref).max())
        t_or = time.perf_counter() - t
        t = time.perf_counter()
        ex = fb.bilateral_exact_gpu(img, s, c.range_family, c.sigma_r, 0, c.height)
        t_ex = time.perf_counter() - t
        err = float(np.abs(fast - ex).max())
        print(f"{name} | {index} ({c.width}x{c.height}) | {par:.3e} | {err:.3e} | {bound:.4e} | {t_or:.1f} | {t_ex:.1f}",
              flush=True)
