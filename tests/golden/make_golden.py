#!/usr/bin/env python
"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Runs only in the build container (needs oracle/_ref/libfbf_ref.so, i.e. the
unmodified reference headers under /root/reference compiled by oracle/Makefile).
The fixtures are committed; tests read them on any box.

Contents (all fp64 unless noted):
  fits.npz      : per BASELINE config c1..c5 the fixed-N fit d_0..d_N, residual
                  norm and max pointwise error (kernel_approx.hpp QrState, T=255),
                  plus progressive_fit(gauss 30, T=217, eps 1e-3)  [test_kernel_approx.cpp:139-158]
  spatial.npz   : profiles / radius / w0 for sigma_s in {1,1.5,2,2.5,3,4,5,8} and box radii {1..5}
  filters.npz   : per config a small crop-sized image from the config's generator
                  parameters (fp32 values) and the reference bilateral_fast output
                  (c3 with the eps < w0 precondition bypassed), plus random integer
                  images with the reference test suite's windows
  exact.npz     : bilateral_exact outputs for two small images (bound checks)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference  # noqa: E402
from paper_1603_08081_b200.configs import CONFIGS, T_FIXED  # noqa: E402
import paper_1603_08081_b200 as fb  # noqa: E402  (host-only entry points: synth generator)


def main():
    ref = Reference()
    fits = {}
    for name, c in CONFIGS.items():
        d, rn, mx = ref.fit_fixed(c.range_family, c.sigma_r, T_FIXED, c.N)
        fits[f"{name}_d"] = d
        fits[f"{name}_residual"] = np.array(rn)
        fits[f"{name}_eps"] = np.array(mx)
    d, n, rn, mx = ref.progressive_fit(0, 30.0, 217, 1e-3)
    fits["prog_g30_T217_e1e-3_d"] = d
    fits["prog_g30_T217_e1e-3_N"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "fits.npz"), **fits)

    sp = {}
    for s in (1.0, 1.5, 2.0, 2.5, 3.0, 4.0, 5.0, 8.0):
        r, p, w0 = ref.make_spatial(0, s)
        sp[f"g{s}_profile"], sp[f"g{s}_radius"], sp[f"g{s}_w0"] = p, np.array(r), np.array(w0)
    for r in range(1, 6):
        rr, p, w0 = ref.make_spatial(1, r)
        sp[f"b{r}_profile"], sp[f"b{r}_w0"] = p, np.array(w0)
    np.savez_compressed(os.path.join(HERE, "spatial.npz"), **sp)

    flt = {}
    sizes = {"c1": (64, 48), "c2": (72, 56), "c3": (64, 40), "c4": (96, 80), "c5": (64, 64)}
    for name, c in CONFIGS.items():
        w, h = sizes[name]
        img = fb.synth_image(c.seeds[0], w, h, max(1, c.rects // 8), c.noise)  # fp32 values
        kind = 1 if c.spatial == "box" else 0
        d = fits[f"{name}_d"]
        out, rc, msg = ref.bilateral_fast(img.astype(np.float64), kind, float(c.sigma_s), d, T_FIXED,
                                          float(fits[f"{name}_eps"]), c.check_epsilon)
        assert rc == 0, msg
        flt[f"{name}_img"], flt[f"{name}_out"] = img, out
    rng = np.random.default_rng(20260819)
    for i, (w, h, s) in enumerate([(16, 16, 1.0), (7, 5, 1.0), (13, 9, 1.5), (1, 9, 1.0), (3, 3, 2.0)]):
        img = rng.integers(0, 256, (h, w)).astype(np.float64)
        d, _, mx = ref.fit_fixed(0, 30.0, 255, 10)
        out, rc, msg = ref.bilateral_fast(img, 0, s, d, 255, mx)
        assert rc == 0, msg
        flt[f"rand{i}_img"], flt[f"rand{i}_out"], flt[f"rand{i}_sigma"] = img, out, np.array(s)
    flt["rand_d"] = ref.fit_fixed(0, 30.0, 255, 10)[0]
    flt["rand_eps"] = np.array(ref.fit_fixed(0, 30.0, 255, 10)[2])
    np.savez_compressed(os.path.join(HERE, "filters.npz"), **flt)

    ex = {}
    for i, (w, h, s, sr) in enumerate([(40, 32, 2.0, 30.0), (33, 21, 3.0, 20.0)]):
        img = rng.integers(0, 256, (h, w)).astype(np.float64)
        ex[f"e{i}_img"] = img
        ex[f"e{i}_out"] = ref.bilateral_exact(img, 0, s, 0, sr)
        ex[f"e{i}_sigma"], ex[f"e{i}_sr"] = np.array(s), np.array(sr)
    np.savez_compressed(os.path.join(HERE, "exact.npz"), **ex)
    for f in ("fits", "spatial", "filters", "exact"):
        print(f, os.path.getsize(os.path.join(HERE, f + ".npz")), "bytes")


if __name__ == "__main__":
    main()
