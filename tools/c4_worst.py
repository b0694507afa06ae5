"""Diagnose the worst |fast - exact| pixels of c4: their denominators Q and the
fp32 vs fp64 (Q, P) errors (harmonic-split partial sums on a strip around them)."""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
c = CONFIGS[name]
s, a = spatial_of(c), approx_of(c)
img = image_of(c)
fast = fb.bilateral_fast(img, s, a, check_epsilon=c.check_epsilon)
ex = fb.bilateral_exact_gpu(img, s, c.range_family, c.sigma_r, 0, c.height)
err = np.abs(fast - ex)
bound = fb.error_bound(255, a.max_pointwise_error, s.w0)
print(f"{name}: max err {err.max():.3e}, bound {bound:.3e}, pixels over bound {(err > bound).sum()}, "
      f">1e-4 {(err > 1e-4).sum()}, >2e-4 {(err > 2e-4).sum()}")
W = s.radius
d = np.array(a.d, dtype=np.float64)
om = a.omega
prof = np.array(s.profile, dtype=np.float64)
w2 = np.outer(prof, prof)
idx = np.argsort(err.ravel())[::-1][:6]
for k in idx:
    y, x = divmod(int(k), c.width)
    ys = np.clip(np.arange(y - W, y + W + 1), 0, c.height - 1)  # (interior pixels only are exact here)
    xs = np.clip(np.arange(x - W, x + W + 1), 0, c.width - 1)
    win = img[np.ix_(ys, xs)].astype(np.float64)
    fi = float(img[y, x])
    n = np.arange(len(d))
    phi = (d[None, None, :] * np.cos(n[None, None, :] * om * (win[..., None] - fi))).sum(-1)
    Q = (w2 * phi).sum()
    P = (w2 * phi * (win - 128.0)).sum()
    print(f"  ({y},{x}) f={fi:.2f} err={err[y, x]:.3e} fast={fast[y, x]:.5f} exact={ex[y, x]:.5f} "
          f"Q64={Q:.5f} out64={128 + P / Q:.5f} window std={win.std():.1f}")
