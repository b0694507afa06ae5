"""Host-entry e2e time of one config (median / mean of 40 calls), for pipeline sweeps:
FBF_HOST_CHUNKS / FBF_HOST_EDGE / FBF_HOST_INHERIT_GROUPS from the environment."""
import os, sys, time, ctypes, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
img = image_of(c).astype(np.float32)
s, a = spatial_of(c), approx_of(c)
src = torch.from_numpy(img).pin_memory(); dst = torch.empty_like(src).pin_memory()
g = fb.whole_geometry(c.width, c.height, 1); f = fb._filter_struct(s, a, c.check_epsilon)
bad = ctypes.c_longlong(-1)
ps, pd = ctypes.cast(src.data_ptr(), fb._F), ctypes.cast(dst.data_ptr(), fb._F)
call = lambda: fb._check(fb.lib.fbf_bilateral_fast_host(ctypes.byref(g), ctypes.byref(f), ps, pd, 0, ctypes.byref(bad)))
for _ in range(3): call()
ts = []
for _ in range(40):
    t = time.perf_counter(); call(); ts.append(time.perf_counter() - t)
px = c.width * c.height
tag = " ".join(f"{k}={os.environ[k]}" for k in ("FBF_HOST_CHUNKS", "FBF_HOST_EDGE", "FBF_HOST_INHERIT_GROUPS") if k in os.environ)
print(f"{c.name} {tag or 'default'}: median {statistics.median(ts)*1e3:.3f} ms ({px/statistics.median(ts)/1e6:.0f} Mpx/s), "
      f"mean {statistics.mean(ts)*1e3:.3f} ms ({px/statistics.mean(ts)/1e6:.0f} Mpx/s)")
