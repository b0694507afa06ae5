"""PCIe copy rates on the box (pinned 16 MiB = one c2 image) and the host entry's e2e per strip count."""
import os, sys, time, ctypes, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of

n = 2048 * 2048
h = torch.empty(n, dtype=torch.float32).pin_memory(); h2 = torch.empty_like(h).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda"); d2 = torch.empty_like(d)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        a = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    return statistics.median(ts) * 1e3
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print(f"H2D 16 MiB: {t(lambda: d.copy_(h, non_blocking=True)):.3f} ms")
print(f"D2H 16 MiB: {t(lambda: h2.copy_(d2, non_blocking=True)):.3f} ms")
print(f"H2D || D2H: {t(both):.3f} ms")
c = CONFIGS["c2"]; img = image_of(c).astype(np.float32); s, a = spatial_of(c), approx_of(c)
src = torch.from_numpy(img).pin_memory(); dst = torch.empty_like(src).pin_memory()
g = fb.whole_geometry(c.width, c.height, 1); f = fb._filter_struct(s, a)
bad = ctypes.c_longlong(-1)
ps, pd = ctypes.cast(src.data_ptr(), fb._F), ctypes.cast(dst.data_ptr(), fb._F)
call = lambda: fb._check(fb.lib.fbf_bilateral_fast_host(ctypes.byref(g), ctypes.byref(f), ps, pd, 0, ctypes.byref(bad)))
for k in ("1", "2", "3", "4", "6"):
    os.environ["FBF_HOST_CHUNKS"] = k
    print(f"host entry K={k}: {t(call, 30):.3f} ms")
