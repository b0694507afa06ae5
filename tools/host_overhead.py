import sys, os, time, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1603_08081_b200 as fb
s = fb.make_spatial_gaussian(3.0)
a = fb.fit_fixed(fb.RANGE_GAUSSIAN, 20.0, 255, 12)
for h, w in ((64, 64), (512, 512)):
    src = torch.from_numpy(np.random.default_rng(0).random((h, w), dtype=np.float32) * 255).pin_memory()
    dst = torch.empty_like(src).pin_memory()
    g = fb.whole_geometry(w, h, 1)
    f = fb._filter_struct(s, a)
    bad = ctypes.c_longlong(-1)
    ps, pd = ctypes.cast(src.data_ptr(), fb._F), ctypes.cast(dst.data_ptr(), fb._F)
    call = lambda: fb.lib.fbf_bilateral_fast_host(ctypes.byref(g), ctypes.byref(f), ps, pd, 0, ctypes.byref(bad))
    for _ in range(5): call()
    t = time.perf_counter(); n = 200
    for _ in range(n): call()
    dt = (time.perf_counter() - t) / n
    print(f"{h}x{w}: {dt*1e6:.1f} us per host call")
