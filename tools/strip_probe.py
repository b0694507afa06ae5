"""Device time of the c2 host pipeline's four row strips run back to back (no copies) + host cost of the
group-model queries; FBF_LIBRARY selects the build."""
import os, sys, time, ctypes, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of

c = CONFIGS["c2"]
s, a = spatial_of(c), approx_of(c)
W = s.radius
img = torch.from_numpy(image_of(c).astype(np.float32)).cuda()
out = torch.empty_like(img)
cuts = [0, 256, 1024, 1776, 2048]
geos = []
for o0, o1 in zip(cuts[:-1], cuts[1:]):
    g = fb.whole_geometry(c.width, c.height, 1)
    s0, s1 = max(0, o0 - W), min(c.height, o1 + W)
    g.src_row0, g.src_rows, g.out_row0, g.out_rows = s0, s1 - s0, o0, o1 - o0
    geos.append(g)
t = time.perf_counter()
for _ in range(1000):
    for g in geos:
        fb.lib.fbf_workspace_bytes(ctypes.byref(g), W, 0)
        fb.lib.fbf_harmonic_groups(ctypes.byref(g), W, a.N)
print(f"host: {(time.perf_counter() - t) / 4000 * 1e6:.2f} us per (workspace_bytes + harmonic_groups) query")
ws = [torch.empty(fb.workspace_bytes(g, W, "fused"), dtype=torch.uint8, device="cuda") for g in geos]
bad = torch.full((4,), -1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
def run():
    for k, g in enumerate(geos):
        fb.bilateral_fast_device(img.data_ptr() + 4 * g.src_row0 * c.width, out.data_ptr() + 4 * g.out_row0 * c.width, g, s, a,
                                 ws[k].data_ptr(), ws[k].numel(), bad.data_ptr() + 8 * k, st.cuda_stream)
for _ in range(3): run()
torch.cuda.synchronize()
ts, hs = [], []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h = time.perf_counter(); e0.record(); run(); hs.append(time.perf_counter() - h); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{os.path.basename(os.environ.get('FBF_LIBRARY', 'product'))}: 4 strips device {statistics.median(ts):.4f} ms, host issue {statistics.median(hs)*1e3:.4f} ms")
