"""Per-CTA timing of the fused kernel (FBF_PHASE_PROF build): duration spread,
steps per CTA, start skew, and the SM / die of the slowest CTAs."""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
os.environ["FBF_LIBRARY"] = os.path.join(HERE, "..", "paper_1603_08081_b200", "_lib", "libfourierbf_b200_prof.so")
sys.path.insert(0, os.path.join(HERE, ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1603_08081_b200 as fb  # noqa: E402
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of  # noqa: E402


def main(name):
    c = CONFIGS[name]
    img = torch.from_numpy(image_of(c).astype(np.float32)).cuda()
    sp, ap = spatial_of(c), approx_of(c)
    geo = fb.whole_geometry(img.shape[-1], img.shape[-2], 1 if img.dim() == 2 else img.shape[0])
    out = torch.empty_like(img)
    ws_bytes = fb.workspace_bytes(geo, sp.radius, "fused")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    bad = torch.empty(1, dtype=torch.int64, device="cuda")
    fn = fb.lib.fbf_debug_phase_prof
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    buf = (ctypes.c_ulonglong * (32 + 4096))()
    for rep in range(3):
        fb.bilateral_fast_device(img.data_ptr(), out.data_ptr(), geo, sp, ap, ws.data_ptr(), ws_bytes,
                                 bad.data_ptr(), check_epsilon=c.check_epsilon)
        torch.cuda.synchronize()
        fn(buf)
    rec = np.array(buf[32:], dtype=np.float64).reshape(-1, 4)
    rec = rec[rec[:, 2] > 0]
    t0 = rec[:, 1].min()
    start, end, steps, sm = rec[:, 1] - t0, rec[:, 2] - t0, rec[:, 3], rec[:, 0]
    dur = end - start
    print(f"{name}: {len(rec)} CTAs; kernel span {end.max() / 1e3:.1f} us")
    print(f"  start skew: max {start.max() / 1e3:.2f} us")
    print(f"  duration us: min {dur.min() / 1e3:.1f} mean {dur.mean() / 1e3:.1f} max {dur.max() / 1e3:.1f}")
    print(f"  end us:      min {end.min() / 1e3:.1f} mean {end.mean() / 1e3:.1f} max {end.max() / 1e3:.1f}")
    print(f"  steps: min {steps.min():.0f} mean {steps.mean():.1f} max {steps.max():.0f}")
    per = dur / np.maximum(steps, 1)
    print(f"  ns/step: min {per.min():.0f} mean {per.mean():.0f} max {per.max():.0f}")
    lo = sm < np.median(sm)
    print(f"  ns/step by SM half: low {per[lo].mean():.0f}  high {per[~lo].mean():.0f}")
    order = np.argsort(-end)[:8]
    print("  latest CTAs (sm, steps, start, end, ns/step):")
    for i in order:
        print(f"    sm {sm[i]:4.0f} steps {steps[i]:4.0f} start {start[i] / 1e3:7.2f} end {end[i] / 1e3:8.1f} {per[i]:6.0f}")
    c_ = np.corrcoef(steps, dur)[0, 1] if steps.std() > 0 else float('nan')
    print(f"  corr(steps, duration) = {c_:.2f}")


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c2"]:
        main(n)
