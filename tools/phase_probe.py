"""Per-phase cycle split of the fused kernel's step loop (diagnostics).

Loads the FBF_PHASE_PROF build (make -C paper_1603_08081_b200/csrc prof),
runs one bench config once and prints the average cycles thread 0 of a CTA
spends per step in each phase."""
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

NAMES = ["loop top", "S1 wait", "row pass", "TMA waits", "S2 wait", "col FIR + next mod", "prologue mod",
         "demod + stores", "TMA issue (leader)"]


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
    buf = (ctypes.c_ulonglong * 32)()
    for rep in range(3):
        fb.bilateral_fast_device(img.data_ptr(), out.data_ptr(), geo, sp, ap, ws.data_ptr(), ws_bytes,
                                 bad.data_ptr(), check_epsilon=c.check_epsilon)
        torch.cuda.synchronize()
        fn(buf)
    print(f"{name}: cycles per step, thread 0 (TMA leader) | thread 32 (warp 1)")
    tot = [0, 0]
    for i in range(9):
        v = [buf[10 * k + i] / max(buf[10 * k + 9], 1) for k in (0, 1)]
        tot = [tot[k] + v[k] for k in (0, 1)]
        print(f"  {NAMES[i]:<22} {v[0]:8.0f} {v[1]:8.0f}")
    print(f"  {'total':<22} {tot[0]:8.0f} {tot[1]:8.0f}")


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c2"]:
        main(n)
