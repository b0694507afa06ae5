"""Time the recursive (IIR, fp64) backend vs the fused FIR on a bench config
(device-resident, CUDA events; diagnostics for DESIGN.md)."""
import sys
import os

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1603_08081_b200 as fb  # noqa: E402
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    c = CONFIGS[name]
    img = torch.from_numpy(image_of(c).astype(np.float32)).cuda()
    s, a = spatial_of(c), approx_of(c)
    geo = fb.whole_geometry(c.width, c.height, 1)
    out = torch.empty_like(img)
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for variant in ("fused", "recursive"):
        wsb = fb.workspace_bytes(geo, s.radius, variant)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        run = lambda: fb.bilateral_fast_device(img.data_ptr(), out.data_ptr(), geo, s, a, ws.data_ptr(), wsb,  # noqa
                                               bad.data_ptr(), st, variant, c.check_epsilon)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{name} {variant:9s} {ms:8.3f} ms  {c.width * c.height / ms / 1e3:9.1f} Mpixel/s")
