"""Per-rank device time of bench.py's multi-GPU sharding, simulated on one GPU:
each rank's shard (row strip + halo, or image range) is filtered with the
device entry points and timed with CUDA events; the predicted N-GPU value is
total pixels / max over ranks.  Diagnostics for strong-scaling (c2) and weak
(c5) behaviour; the real N-GPU numbers come from bench.py under torchrun."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1603_08081_b200 as fb  # noqa: E402
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of  # noqa: E402
from paper_1603_08081_b200.shard import geometry, plan  # noqa: E402


def rank_ms(c, s, a, world, rank, reps=5):
    sh = plan(c.width, c.height, c.batch, s.radius, world, rank)
    geo = geometry(sh, c.width, c.height)
    if c.batch > 1:
        host = np.stack([image_of(c, i) for i in sh.images[:2]] * (len(sh.images) // 2 + 1))[:len(sh.images)]
    else:
        host = image_of(c, 0, sh.src_row0, sh.src_rows)[None]
    src = torch.from_numpy(host.astype(np.float32)).cuda()
    dst = torch.empty((host.shape[0], sh.out_rows, c.width), dtype=torch.float32, device="cuda")
    wsb = fb.workspace_bytes(geo, s.radius, "fused")
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    run = lambda: fb.bilateral_fast_device(src.data_ptr(), dst.data_ptr(), geo, s, a, ws.data_ptr(), wsb,  # noqa
                                           bad.data_ptr(), st, "fused", c.check_epsilon)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name in sys.argv[1:] or ["c2"]:
    c = CONFIGS[name]
    s, a = spatial_of(c), approx_of(c)
    px = c.width * c.height * c.batch
    base = None
    for world in (1, 2, 4, 8):
        ranks = range(world) if c.batch == 1 else [0]
        t = max(rank_ms(c, s, a, world, r) for r in ranks)
        base = base or t
        print(f"{name} N={world}: max rank {t:8.3f} ms -> {px / t / 1e3:9.1f} Mpixel/s, "
              f"speed-up {base / t:5.2f} (efficiency {base / t / world:5.1%})")
