"""GPU: harmonic split (partial (Q, P) sums over harmonic ranges + finish).

Used inside one GPU for small images (CTA groups, automatic) and across GPUs
(NCCL all-reduce of the partial planes, paper_1603_08081_b200.shard.harmonic_split_filter).
The multi-rank sum is emulated here rank by rank on one GPU (no kernel waits
on another)."""
import numpy as np
import pytest

import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of
from paper_1603_08081_b200.shard import harmonic_range, harmonic_split_filter

pytestmark = pytest.mark.gpu


def _bufs(img, geo, s, variant="fused"):
    import torch
    dev = torch.device("cuda", 0)
    src = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).to(dev)
    ws = torch.empty(fb.workspace_bytes(geo, s.radius, variant), dtype=torch.uint8, device=dev)
    dst = torch.empty((geo.batch, geo.out_rows, geo.width), dtype=torch.float32, device=dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    return src, ws, dst, bad


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
@pytest.mark.parametrize("variant", ["fused", "naive"])
def test_full_range_partial_then_finish_is_the_filter(name, variant):
    import torch
    c = CONFIGS[name]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    geo = fb.whole_geometry(c.width, c.height)
    src, ws, dst, bad = _bufs(img, geo, s, variant)
    harmonic_split_filter(src, geo, s, a, ws, dst, bad, variant=variant, check_epsilon=c.check_epsilon)
    torch.cuda.synchronize()
    # the filter = one device launch over the same geometry (the host entry may
    # pipeline larger calls in strips with their own harmonic grouping)
    ref = torch.empty_like(dst)
    fb.bilateral_fast_device(src.data_ptr(), ref.data_ptr(), geo, s, a, ws.data_ptr(), ws.numel(), bad.data_ptr(),
                             0, variant, c.check_epsilon)
    torch.cuda.synchronize()
    assert np.array_equal(dst.cpu().numpy(), ref.cpu().numpy())
    host = fb.bilateral_fast(img, s, a, variant=variant, check_epsilon=c.check_epsilon)
    assert np.abs(dst.cpu().numpy()[0] - host).max() <= 2e-4


@pytest.mark.parametrize("world", [2, 3, 8])
def test_ranks_partial_sums_add_up(world):
    """Each emulated rank's partial plane over its harmonic range; their sum
    (the NCCL all-reduce) divided == the whole filter to fp32 rounding."""
    import torch
    c = CONFIGS["c1"]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    geo = fb.whole_geometry(c.width, c.height)
    src, ws, dst, bad = _bufs(img, geo, s)
    st = torch.cuda.current_stream().cuda_stream
    fb.prepare_device(src.data_ptr(), geo, s, a, ws.data_ptr(), ws.numel(), st)
    total = torch.zeros((1, c.height, c.width, 2), dtype=torch.float32, device=src.device)
    for r in range(world):
        lo, hi = harmonic_range(a.N, world, r)
        if hi <= lo:
            continue
        part = torch.zeros_like(total)
        fb.partial_sums_device(part.data_ptr(), geo, s, a, lo, hi, ws.data_ptr(), ws.numel(), st)
        total += part
    fb.finish_device(total.data_ptr(), dst.data_ptr(), geo, s, a, bad.data_ptr(), st)
    torch.cuda.synchronize()
    ref = fb.bilateral_fast(img, s, a)
    assert float(np.abs(dst.cpu().numpy()[0] - ref).max()) <= 1e-3
    assert int(bad.item()) == -1
