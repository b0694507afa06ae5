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
    """The split path over all harmonics on one rank == one device launch == the host entry, bit for bit."""
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
    assert np.array_equal(dst.cpu().numpy()[0], host)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_ranks_partial_sums_add_up(world):
    """Each emulated rank's partial plane over its harmonic range; their fp64 sum
    (what the NCCL all-reduce computes, in any order) divided == the whole
    filter bit for bit: the partial values are exact multiples of the call's
    fixed-point grid."""
    import torch
    c = CONFIGS["c1"]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    geo = fb.whole_geometry(c.width, c.height)
    src, ws, dst, bad = _bufs(img, geo, s)
    st = torch.cuda.current_stream().cuda_stream
    fb.prepare_device(src.data_ptr(), geo, s, a, ws.data_ptr(), ws.numel(), st)
    parts = []
    for r in range(world):
        lo, hi = harmonic_range(a.N, world, r)
        if hi <= lo:
            continue
        part = torch.zeros((1, c.height, c.width, 2), dtype=torch.float64, device=src.device)
        fb.partial_sums_device(part.data_ptr(), geo, s, a, lo, hi, ws.data_ptr(), ws.numel(), st)
        parts.append(part)
    for order in (parts, parts[::-1]):
        total = torch.zeros_like(parts[0])
        for p in order:
            total += p
        fb.finish_device(total.data_ptr(), dst.data_ptr(), geo, s, a, bad.data_ptr(), st)
        torch.cuda.synchronize()
        assert np.array_equal(dst.cpu().numpy()[0], fb.bilateral_fast(img, s, a))
        assert int(bad.item()) == -1


@pytest.mark.parametrize("variant", ["fused", "naive"])
@pytest.mark.parametrize("n_lo,n_hi", [(0, 13), (0, 1), (3, 9), (12, 13)])
def test_partial_sums_match_the_oracle(oracle, variant, n_lo, n_hi):
    """GPU partial (Q, P) over [n_lo, n_hi) against the fp64 oracle's
    (fbo_partial_sums, bilateral.hpp:126-144 restricted to those harmonics)."""
    import torch
    c = CONFIGS["c1"]
    s, a = spatial_of(c), approx_of(c)
    img = image_of(c)[:96, :160].copy()
    geo = fb.whole_geometry(160, 96)
    src, ws, dst, bad = _bufs(img, geo, s, variant)
    st = torch.cuda.current_stream().cuda_stream
    fb.prepare_device(src.data_ptr(), geo, s, a, ws.data_ptr(), ws.numel(), st, variant)
    part = torch.zeros((1, 96, 160, 2), dtype=torch.float64, device=src.device)
    fb.partial_sums_device(part.data_ptr(), geo, s, a, n_lo, n_hi, ws.data_ptr(), ws.numel(), st, variant)
    torch.cuda.synchronize()
    got = part.cpu().numpy()[0]
    P, Q = oracle.partial_sums(img.astype(np.float64), s.profile, s.radius, a.d, a.omega, n_lo, n_hi)
    # the kernel works on f' = f - 128 (shift equivariance): P' = P - 128 Q
    assert float(np.abs(got[..., 0] - Q).max()) <= 2e-6
    assert float(np.abs(got[..., 1] - (P - 128.0 * Q)).max()) <= 5e-4


@pytest.mark.skipif("not __import__('torch').cuda.device_count() >= 2")
def test_harmonic_split_over_nccl_is_the_filter(tmp_path):
    """Two ranks over NCCL (needs two visible GPUs): harmonic_split_filter == one GPU, bit for bit."""
    import subprocess
    import sys
    import os
    script = tmp_path / "hs.py"
    script.write_text(HSPLIT_SCRIPT)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", str(script)],
                       capture_output=True, text=True, timeout=600, env=env, cwd=fb.__path__[0] + "/..")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "HSPLIT OK" in r.stdout


HSPLIT_SCRIPT = """
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of
from paper_1603_08081_b200.shard import harmonic_split_filter
rank = int(os.environ["RANK"]); torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
c = CONFIGS["c1"]; img, s, a = image_of(c), spatial_of(c), approx_of(c)
geo = fb.whole_geometry(c.width, c.height)
dev = torch.device("cuda", rank)
src = torch.from_numpy(img).to(dev)
ws = torch.empty(fb.workspace_bytes(geo, s.radius), dtype=torch.uint8, device=dev)
dst = torch.empty((1, c.height, c.width), dtype=torch.float32, device=dev)
bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
harmonic_split_filter(src, geo, s, a, ws, dst, bad)
torch.cuda.synchronize()
if rank == 0:
    assert np.array_equal(dst.cpu().numpy()[0], fb.bilateral_fast(img, s, a))
    print("HSPLIT OK")
dist.destroy_process_group()
"""
