"""GPU: the device-resident C-ABI path (fbf_prepare_device + fbf_filter_prepared_device
on torch-allocated HBM buffers), as bench.py and the multi-GPU driver use it.

* row strips with W halo rows (the multi-GPU shard plan, emulated rank by rank
  on one GPU -- no rank waits on another) reassemble to the whole-image result
  bit for bit, at full BASELINE sizes (a size-independent property);
* the harmonic range is a pure function of the inputs (bit-identical reruns).
"""
import numpy as np
import pytest

import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, approx_of, image_of, spatial_of
from paper_1603_08081_b200.shard import geometry, plan

pytestmark = pytest.mark.gpu


def run_device(img_rows, geo, s, a, variant="fused", check_eps=True):
    import torch
    dev = torch.device("cuda", 0)
    src = torch.from_numpy(np.ascontiguousarray(img_rows, dtype=np.float32)).to(dev)
    nb = 1 if img_rows.ndim == 2 else img_rows.shape[0]
    dst = torch.empty((nb, geo.out_rows, geo.width), dtype=torch.float32, device=dev)
    ws_bytes = fb.workspace_bytes(geo, s.radius, variant)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    fb.prepare_device(src.data_ptr(), geo, s, a, ws.data_ptr(), ws_bytes, st, variant, check_eps)
    fb.filter_prepared_device(dst.data_ptr(), geo, s, a, ws.data_ptr(), ws_bytes, bad.data_ptr(), st, variant,
                              check_eps)
    torch.cuda.synchronize()
    assert int(bad.item()) == -1
    return dst.cpu().numpy()


@pytest.mark.parametrize("name,world", [("c2", 8), ("c4", 8), ("c1", 3), ("c3", 5)])
def test_row_strips_reassemble_bit_identically(name, world):
    c = CONFIGS[name]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    wg = fb.whole_geometry(c.width, c.height)
    whole = run_device(img, wg, s, a, check_eps=c.check_epsilon)[0]
    parts, groups = [], set()
    for r in range(world):
        sh = plan(c.width, c.height, 1, s.radius, world, r)
        g = geometry(sh, c.width, c.height)
        groups.add(fb.harmonic_groups(g, s.radius, a.N))
        parts.append(run_device(img[sh.src_row0:sh.src_row0 + sh.src_rows], g, s, a, check_eps=c.check_epsilon)[0])
    parts = np.concatenate(parts)
    # bit for bit, whatever harmonic grouping each strip picked (fixed-point sums)
    assert np.array_equal(parts, whole), sorted(groups)


def test_batch_shards_match_whole_batch():
    c = CONFIGS["c5"]
    s, a = spatial_of(c), approx_of(c)
    imgs = np.stack([image_of(c, i) for i in range(8)])
    whole = run_device(imgs, fb.whole_geometry(c.width, c.height, 8), s, a)
    for r in range(4):
        sh = plan(c.width, c.height, 8, s.radius, 4, r)
        part = run_device(imgs[sh.images], geometry(sh, c.width, c.height), s, a)
        assert np.array_equal(part, whole[sh.images])


def test_device_path_matches_host_path():
    c = CONFIGS["c1"]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    dev = run_device(img, fb.whole_geometry(c.width, c.height), s, a)[0]
    assert np.array_equal(dev, fb.bilateral_fast(img, s, a))


@pytest.mark.parametrize("shape", [(1536, 2048), (3, 1024, 1024), (4096, 1024)])
def test_pipelined_host_path_matches_one_launch(shape):
    """fbf_bilateral_fast_host cuts >= 1 Mpx calls into row strips (one image) or
    image chunks (batches) on two streams so the copies overlap the kernels.
    Each chunk picks its own harmonic grouping; the fixed-point (Q, P) sums
    make the result equal one launch bit for bit anyway."""
    c = CONFIGS["c2"]
    s, a = spatial_of(c), approx_of(c)
    rng = np.random.default_rng(sum(shape))
    img = np.clip(rng.normal(128, 60, shape), 0, 255).astype(np.float32)
    batch = 1 if len(shape) == 2 else shape[0]
    h, w = shape[-2], shape[-1]
    dev = run_device(img.reshape(batch, h, w), fb.whole_geometry(w, h, batch), s, a).reshape(shape)
    assert np.array_equal(dev, fb.bilateral_fast(img, s, a))


def test_pipelined_host_path_reports_the_first_collapse():
    rng = np.random.default_rng(9)
    img = rng.integers(0, 256, (1536, 2048)).astype(np.float32)
    lying = fb.FourierKernelApprox(255, np.pi / 255, 0, np.array([0.0]), 0.0, 0.0)
    with pytest.raises(fb.FilterError, match=r"pixel \(0, 0\)"):
        fb.bilateral_fast(img, fb.make_spatial_gaussian(2.0), lying)


def test_host_entry_is_reentrant_across_threads():
    """bilateral.hpp's contract (SURVEY §8(b) threading): pure and reentrant;
    the host entry keeps one stream / buffer / graph per calling thread."""
    import threading
    c = CONFIGS["c1"]
    s, a = spatial_of(c), approx_of(c)
    rng = np.random.default_rng(77)
    imgs = [np.clip(rng.normal(128, 60, (300 + 40 * k, 280)), 0, 255).astype(np.float32) for k in range(4)]
    want = [fb.bilateral_fast(im, s, a) for im in imgs]
    got = [[None] * 4 for _ in range(2)]
    errors = []

    def worker(t):
        try:
            for rep in range(3):
                for k in range(4):
                    got[t][k] = fb.bilateral_fast(imgs[(k + t) % 4], s, a)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors
    for t in range(2):
        for k in range(4):
            assert np.array_equal(got[t][k], want[(k + t) % 4])


def test_group_model_picks_and_finish_mode():
    """The harmonic-group model (the kernel's own cuts replayed on the launch plan): c2 splits its
    harmonics in two (step granularity + prologues), the long runs of c4 / c5 stay in one group, the small
    c1 takes one harmonic per group; the count never exceeds the planes the workspace holds (16).  With
    groups the n = 0 kernel closes the call in finish mode: three launches (prep, fused, n = 0), and the
    result equals the partial-sums route (fused + finish_groups) bit for bit."""
    import torch
    picks = {}
    for name, c in CONFIGS.items():
        g = fb.whole_geometry(c.width, c.height, c.batch)
        picks[name] = fb.harmonic_groups(g, spatial_of(c).radius, c.N)
        assert 1 <= picks[name] <= 16
        assert fb.launches_per_call(g, spatial_of(c), approx_of(c)) == 3
    assert picks["c2"] == 2 and picks["c4"] == 1 and picks["c5"] == 1 and picks["c1"] >= 6, picks
    # finish mode (filter) against partial sums over the full range + fbf_finish_device
    c = CONFIGS["c1"]
    img, s, a = image_of(c), spatial_of(c), approx_of(c)
    geo = fb.whole_geometry(c.width, c.height)
    out = run_device(img, geo, s, a)[0]
    dev = torch.device("cuda", 0)
    src = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).to(dev)
    ws = torch.empty(fb.workspace_bytes(geo, s.radius, "fused"), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    fb.prepare_device(src.data_ptr(), geo, s, a, ws.data_ptr(), ws.numel(), st)
    pq = torch.empty((c.height, c.width, 2), dtype=torch.float64, device=dev)
    fb.partial_sums_device(pq.data_ptr(), geo, s, a, 0, a.N + 1, ws.data_ptr(), ws.numel(), st)
    dst = torch.empty((c.height, c.width), dtype=torch.float32, device=dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    fb.finish_device(pq.data_ptr(), dst.data_ptr(), geo, s, a, bad.data_ptr(), st)
    torch.cuda.synchronize()
    assert int(bad.item()) == -1
    assert np.array_equal(dst.cpu().numpy(), out)
