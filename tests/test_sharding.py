"""CPU, world_size 2 over gloo: the multi-GPU partition (paper_1603_08081_b200.shard)
is exact.  Each rank filters its own strip / images with the fp64 oracle from
only the source rows its plan holds, the strips are gathered over gloo, and the
reassembled image must equal the whole-image oracle bit for bit.  The same
plans are checked against the C-ABI's halo validation (used by every launch)."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.shard import geometry, mirror_index, plan, source_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plan_covers_and_halos_are_exact():
    for (h, W, world) in ((100, 9, 2), (100, 9, 8), (64, 24, 8), (7, 3, 4), (2048, 15, 8), (10, 12, 3)):
        seen = []
        for r in range(world):
            s = plan(37, h, 1, W, world, r)
            seen += list(range(s.out_row0, s.out_row0 + s.out_rows))
            need = {mirror_index(y + k, h) for y in range(s.out_row0, s.out_row0 + s.out_rows)
                    for k in range(-W, W + 1)}
            if need:
                assert min(need) >= s.src_row0 and max(need) < s.src_row0 + s.src_rows
                assert (s.src_row0, s.src_row0 + s.src_rows) == (min(need), max(need) + 1)
        assert seen == list(range(h))
    # batches split by image, no halo
    parts = [plan(16, 16, 10, 4, 4, r) for r in range(4)]
    assert sum((p.images for p in parts), []) == list(range(10))
    assert all(p.src_rows == 16 and p.out_rows == 16 for p in parts)


def test_plans_pass_the_abi_halo_check():
    s, a = fb.make_spatial_gaussian(5.0), fb.fit_fixed(0, 20.0, 255, 20)  # config c2
    f = fb._filter_struct(s, a)
    for r in range(8):
        g = geometry(plan(2048, 2048, 1, s.radius, 8, r), 2048, 2048)
        rc = fb.lib.fbf_bilateral_fast_device(ctypes.byref(g), ctypes.byref(f), None, None, None, 0, None, 0,
                                              None)
        # validation passes geometry + halo and stops at the (absent) workspace
        assert rc == fb.FBF_EINVAL and "workspace" in fb.lib.fbf_last_error().decode()


def _worker(rank, world, port, img, W, prof, w0, d, eps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle
    h, w = img.shape
    s = plan(w, h, 1, W, world, rank)
    held = img[s.src_row0:s.src_row0 + s.src_rows]          # only the rows the plan ships
    # embed the held rows at their global position (rows outside are poisoned)
    local = np.full_like(img, np.nan)
    local[s.src_row0:s.src_row0 + s.src_rows] = held
    out, rc, _ = Oracle().bilateral_fast(local, prof, W, w0, d, np.pi / 255, eps, True, s.out_row0,
                                         s.out_row0 + s.out_rows)
    parts = [None] * world
    dist.all_gather_object(parts, (s.out_row0, out))
    if rank == 0:
        q.put(parts)
    dist.barrier()
    dist.destroy_process_group()


def _hsplit_worker(rank, world, port, img, W, prof, d, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle
    from paper_1603_08081_b200.shard import harmonic_range
    n_lo, n_hi = harmonic_range(len(d) - 1, world, rank)
    P, Q = Oracle().partial_sums(img, prof, W, d, np.pi / 255, n_lo, n_hi)
    t = torch.from_numpy(np.stack([P, Q]))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)  # the NCCL all-reduce of the GPU path, on gloo
    if rank == 0:
        q.put(t.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_harmonic_split_over_gloo_sums_to_the_whole(oracle, world):
    """Harmonic-split mode: per-rank partial (P, Q) over disjoint harmonic ranges,
    summed by an all-reduce, divided -> the whole filter (to rounding)."""
    rng = np.random.default_rng(9)
    img = rng.integers(0, 256, (29, 23)).astype(np.float64)
    W, prof, w0 = oracle.spatial_gaussian(1.5)
    d, _, eps = oracle.fit_fixed(0, 25.0, 255, 13)
    whole, rc, _ = oracle.bilateral_fast(img, prof, W, w0, d, np.pi / 255, eps)
    assert rc == 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_hsplit_worker, args=(r, world, port, img, W, prof, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    PQ = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.allclose(PQ[0] / PQ[1], whole, rtol=0, atol=1e-10)


@pytest.mark.parametrize("world", [2])
def test_strips_over_gloo_reassemble_bit_identically(oracle, world):
    rng = np.random.default_rng(7)
    img = rng.integers(0, 256, (53, 31)).astype(np.float64)
    W, prof, w0 = oracle.spatial_gaussian(2.0)
    d, _, eps = oracle.fit_fixed(0, 25.0, 255, 9)
    whole, rc, _ = oracle.bilateral_fast(img, prof, W, w0, d, np.pi / 255, eps)
    assert rc == 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, img, W, prof, w0, d, eps, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([o for _, o in sorted(parts, key=lambda t: t[0])])
    assert np.array_equal(got, whole)  # no NaN leaked in: the halo held every row read
