"""Multi-GPU work partitioning for one 8xB200 box.

Every output pixel depends only on input pixels within W rows/columns, so the
path partitions with no data exchange:

* one large image  -> row strips: rank r produces rows [r*H/G, (r+1)*H/G) and
  holds those rows plus W halo rows above and below (mirror padding only at the
  global image edges, via the geometry's global row index);
* a batch of images -> images split evenly by rank, no halo.

No collective touches the data path; the launcher only uses torch.distributed
for the start/stop barrier and the max-over-ranks timing.  The strip plan is
exact: the union of the ranks' outputs is the whole image and each strip's
source rows are exactly the (mirrored) rows its outputs read.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List


ROW_ALIGN = 16  # = the fused kernel's rows per column-pass block (KC)


@dataclass(frozen=True)
class Shard:
    images: List[int]   # batch indices owned by the rank
    out_row0: int       # first output row (global)
    out_rows: int
    src_row0: int       # first source row held (global), includes the halo
    src_rows: int


def mirror_index(i: int, n: int) -> int:
    """image.hpp:34-40"""
    if 0 <= i < n:
        return i
    period = 2 * n
    j = i % period
    return j if j < n else period - 1 - j


def source_rows(out_row0: int, out_rows: int, height: int, radius: int):
    """[lo, hi) of the global rows that output rows [out_row0, out_row0+out_rows) read."""
    rows = {mirror_index(y + k, height)
            for y in list(range(out_row0, min(out_row0 + out_rows, out_row0 + 2 * radius + 1)))
            + list(range(max(out_row0, out_row0 + out_rows - 2 * radius - 1), out_row0 + out_rows))
            for k in range(-radius, radius + 1)}
    return min(rows), max(rows) + 1


def plan(width: int, height: int, batch: int, radius: int, world: int, rank: int) -> Shard:
    if not 0 <= rank < world:
        raise ValueError("rank outside the world")
    if batch > 1:
        b0, b1 = batch * rank // world, batch * (rank + 1) // world
        return Shard(list(range(b0, b1)), 0, height, 0, height)
    # cuts on multiples of ROW_ALIGN: the kernel's column-pass blocks then start
    # at the same global rows as in a single-GPU run (bit-identical results)
    def cut(k):
        return 0 if k == 0 else height if k == world else (height * k // world) // ROW_ALIGN * ROW_ALIGN
    r0, r1 = cut(rank), cut(rank + 1)
    lo, hi = source_rows(r0, r1 - r0, height, radius) if r1 > r0 else (r0, r0)
    return Shard([0], r0, r1 - r0, lo, hi - lo)


def harmonic_range(N: int, world: int, rank: int):
    """[n_lo, n_hi) of the harmonics 0..N assigned to `rank` in the harmonic-split mode."""
    return (N + 1) * rank // world, (N + 1) * (rank + 1) // world


def harmonic_split_filter(src, geo, spatial, approx, workspace, dst, bad, group=None, variant="fused",
                          check_epsilon=True):
    """Harmonic-split mode: every rank holds the whole image,
    computes the (Q, P) partial sums of its harmonic range, the partial planes
    are summed over ranks with one NCCL all-reduce over NVLink, and every rank
    divides.  For single images too small to split by rows.  `src`, `dst`,
    `workspace`, `bad` are torch CUDA tensors; returns nothing (dst filled)."""
    import torch
    import torch.distributed as dist
    from . import finish_device, partial_sums_device, prepare_device
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n_lo, n_hi = harmonic_range(approx.N, world, rank)
    st = torch.cuda.current_stream().cuda_stream
    # exact fp64 partial sums (multiples of the call's fixed-point grid): the
    # all-reduce adds them exactly, so the result is the single-GPU bits
    pq = torch.zeros((geo.batch, geo.out_rows, geo.width, 2), dtype=torch.float64, device=src.device)
    prepare_device(src.data_ptr(), geo, spatial, approx, workspace.data_ptr(), workspace.numel(), st, variant,
                   check_epsilon)
    if n_hi > n_lo:
        partial_sums_device(pq.data_ptr(), geo, spatial, approx, n_lo, n_hi, workspace.data_ptr(),
                            workspace.numel(), st, variant, check_epsilon)
    if world > 1:
        dist.all_reduce(pq, op=dist.ReduceOp.SUM, group=group)
    finish_device(pq.data_ptr(), dst.data_ptr(), geo, spatial, approx, bad.data_ptr(), st, check_epsilon)


def geometry(shard: Shard, width: int, height: int):
    """fbf_geometry for a rank's shard (dense per-image buffers)."""
    from . import Geometry, whole_geometry
    if len(shard.images) > 1 or shard.src_rows == height:
        g = whole_geometry(width, height, len(shard.images))
        g.out_row0, g.out_rows = shard.out_row0, shard.out_rows
        g.dst_bstride = shard.out_rows * width
        return g
    g = Geometry()
    g.width, g.height, g.batch = width, height, 1
    g.src_row0, g.src_rows = shard.src_row0, shard.src_rows
    g.out_row0, g.out_rows = shard.out_row0, shard.out_rows
    g.src_pitch = g.dst_pitch = width
    g.src_bstride = shard.src_rows * width
    g.dst_bstride = shard.out_rows * width
    return g
