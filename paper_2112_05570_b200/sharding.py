"""Multi-GPU plumbing: rays shard by global index, the mesh is replicated, and
the only collective is one all-reduce of the per-GPU histograms (K7).

The reference is single-process; queries are pure and may
run concurrently, so sharding by ray index reproduces the
single-GPU per-ray results exactly and the summed histograms equal the
single-GPU histogram.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    first: int  # first global ray index of this rank
    count: int  # rays traced by this rank


def weak_shard(rank: int, world: int, rays_per_rank: int) -> Shard:
    """Per-rank work fixed: rank r traces global indices [r*n, (r+1)*n)."""
    if not (0 <= rank < world) or rays_per_rank < 0:
        raise ValueError("bad shard arguments")
    return Shard(rank * rays_per_rank, rays_per_rank)


def strong_shard(rank: int, world: int, total: int) -> Shard:
    """Total work fixed: contiguous near-equal ranges [floor(r*N/W), floor((r+1)*N/W))."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard arguments")
    lo = rank * total // world
    hi = (rank + 1) * total // world
    return Shard(lo, hi - lo)


def allreduce_histogram(hist, group=None):
    """Sum the int64 histograms of all ranks in place (NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def histogram_host(seg, steps, status=None):
    """Host restatement of the K7 histogram layout (include/mwt.h MWT_HIST_*)
    for per-ray results that already live on the host."""
    import numpy as np

    from . import _lib
    h = np.zeros(_lib.HIST_LEN, dtype=np.int64)
    steps = np.asarray(steps, dtype=np.int64)
    bins = np.clip(steps, 0, _lib.HIST_STEP_BINS - 1)
    h[:_lib.HIST_STEP_BINS] = np.bincount(bins, minlength=_lib.HIST_STEP_BINS)
    seg = np.asarray(seg)
    h[_lib.HIST_HIT] = int((seg >= 0).sum())
    h[_lib.HIST_MISS] = int((seg < 0).sum())
    h[_lib.HIST_STEPS_SUM] = int(np.clip(steps, 0, None).sum())
    if status is not None:
        st = np.asarray(status, dtype=np.uint32)
        for b in range(12):
            h[_lib.HIST_STATUS0 + b] = int(((st >> b) & 1).sum())
    return h
