"""Multi-GPU plumbing: one process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).

The sweep shards with no data-path exchange: rank g sweeps the diagonal band
[cuts[g], cuts[g+1]) of equal triangle area (mprof_band_cuts) into a partial comparison-space
profile (cmp, idx) — the reference's own worker decomposition
(/root/reference/proj/src/detail/diag_scan.hpp:228-256) lifted to GPUs. The single exchange is
the final MinBuffer::absorb (diag_scan.hpp:45-52), done here as two all-reduce(MIN) calls
(ncclMin over float64 values, then over the int64 indices of the ranks that hold the minimum),
which reproduces the lexicographic (value, index) minimum exactly. The finalize (distance of each
chosen pair recomputed directly) is split the same way: rank g converts entries
shard_range(L, g, world) with mprof_finalize_range_device and the slices are all-gathered.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import band_cuts

INT64_MAX = (1 << 63) - 1


def band_for_rank(n: int, m: int, exclusion: int, rank: int, world: int) -> tuple[int, int]:
    cuts = band_cuts(n, m, exclusion, world)
    return cuts[rank], cuts[rank + 1]


def merge_min_(cmp: torch.Tensor, idx: torch.Tensor, group=None) -> None:
    """In-place lexicographic (cmp, idx) minimum across ranks. idx < 0 means "no neighbour"
    (cmp = +inf there). Works for CUDA tensors on NCCL and CPU tensors on gloo."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    gmin = cmp.clone()
    dist.all_reduce(gmin, op=dist.ReduceOp.MIN, group=group)
    cand = torch.where((cmp == gmin) & (idx >= 0), idx, torch.full_like(idx, INT64_MAX))
    dist.all_reduce(cand, op=dist.ReduceOp.MIN, group=group)
    cmp.copy_(gmin)
    idx.copy_(torch.where(cand == INT64_MAX, torch.full_like(idx, -1), cand))


def shard_size(L: int, world: int) -> int:
    return -(-L // world)


def shard_range(L: int, rank: int, world: int) -> tuple[int, int]:
    """Entries [lo, hi) of an L-entry profile this rank finalizes (equal slices, last one short)."""
    s = shard_size(L, world)
    return min(L, rank * s), min(L, (rank + 1) * s)


def gather_shards_(x: torch.Tensor, group=None) -> None:
    """x has world * shard_size entries; rank g owns slice g. Afterwards every rank holds every
    slice (NCCL all-gather in place; gloo via a list gather)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    s = x.numel() // world
    mine = x[rank * s:(rank + 1) * s]
    if x.is_cuda:
        dist.all_gather_into_tensor(x, mine, group=group)
    else:
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine.clone(), group=group)
        x.copy_(torch.cat(parts))


def finalize_sharded(mp, d_t: int, n: int, cmp: torch.Tensor, idx: torch.Tensor, cfg,
                     P: torch.Tensor, ctx=None, group=None) -> None:
    """Merged (cmp, idx) on every rank -> P (length world * shard_size(L), first L valid) on
    every rank, each rank finalizing only its own slice."""
    L = cmp.numel()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(L, rank, world)
    mp.finalize_range_device(d_t, n, cmp.data_ptr(), idx.data_ptr(), cfg, P.data_ptr(), lo, hi,
                             ctx=ctx)
    gather_shards_(P, group)
