"""Multi-GPU plumbing: one process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).

The sweep shards with no data-path exchange: rank g sweeps the diagonal band
[cuts[g], cuts[g+1]) of equal triangle area (mprof_band_cuts) into a partial comparison-space
profile (cmp, idx) — the reference's own worker decomposition
(/root/reference/proj/src/detail/diag_scan.hpp:228-256) lifted to GPUs. The single exchange is
the final MinBuffer::absorb (diag_scan.hpp:45-52), done here as two all-reduce(MIN) calls
(ncclMin over float64 values, then over the int64 indices of the ranks that hold the minimum),
which reproduces the lexicographic (value, index) minimum exactly.
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
