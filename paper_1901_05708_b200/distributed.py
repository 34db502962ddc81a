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

PeerExchange is the fused alternative (the default of bench.py): the partial profiles live in
CUDA-IPC buffers every rank maps, and ONE kernel per rank (mprof_merge_finalize_peers) loads
the W partials of its slice over NVLink, merges, finalizes and stores the slice of (P, I)
straight into every rank's output buffers — no ncclMin, no separate finalize, no all-gather.
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


NO_INDEX32 = 0xFFFFFFFF  # "no neighbour" in a packed key: sorts after every real index


def pack_keys(cmp: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """FP32-mode merge keys, int64, ordered like the lexicographic (value, index) pairs of the
    float32-rounded values: high half = the float's order-preserving integer (non-negative
    floats keep their bits, negative ones map below them), low half = the uint32 index, "no
    neighbour" (idx < 0) packing as NO_INDEX32. Rounding to float32 is monotone, so the order
    is exact for the rounded values. Needs L < 2^32."""
    bits = cmp.to(torch.float32).view(torch.int32).to(torch.int64)
    high = torch.where(bits >= 0, bits, (~bits) - (1 << 31))
    low = torch.where(idx >= 0, idx, torch.full_like(idx, NO_INDEX32))
    return (high << 32) | low


def unpack_keys(key: torch.Tensor, cmp: torch.Tensor, idx: torch.Tensor) -> None:
    """Inverse of pack_keys into (cmp as float64 of the float32 value, idx with -1 restored)."""
    low = key & 0xFFFFFFFF
    idx.copy_(torch.where(low == NO_INDEX32, torch.full_like(low, -1), low))
    high = key >> 32
    bits = torch.where(high >= 0, high, ~(high + (1 << 31)))
    cmp.copy_(bits.to(torch.int32).view(torch.float32).to(torch.float64))


def merge_min_packed_(cmp: torch.Tensor, idx: torch.Tensor, group=None) -> None:
    """FP32 mode: the merge as ONE all-reduce(MIN) over packed 64-bit (value, index) keys (the
    north star's ncclMin on uint64 keys; 8 bytes per entry instead of two 8-byte passes). The
    FP32 sweep's candidate values are float-valued already; the FP64 seeds round to float32 here,
    which only reorders candidates that tie at float precision (inside FP32 mode's stated bound),
    and finalize recomputes the reported distance of the chosen pair in FP64."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    key = pack_keys(cmp, idx)
    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    unpack_keys(key, cmp, idx)


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


class PeerExchange:
    """Per-rank partial (cmp, idx) and output (P, I) buffers of L entries, allocated with
    mprof_ipc_alloc and mapped by every other rank (handles exchanged with all_gather_object).

    merge_finalize() runs after this rank's sweep wrote `cmp`/`idx`; afterwards `P`/`I` of EVERY
    rank hold the merged, finalized profile. Cross-rank ordering: barrier="nccl" uses a
    one-element all-reduce on the current stream as a stream-ordered barrier (no host sync, one
    process per GPU); barrier="host" synchronizes the device and calls dist.barrier (gloo, or
    several processes sharing a GPU, where NCCL cannot run)."""

    def __init__(self, mp, L: int, ctx=None, group=None, barrier: str = "host"):
        self.mp, self.L, self.ctx, self.group, self.barrier = mp, L, ctx, group, barrier
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world > mp.MAX_PEERS:
            raise ValueError(f"at most {mp.MAX_PEERS} ranks")
        self.own = {}
        handles = {}
        for k in ("cmp", "idx", "P", "I"):
            self.own[k], handles[k] = mp.ipc_alloc(8 * L, ctx=ctx)
        allh = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(allh, handles, group=group)
        else:
            allh = [handles]
        self.opened = []
        self.peer = {k: [] for k in ("cmp", "idx", "P", "I")}
        for r, h in enumerate(allh):
            for k in self.peer:
                if r == self.rank:
                    ptr = self.own[k]
                else:
                    ptr = mp.ipc_open(h[k], ctx=ctx)
                    self.opened.append(ptr)
                self.peer[k].append(ptr)
        self.cmp, self.idx, self.P, self.I = (self.own[k] for k in ("cmp", "idx", "P", "I"))

    def _barrier(self) -> None:
        if self.world == 1:
            return
        if self.barrier == "nccl":
            import torch
            if getattr(self, "_flag", None) is None:
                self._flag = torch.zeros(1, dtype=torch.int32, device="cuda")
            dist.all_reduce(self._flag, group=self.group)
        else:
            import torch
            torch.cuda.synchronize()
            dist.barrier(group=self.group)

    def merge_finalize(self, d_t: int, n: int, cfg) -> None:
        lo, hi = shard_range(self.L, self.rank, self.world)
        self._barrier()  # every rank's partial is complete
        self.mp.merge_finalize_peers(d_t, n, cfg, self.peer["cmp"], self.peer["idx"],
                                     self.peer["P"], self.peer["I"], lo, hi, ctx=self.ctx)
        self._barrier()  # every slice has landed in every rank's (P, I)

    def tensor(self, name: str):
        """Zero-copy torch view of this rank's own buffer ("cmp", "idx", "P" or "I")."""
        import torch

        class _Raw:
            pass
        raw = _Raw()
        raw.__cuda_array_interface__ = {
            "shape": (self.L,), "typestr": "<i8" if name in ("idx", "I") else "<f8",
            "data": (self.own[name], False), "version": 2, "strides": None}
        return torch.as_tensor(raw, device="cuda")

    def close(self) -> None:
        for ptr in self.opened:
            self.mp.ipc_close(ptr, ctx=self.ctx)
        self.opened = []
        for k in list(self.own):
            self.mp.ipc_free(self.own.pop(k), ctx=self.ctx)
