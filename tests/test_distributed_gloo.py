"""Multi-process merge path on CPU (gloo, world_size 2 and 3): each rank produces the partial
comparison-space profile of its equal-area diagonal band (here with the CPU oracle standing in
for the GPU sweep), then paper_1901_05708_b200.distributed.merge_min_ (two all_reduce(MIN)
calls, the ncclMin merge the GPU ranks use) must reproduce the single-process profile exactly —
MinBuffer::absorb semantics (/root/reference/proj/src/detail/diag_scan.hpp:45-52)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as tmp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_dir, packed=False):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import oracle
    from paper_1901_05708_b200.distributed import band_for_rank, merge_min_, merge_min_packed_

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t, m, fam, p, excl = case
    k_lo, k_hi = band_for_rank(t.size, m, excl, rank, world)
    cmp, _, idx = oracle.scan(t, m, fam, p, exclusion=excl, k_lo=k_lo, k_hi=k_hi, threads=1)
    c = torch.from_numpy(cmp.copy())
    i = torch.from_numpy(idx.copy())
    if packed:
        c = c.to(torch.float32).to(torch.float64)  # FP32-mode partials hold float values
        merge_min_packed_(c, i)
    else:
        merge_min_(c, i)
    if rank == 0:
        np.save(os.path.join(out_dir, "cmp.npy"), c.numpy())
        np.save(os.path.join(out_dir, "idx.npy"), i.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("fam,p,excl", [(0, 2.0, 1), (1, 3.0, 5), (2, 2.0, 1)])
def test_band_merge_matches_single_process(tmp_path, world, fam, p, excl):
    import oracle
    r = np.random.default_rng(world * 10 + fam)
    t = np.cumsum(r.standard_normal(900))
    if fam == 2:
        t[100:160] = t[100]  # flat run: exact ties at -m^2
        t[600:640] = t[600]
    m = 24
    case = (t, m, fam, p, excl)
    tmp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    cmp = np.load(tmp_path / "cmp.npy")
    idx = np.load(tmp_path / "idx.npy")
    c_full, _, i_full = oracle.scan(t, m, fam, p, exclusion=excl, threads=1)
    assert np.array_equal(cmp, c_full)
    assert np.array_equal(idx, i_full)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("fam,p,excl", [(0, 2.0, 1), (2, 2.0, 7)])
def test_packed_key_merge_matches_float_lexicographic_min(tmp_path, world, fam, p, excl):
    """FP32-mode merge (one all-reduce over packed 64-bit keys) = the lexicographic (value,
    index) minimum of the float32-rounded band partials, entry by entry."""
    import oracle
    from paper_1901_05708_b200.distributed import band_for_rank
    r = np.random.default_rng(40 + world * 10 + fam)
    t = np.cumsum(r.standard_normal(700))
    if fam == 2:
        t[200:260] = t[200]
    m = 20
    case = (t, m, fam, p, excl)
    tmp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path), True), nprocs=world,
              join=True)
    cmp = np.load(tmp_path / "cmp.npy")
    idx = np.load(tmp_path / "idx.npy")
    L = t.size - m + 1
    best_v = np.full(L, np.inf)
    best_i = np.full(L, np.iinfo(np.int64).max)
    for g in range(world):
        k_lo, k_hi = band_for_rank(t.size, m, excl, g, world)
        c, _, i = oracle.scan(t, m, fam, p, exclusion=excl, k_lo=k_lo, k_hi=k_hi, threads=1)
        v = c.astype(np.float32).astype(np.float64)
        ii = np.where(i >= 0, i, np.iinfo(np.int64).max)
        better = (v < best_v) | ((v == best_v) & (ii < best_i))
        best_v = np.where(better, v, best_v)
        best_i = np.where(better, ii, best_i)
    best_i = np.where(best_i == np.iinfo(np.int64).max, -1, best_i)
    assert np.array_equal(cmp, best_v)
    assert np.array_equal(idx, best_i)
    # and the argmin agrees with the FP64 merge wherever the float rounding separates values
    c_full, _, i_full = oracle.scan(t, m, fam, p, exclusion=excl, threads=1)
    assert np.mean(idx == i_full) > 0.95


def test_pack_keys_roundtrip_and_order():
    from paper_1901_05708_b200.distributed import pack_keys, unpack_keys
    c = torch.tensor([0.0, 1.5, 1.5, np.inf, 2.0, 0.25, -3.0, -0.5, -3.0], dtype=torch.float64)
    i = torch.tensor([3, 7, 2, -1, 0, 9, 4, 1, 0], dtype=torch.int64)
    k = pack_keys(c, i)
    order = torch.argsort(k).tolist()
    assert order == [8, 6, 7, 0, 5, 2, 1, 4, 3]  # by value, ties by index, (+inf, none) last
    c2, i2 = torch.empty_like(c), torch.empty_like(i)
    unpack_keys(k, c2, i2)
    assert torch.equal(c2, c) and torch.equal(i2, i)


def test_band_partition_covers_every_diagonal_once():
    from paper_1901_05708_b200.distributed import band_for_rank
    n, m, excl = 5000, 37, 3
    for world in (1, 2, 4, 8):
        bands = [band_for_rank(n, m, excl, r, world) for r in range(world)]
        assert bands[0][0] == excl and bands[-1][1] == n - m + 1
        assert all(a[1] == b[0] for a, b in zip(bands[:-1], bands[1:]))


def _gather_worker(rank, world, port, L, out_dir):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_1901_05708_b200.distributed import gather_shards_, shard_range, shard_size

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = torch.full((world * shard_size(L, world),), -1.0, dtype=torch.float64)
    lo, hi = shard_range(L, rank, world)
    x[lo:hi] = torch.arange(lo, hi, dtype=torch.float64) * 0.5  # this rank's finalized slice
    gather_shards_(x)
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x[:L].numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 7), (3, 10), (3, 3), (4, 2)])
def test_sharded_finalize_gather(tmp_path, world, L):
    """Range-split finalize: every rank ends with all L entries, each written by its owner."""
    tmp.spawn(_gather_worker, args=(world, _free_port(), L, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"x{r}.npy"), np.arange(L) * 0.5)
