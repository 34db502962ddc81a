"""Fused multi-process merge over peer memory (mprof_merge_finalize_peers + CUDA IPC buffers,
paper_1901_05708_b200.distributed.PeerExchange): W processes each sweep one equal-area diagonal
band, then ONE kernel per rank merges the W partial profiles of its slice (lexicographic
MinBuffer::absorb, /root/reference/proj/src/detail/diag_scan.hpp:45-52), finalizes it and stores
it into every rank's (P, I). Here all ranks share cuda:0 (IPC works between processes on one
device; host barriers over gloo order them, no kernel waits on another process): the result must
equal the single-process profile — bit-identical in the parity build (exact mode), within the
parity rules of the oracle in the fast mode."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as tmp  # noqa: E402

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, t, m, fam, p, excl, exact, out_dir):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import paper_1901_05708_b200 as mp
    from paper_1901_05708_b200.distributed import PeerExchange, band_for_rank

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    kind = {0: mp.DistanceKind.euclidean(), 1: mp.DistanceKind.pnorm(p),
            2: mp.DistanceKind.znormalized()}[fam]
    cfg = mp.ProfileConfig(m, kind)
    cfg.exclusion = excl
    if exact:
        cfg.exact, cfg.refresh_interval = True, 256
    n = t.size
    L = n - m + 1
    px = PeerExchange(mp, L, barrier="host")
    d_t = torch.tensor(t, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    k_lo, k_hi = band_for_rank(n, m, excl, rank, world)
    mp.sweep_device(d_t.data_ptr(), n, cfg, k_lo, k_hi, px.cmp, px.idx)
    px.merge_finalize(d_t.data_ptr(), n, cfg)
    np.save(os.path.join(out_dir, f"P{rank}.npy"), px.tensor("P").cpu().numpy())
    np.save(os.path.join(out_dir, f"I{rank}.npy"), px.tensor("I").cpu().numpy())
    dist.barrier()
    px.close()
    dist.destroy_process_group()


def _run(tmp_path, world, t, m, fam, p, excl, exact):
    tmp.spawn(_worker, args=(world, _free_port(), t, m, fam, p, excl, exact, str(tmp_path)),
              nprocs=world, join=True)
    P = [np.load(tmp_path / f"P{r}.npy") for r in range(world)]
    I = [np.load(tmp_path / f"I{r}.npy") for r in range(world)]
    for r in range(1, world):  # every rank holds the same whole profile
        assert np.array_equal(P[r], P[0]) and np.array_equal(I[r], I[0])
    return P[0], I[0]


def _series(seed, n=6000):
    r = np.random.default_rng(seed)
    t = 20 + np.cumsum(r.standard_normal(n))
    t[2000:2300] = t[2000]  # flat run (z-norm ties at the flat convention)
    return t


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("fam,p,excl", [(0, 2.0, 1), (1, 3.0, 7), (2, 2.0, 1), (2, 2.0, 64)])
def test_peer_merge_matches_oracle(mp, tmp_path, world, fam, p, excl):
    import oracle
    from oracle.parity import check
    t = _series(world * 7 + fam)
    m = 64
    P, I = _run(tmp_path, world, t, m, fam, p, excl, False)
    _, Pr, Ir = oracle.scan(t, m, fam, p, exclusion=excl)
    rep = check(t, m, fam, P, I, Pr, Ir, tol=1e-9, p=p, abs_bound=2e-6 if fam == 2 else None)
    assert rep.ok, rep.summary()


@pytest.mark.parametrize("fam,p", [(0, 2.0), (1, 1.0)])
def test_peer_merge_exact_mode_bit_identical(mp, tmp_path, fam, p):
    t = _series(99 + fam)
    m = 64
    P, I = _run(tmp_path, 3, t, m, fam, p, 1, True)
    kind = mp.DistanceKind.euclidean() if fam == 0 else mp.DistanceKind.pnorm(p)
    cfg = mp.ProfileConfig(m, kind)
    cfg.exact, cfg.refresh_interval = True, 256
    single = (mp.aamp if fam == 0 else mp.aamp_pnorm)(mp.make_time_series(t), cfg)
    assert np.array_equal(I, single.nn_index)
    assert np.array_equal(P, single.distances)


def test_peer_merge_validation(mp):
    d = torch.zeros(8, dtype=torch.float64, device="cuda")
    cfg = mp.ProfileConfig(4, mp.DistanceKind.euclidean())
    with pytest.raises(mp.Error) as e:
        mp.merge_finalize_peers(d.data_ptr(), 8, cfg, [], [], [d.data_ptr()], [d.data_ptr()], 0, 5)
    assert e.value.code == mp.ErrorCode.BadArgument
    with pytest.raises(mp.Error) as e:
        mp.ipc_open(b"\0" * 63)
    assert e.value.code == mp.ErrorCode.BadArgument
