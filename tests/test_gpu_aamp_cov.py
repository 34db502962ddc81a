"""The covariance-form AAMP kernel (EuclidCov, sweep.cuh): chosen automatically for long windows of
large series (window-scale spread >= kAampCovMinSpread, confirmed by the form probe), forced here
through mprof_ctx_set_form(COV) on small ones. It slides the centred covariance (2 DFMA per cell) and forms
D^2 = S_i + S_j + m (mu_i - mu_j)^2 - 2 cov only for candidate cells. The profile must obey the
same parity rules against the oracle (which restates EuclidScan, /root/reference/proj/src/
diag_scan.cpp:7-24) as the (delta, sigma) kernel, including level-offset series, exact copies
(ties at distance 0) and band merges."""
import numpy as np
import pytest

import oracle
from oracle import EUCLIDEAN
from oracle.parity import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(mp):
    c = mp.Context(0)
    c.set_form(mp.Form.Cov)
    yield c
    c.close()


def _aamp(mp, ctx, t, m, exclusion=1):
    cfg = mp.ProfileConfig(m, mp.DistanceKind.euclidean())
    cfg.exclusion = exclusion
    return mp.aamp(mp.make_time_series(t), cfg, ctx=ctx)


def _parity(t, m, r, exclusion=1):
    _, Pr, Ir = oracle.scan(t, m, EUCLIDEAN, 2.0, exclusion=exclusion)
    rep = check(t, m, EUCLIDEAN, r.distances, r.nn_index, Pr, Ir, tol=1e-9, p=2.0)
    assert rep.ok, rep.summary()
    ok = r.nn_index >= 0
    assert np.all(np.abs(r.nn_index[ok] - np.arange(ok.size)[ok]) >= exclusion)


@pytest.mark.parametrize("exclusion", [1, 700])
def test_cov_form_random_walk(mp, ctx, exclusion):
    t = np.cumsum(np.random.default_rng(5).standard_normal(12000))
    r = _aamp(mp, ctx, t, 1024, exclusion)
    assert r.info.fp64_ops_per_cell == 2.0  # the covariance form was chosen
    _parity(t, 1024, r, exclusion)


def test_cov_form_level_offset(mp, ctx):
    r0 = np.random.default_rng(6)
    t = 1e6 + np.cumsum(r0.standard_normal(9000))
    r = _aamp(mp, ctx, t, 600)
    assert r.info.fp64_ops_per_cell == 2.0
    _parity(t, 600, r)


def test_cov_form_exact_copies(mp, ctx):
    r0 = np.random.default_rng(8)
    t = np.cumsum(r0.standard_normal(14000))
    seg = t[1000:2600].copy()
    for s in (5000, 9000, 12000):  # three exact copies of the segment
        t[s:s + seg.size] = seg
    m = 1024
    r = _aamp(mp, ctx, t, m)
    assert r.info.fp64_ops_per_cell == 2.0
    _parity(t, m, r)
    # windows inside a copy have an exact duplicate: distance exactly 0 (finalize recomputes it)
    for s in (1000, 5000, 9000, 12000):
        for i in (s, s + 100, s + seg.size - m):
            assert r.distances[i] == 0.0


def test_cov_form_bands_merge(mp, ctx):
    torch = pytest.importorskip("torch")
    t = np.cumsum(np.random.default_rng(9).standard_normal(10000))
    m = 1024
    n, L = t.size, t.size - m + 1
    cfg = mp.ProfileConfig(m, mp.DistanceKind.euclidean())
    d_t = torch.tensor(t, device="cuda")
    cm = torch.full((L,), float("inf"), dtype=torch.float64, device="cuda")
    im = torch.full((L,), -1, dtype=torch.int64, device="cuda")
    cuts = mp.band_cuts(n, m, 1, 3)
    for a, b in zip(cuts[:-1], cuts[1:]):
        c = torch.empty(L, dtype=torch.float64, device="cuda")
        i = torch.empty(L, dtype=torch.int64, device="cuda")
        info = mp.sweep_device(d_t.data_ptr(), n, cfg, a, b, c.data_ptr(), i.data_ptr(), ctx=ctx)
        assert info.fp64_ops_per_cell == 2.0
        torch.cuda.synchronize()
        mp.merge_device(cm.data_ptr(), im.data_ptr(), c.data_ptr(), i.data_ptr(), L)
    P = torch.empty(L, dtype=torch.float64, device="cuda")
    mp.finalize_device(d_t.data_ptr(), n, cm.data_ptr(), im.data_ptr(), cfg, P.data_ptr())
    torch.cuda.synchronize()

    class R:
        distances = P.cpu().numpy()
        nn_index = im.cpu().numpy()
    _parity(t, m, R)


def test_cov_form_falls_back_beyond_float_range(mp, ctx):
    # means beyond the float filter tables' range: the (delta, sigma) kernel runs instead
    t = np.cumsum(np.random.default_rng(10).standard_normal(6000))
    t[3000:] += 1e31
    r = _aamp(mp, ctx, t, 1024)
    assert r.info.fp64_ops_per_cell == 3.0
    assert np.all(np.isfinite(r.distances))
