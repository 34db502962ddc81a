"""Streaming extension: build_engine_state / extend_profile. The reference's
acceptance criterion 7 (/root/reference/proj/tests/acceptance.cpp:252-286): 50 rounds of
random series, a build over the first n0 samples, an extension by 1..40 samples, compared with a
from-scratch run of the whole series (1e-9 and identical indices there). The GPU extension plans
the extended series as a fresh build would and sweeps only the fresh sweep's tiles that hold new
cells (the stored entries seed the rest), so the grown profile is BIT-IDENTICAL to a fresh GPU
profile of the extended series (tests/test_engine_state.cpp:31-37 checks it with ==), and within
the parity rules of the oracle."""
import numpy as np
import pytest

import oracle
from oracle import EUCLIDEAN, PNORM, ZNORM
from oracle.parity import check

pytestmark = pytest.mark.gpu


def kind(mp, fam, p):
    return {EUCLIDEAN: mp.DistanceKind.euclidean(), PNORM: mp.DistanceKind.pnorm(p),
            ZNORM: mp.DistanceKind.znormalized()}[fam]


def test_extension_equals_recompute_corpus(mp):
    r = np.random.default_rng(7001)
    fams = [(EUCLIDEAN, 2.0), (PNORM, 2.5), (ZNORM, 2.0)]
    for rnd in range(50):
        n0 = int(30 + r.integers(0, 120))
        extra = int(1 + r.integers(0, 40))
        m = int(2 + r.integers(0, n0 // 3))
        allv = r.uniform(-1, 1, n0 + extra) if rnd % 2 == 0 else r.standard_normal(n0 + extra)
        fam, p = fams[rnd % 3]
        cfg = mp.ProfileConfig(m, kind(mp, fam, p))
        st = mp.build_engine_state(mp.make_time_series(allv[:n0]), cfg)
        grown = mp.extend_profile(st, allv[n0:])
        _, Pr, Ir = oracle.scan(allv, m, fam, p)
        rep = check(allv, m, fam, grown.profile.distances, grown.profile.nn_index, Pr, Ir, tol=1e-9,
                    p=p, abs_bound=2e-6 if fam == ZNORM else None)
        assert rep.ok, (rnd, rep.summary())
        assert grown.ts.size() == n0 + extra
        # the original state is unchanged
        assert st.profile.size() == n0 - m + 1


@pytest.mark.parametrize("fam,p", [(EUCLIDEAN, 2.0), (PNORM, 1.0), (ZNORM, 2.0)])
def test_repeated_extension_large(mp, fam, p):
    r = np.random.default_rng(3)
    t = np.cumsum(r.standard_normal(60000))
    if fam == ZNORM:
        t[20000:20600] = t[20000]        # a flat run in the old part
        t[50000:50400] = t[50000]        # and one in the appended part
    m = 128
    cfg = mp.ProfileConfig(m, kind(mp, fam, p))
    cfg.exclusion = 3
    st = mp.build_engine_state(mp.make_time_series(t[:30000]), cfg)
    for a, b in [(30000, 30001), (30001, 30100), (30100, 45000), (45000, 60000)]:
        st = mp.extend_profile(st, t[a:b])
    _, Pr, Ir = oracle.scan(t, m, fam, p, exclusion=3)
    rep = check(t, m, fam, st.profile.distances, st.profile.nn_index, Pr, Ir, tol=1e-9, p=p,
                abs_bound=2e-6 if fam == ZNORM else None)
    assert rep.ok, rep.summary()


def test_extension_edge_cases(mp):
    st = mp.build_engine_state(mp.make_time_series([0, 1, 2, 1, 0, 1, 2]),
                               mp.ProfileConfig(3, mp.DistanceKind.euclidean()))
    same = mp.extend_profile(st, [])
    assert np.array_equal(same.profile.distances, st.profile.distances)
    with pytest.raises(mp.Error) as e:
        mp.extend_profile(st, [1.0, float("nan")])
    assert e.value.code == mp.ErrorCode.NonFinite
    # SPEC.md: state over the zigzag (m=3) + [1] == aamp([0,1,2,1,0,1,2,1], m=3)
    grown = mp.extend_profile(st, [1.0])
    want = mp.aamp(mp.make_time_series([0, 1, 2, 1, 0, 1, 2, 1]), mp.ProfileConfig(3, mp.DistanceKind.euclidean()))
    assert np.allclose(grown.profile.distances, want.distances, atol=1e-12)
    assert np.array_equal(grown.profile.nn_index, want.nn_index)
    # state over [0,0,0,1] (m=2), append [0] -> distances [0,0,1,1]
    st2 = mp.build_engine_state(mp.make_time_series([0, 0, 0, 1]), mp.ProfileConfig(2, mp.DistanceKind.euclidean()))
    g2 = mp.extend_profile(st2, [0.0])
    assert np.allclose(g2.profile.distances, [0, 0, 1, 1], atol=1e-12)


def test_extension_exact_and_fp32_modes(mp):
    """The extension honours the parity build (exact, refresh_interval) and the FP32 mode: parity
    vs the oracle for exact, genuine pairs within the FP32 bound for FP32."""
    r = np.random.default_rng(12)
    t = 100 + np.cumsum(r.standard_normal(9000))
    m = 64
    for fam, p in [(EUCLIDEAN, 2.0), (PNORM, 3.0)]:
        cfg = mp.ProfileConfig(m, kind(mp, fam, p))
        cfg.exact, cfg.refresh_interval = True, 256
        st = mp.extend_profile(mp.build_engine_state(mp.make_time_series(t[:6000]), cfg), t[6000:])
        _, Pr, Ir = oracle.scan(t, m, fam, p)
        rep = check(t, m, fam, st.profile.distances, st.profile.nn_index, Pr, Ir, tol=1e-9, p=p)
        assert rep.ok, rep.summary()
    for fam, p in [(EUCLIDEAN, 2.0), (ZNORM, 2.0)]:
        cfg = mp.ProfileConfig(m, kind(mp, fam, p))
        cfg.precision = mp.Precision.FP32
        st = mp.extend_profile(mp.build_engine_state(mp.make_time_series(t[:6000]), cfg), t[6000:])
        I = st.profile.nn_index
        assert np.all(I >= 0) and np.all(np.abs(I - np.arange(I.size)) >= 1)
        d = oracle.dist_exact(t, np.arange(I.size), I, m, fam)  # P is the distance of the pair
        assert np.all(np.abs(st.profile.distances - d) <= 1e-9 * np.maximum(1, d) + (2e-6 if fam == ZNORM else 0))
        _, P64, _ = oracle.scan(t, m, fam, p)
        excess = (st.profile.distances - P64) / np.maximum(1, P64)
        assert excess.max() <= (5e-3 if fam == ZNORM else 1e-4), excess.max()


def fresh(mp, t, cfg):
    fam = cfg.kind.family
    ts = mp.make_time_series(t)
    if fam == mp.DistanceFamily.Euclidean:
        return mp.aamp(ts, cfg)
    if fam == mp.DistanceFamily.PNorm:
        return mp.aamp_pnorm(ts, cfg)
    return mp.acamp(ts, cfg)


def test_extension_bit_identical_to_fresh(mp):
    """The reference's own contract (test_engine_state.cpp "many random build-then-extend cases
    match from scratch", acceptance criterion 7): exact equality, ties included (short z-normalized
    windows of uniform noise tie exactly)."""
    r = np.random.default_rng(702)
    fams = [(EUCLIDEAN, 2.0), (PNORM, 2.5), (ZNORM, 2.0), (PNORM, 1.0)]
    for rnd in range(60):
        n0 = int(24 + r.integers(0, 80))
        extra = int(1 + r.integers(0, 40))
        m = int(2 + r.integers(0, n0 // 2))
        allv = r.uniform(-1, 1, n0 + extra) if rnd % 2 == 0 else r.standard_normal(n0 + extra)
        fam, p = fams[rnd % 4]
        cfg = mp.ProfileConfig(m, kind(mp, fam, p))
        st = mp.build_engine_state(mp.make_time_series(allv[:n0]), cfg)
        grown = mp.extend_profile(st, allv[n0:])
        want = fresh(mp, allv, cfg)
        assert np.array_equal(grown.profile.nn_index, want.nn_index), rnd
        assert np.array_equal(grown.profile.distances, want.distances), rnd


@pytest.mark.parametrize("fam,p", [(EUCLIDEAN, 2.0), (ZNORM, 2.0)])
def test_large_extension_incremental_and_bit_identical(mp, fam, p):
    """A C4-prefix series grown by 2 000 samples: only the tiles holding new windows run (fewer
    cells than a fresh sweep) and the result equals the fresh profile bit for bit. (The rows per
    tile are planned on the profile length rounded up to 1/8 of its octave: both lengths here
    plan alike, so the extension is incremental.)"""
    from paper_1901_05708_b200 import workloads as W
    t = W.c4()[: (1 << 18) - 1000]
    cfg = mp.ProfileConfig(1024, kind(mp, fam, p))
    st = mp.build_engine_state(mp.make_time_series(t[:-2000]), cfg)
    grown = mp.extend_profile(st, t[-2000:])
    want = fresh(mp, t, cfg)
    assert grown.info.cells < 0.5 * want.info.cells, (grown.info.cells, want.info.cells)
    assert np.array_equal(grown.profile.nn_index, want.nn_index)
    assert np.array_equal(grown.profile.distances, want.distances)


def test_cancelled_build_is_incomplete(mp):
    """tests/test_engine_state.cpp:128-137: a build cancelled by its observer is incomplete, keeps
    the completed diagonals (ascending from the exclusion) and cannot be extended."""
    r = np.random.default_rng(703)
    t = r.uniform(-1, 1, 64)
    cfg = mp.ProfileConfig(6, mp.DistanceKind.euclidean())
    st = mp.build_engine_state(mp.make_time_series(t), cfg, progress=lambda d, n: d < 10)
    assert not st.complete()
    assert list(st.completed_diagonals) == list(range(1, 11))
    assert st.tail().shape == (10,)
    with pytest.raises(mp.Error) as e:
        mp.extend_profile(st, [0.5])
    assert e.value.code == mp.ErrorCode.IncompleteState
    full = mp.build_engine_state(mp.make_time_series(t), cfg)
    assert full.complete() and len(full.completed_diagonals) == 64 - 6
    # tail cursors: the accumulator of each diagonal's last cell (pos = n - m - k)
    tail = full.tail()
    for k in (1, 7, 58):
        pos = 64 - 6 - k
        assert abs(tail[k - 1] - np.sum((t[pos:pos + 6] - t[pos + k:pos + k + 6]) ** 2)) < 1e-12
