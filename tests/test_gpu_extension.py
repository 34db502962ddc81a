"""Streaming extension: build_engine_state / extend_profile. The reference's
acceptance criterion 7 (/root/reference/proj/tests/acceptance.cpp:252-286): 50 rounds of
random series, a build over the first n0 samples, an extension by 1..40 samples, compared with a
from-scratch run of the whole series (there with 1e-9 and identical indices; here with the GPU
parity rules — the GPU re-derives the new cells, it does not replay the CPU cursors)."""
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
