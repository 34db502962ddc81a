"""Pins the CPU oracle (oracle/mprof_oracle.c) before it is trusted as the parity checker:
(a) the reference's own known-answer tests and golden vectors, (b) the reference's outputs
committed under tests/golden (generated from oracle/_ref by tests/golden/make_golden.py), and
(c) when oracle/_ref is present, bit-exact agreement with the reference library on fresh
seeded corpora."""
import math

import numpy as np
import pytest

import oracle
from oracle import EUCLIDEAN, PNORM, ZNORM
from oracle.parity import within

ZIG = np.array([0, 1, 2, 1, 0, 1, 2], dtype=np.float64)  # tests/helpers.hpp:23


def scan(t, m, fam=EUCLIDEAN, p=2.0, **kw):
    _, P, I = oracle.scan(t, m, fam, p, **kw)
    return P, I


# ---- (a) known answers from the reference's tests ------------------------------------------

def test_step_primitives_known_values():
    L = oracle.olib()
    # tests/test_aamp.cpp:45-53
    assert L.or_incremental_euclidean_step(3.0, 0.0, 1.0, 1.0, 0.0) == 3.0
    assert L.or_incremental_euclidean_step(8.0, 0.0, 2.0, 1.0, 1.0) == 4.0
    assert L.or_incremental_euclidean_step(0.0, 5.0, 5.0, 7.0, 7.0) == 0.0
    assert L.or_incremental_euclidean_step(1e-30, 1.0, 2.0, 0.0, 0.0) == 0.0  # clamp
    # tests/test_aamp.cpp:55-61
    assert L.or_incremental_pnorm_step(3.0, 0.0, 1.0, 1.0, 0.0, 3.0) == 3.0
    assert L.or_incremental_pnorm_step(8.0, 1.0, 1.0, 0.0, 2.0, 3.0) == 16.0
    assert L.or_incremental_pnorm_step(4.0, 0.0, 2.0, 1.0, 1.0, 2.0) == \
        L.or_incremental_euclidean_step(4.0, 0.0, 2.0, 1.0, 1.0)


def test_diag_stats_known_values():
    L = oracle._stats_fns()
    t = np.ascontiguousarray(ZIG)
    s1 = L.or_direct_stats(t.ctypes.data, 0, 1, 3)  # tests/test_acamp.cpp:52-60
    assert (s1.sum_left, s1.sum_right, s1.sumsq_left, s1.sumsq_right, s1.dot) == (3, 4, 5, 6, 4)
    assert (s1.offset, s1.pos) == (1, 0)
    s2 = L.or_direct_stats(t.ctypes.data, 0, 2, 3)  # :62-67
    assert (s2.sum_left, s2.sum_right, s2.sumsq_left, s2.sumsq_right, s2.dot) == (3, 3, 5, 5, 1)
    s = L.or_advance_stats(s1, ZIG[0], ZIG[1], ZIG[3], ZIG[4])  # :81-90
    assert (s.sum_left, s.sum_right, s.sumsq_left, s.sumsq_right, s.dot, s.pos) == (4, 3, 6, 5, 4, 1)
    flat = np.full(5, 2.0)
    sf = L.or_direct_stats(flat.ctypes.data, 0, 1, 3)  # :69-73
    assert (sf.sum_left, sf.sumsq_left, sf.dot) == (6, 12, 12)


def test_f_values_and_inverse():
    L = oracle._stats_fns()
    t = np.ascontiguousarray(ZIG)
    import ctypes as C
    f = lambda k: L.or_f_value(C.byref(L.or_direct_stats(t.ctypes.data, 0, k, 3)), 3.0, 0.0)
    # tests/test_acamp.cpp:109-119
    assert within(f(4), -9.0, 1e-12) and within(f(2), 9.0, 1e-12) and within(f(1), 0.0, 1e-12)
    z = lambda k: L.or_znorm_sq_from_stats(C.byref(L.or_direct_stats(t.ctypes.data, 0, k, 3)), 3, 3e-12)
    # :102-107
    assert z(4) == 0.0 and within(z(2), 12.0, 1e-12) and within(z(1), 6.0, 1e-12)
    O = oracle.olib()
    # :127-131
    assert within(O.or_f_to_dz(-9.0, 3), 0.0, 1e-12)
    assert within(O.or_f_to_dz(9.0, 3), math.sqrt(12.0), 1e-12)
    assert within(O.or_f_to_dz(0.0, 3), math.sqrt(6.0), 1e-12)


def test_zigzag_profiles():
    # Euclidean: tests/test_aamp.cpp:63-72
    P, I = scan(ZIG, 3)
    assert np.all(within(P, [0, math.sqrt(3), math.sqrt(3), math.sqrt(3), 0], 1e-12))
    assert list(I) == [4, 0, 1, 0, 0]
    # p = 3: tests/acceptance.cpp:193-201
    P, _ = scan(ZIG, 3, PNORM, 3.0)
    c3 = 3 ** (1 / 3)
    assert np.all(within(P, [0, c3, c3, c3, 0], 1e-9))
    # z-norm both spaces: tests/test_acamp.cpp:181-191
    for use_f in (True, False):
        _, P, I = oracle.scan(ZIG, 3, ZNORM, use_f=use_f)
        assert np.all(within(P, [0, math.sqrt(6), math.sqrt(6), math.sqrt(6), 0], 1e-12))
        assert I[0] == 4 and I[4] == 0


def test_ties_resolve_to_smallest_index():
    # tests/test_aamp.cpp:74-83
    P, I = scan([0, 0, 0, 1], 2)
    assert P[0] == 0.0 and P[1] == 0.0 and within(P[2], 1.0, 1e-15)
    assert list(I) == [1, 0, 0]


def test_flat_convention():
    # tests/test_acamp.cpp:205-220, acceptance.cpp:346-360
    t = [5, 5, 5, 1, 2]
    Pb, _ = oracle.brute(t, 2, ZNORM)
    for use_f in (True, False):
        _, P, I = oracle.scan(t, 2, ZNORM, use_f=use_f)
        assert np.all(within(P, [0, 0, 2, 2], 1e-12)) and np.all(within(P, Pb, 1e-12))
        assert np.all(np.isfinite(P))
        assert I[1] == 0


def test_no_admissible_pair_and_wide_exclusion():
    # tests/test_aamp.cpp:213-228: exclusion 16, n=24, m=4 -> entries 5..15 unresolved
    r = np.random.default_rng(511)
    t = r.uniform(-1, 1, 24)
    P, I = scan(t, 4, exclusion=16)
    Pb, Ib = oracle.brute(t, 4, exclusion=16)
    assert np.all(np.isinf(P) == np.isinf(Pb)) and np.all((I < 0) == (Ib < 0))
    assert np.isinf(P[10]) and I[10] == -1
    fin = np.isfinite(P)
    assert np.all(within(P[fin], Pb[fin], 1e-9))
    # tests/test_aamp.cpp:276-290
    t = r.uniform(-1, 1, 96)
    P, I = scan(t, 8, exclusion=4)
    Pb, _ = oracle.brute(t, 8, exclusion=4)
    assert np.all(within(P, Pb, 1e-9))
    assert np.all(np.abs(I - np.arange(I.size)) >= 4)


def test_refresh_on_offset_series():
    # tests/test_aamp.cpp:174-187
    r = np.random.default_rng(505)
    t = r.uniform(-1, 1, 600) + 1e8
    P, _ = scan(t, 16, refresh=32)
    Pb, _ = oracle.brute(t, 16)
    assert np.all(within(P, Pb, 1e-9))


@pytest.mark.parametrize("fam,p,tol", [(EUCLIDEAN, 2.0, 1e-8), (PNORM, 1.0, 1e-7), (PNORM, 3.0, 1e-7),
                                       (PNORM, 4.5, 1e-7), (ZNORM, 2.0, 1e-6)])
def test_scan_agrees_with_brute(fam, p, tol):
    # acceptance.cpp:79-144 tolerances
    r = np.random.default_rng(7 + int(10 * p) + fam)
    for c in range(12):
        n = int(16 + r.integers(0, 200))
        m = int(2 + r.integers(0, n // 2 - 1))
        t = r.uniform(-1, 1, n) if c % 2 == 0 else r.standard_normal(n)
        P, I = scan(t, m, fam, p)
        Pb, _ = oracle.brute(t, m, fam, p)
        assert np.all(within(P, Pb, tol)), (c, n, m)
        d = np.array([oracle.olib().or_dist(np.ascontiguousarray(t).ctypes.data, i, int(I[i]), m, fam, p, 1e-12 * m)
                      for i in range(P.size)])
        assert np.all(within(d, Pb, tol))


def test_threads_do_not_change_result():
    r = np.random.default_rng(509)
    t = r.standard_normal(240)
    for fam, p in [(EUCLIDEAN, 2.0), (PNORM, 3.0), (ZNORM, 2.0)]:
        c1, P1, I1 = oracle.scan(t, 10, fam, p, threads=1)
        for w in (2, 5):
            c2, P2, I2 = oracle.scan(t, 10, fam, p, threads=w)
            assert np.array_equal(c1, c2) and np.array_equal(P1, P2) and np.array_equal(I1, I2)


def test_bands_merge_to_full_scan():
    """Partial scans of disjoint diagonal bands merge (lexicographic min) to the full scan."""
    r = np.random.default_rng(3)
    t = np.cumsum(r.standard_normal(700))
    m = 20
    cfull, _, Ifull = oracle.scan(t, m)
    L = t.size - m + 1
    cuts = [1, 90, 300, L]
    cmp = np.full(L, np.inf)
    idx = np.full(L, -1)
    for a, b in zip(cuts[:-1], cuts[1:]):
        c, _, I = oracle.scan(t, m, k_lo=a, k_hi=b)
        better = (c < cmp) | ((c == cmp) & (I < idx) & (I >= 0))
        cmp = np.where(better, c, cmp)
        idx = np.where(better, I, idx)
    assert np.array_equal(cmp, cfull) and np.array_equal(idx, Ifull)


# ---- (b) committed reference outputs ----------------------------------------------------------

def test_fixtures_match_reference_bit_exact(golden):
    g = golden["fixtures"]
    for name, fam, p in [("euclidean", EUCLIDEAN, 2.0), ("pnorm", PNORM, 3.0), ("znorm", ZNORM, 2.0)]:
        t = g[f"{name}_t"]
        assert t.size == 1000
        P, I = scan(t, 50, fam, p)
        assert np.array_equal(P, g[f"{name}_P"]) and np.array_equal(I, g[f"{name}_I"]), name
        if fam == ZNORM:
            _, P, I = oracle.scan(t, 50, fam, use_f=False)
            assert np.array_equal(P, g[f"{name}_Psq"]) and np.array_equal(I, g[f"{name}_Isq"])
        Pb, Ib = oracle.brute(t, 50, fam, p)
        assert np.array_equal(Pb, g[f"{name}_Pbrute"]) and np.array_equal(Ib, g[f"{name}_Ibrute"])


def test_corpus_matches_reference_bit_exact(golden):
    g = golden["corpus"]
    for c in range(int(g["count"])):
        t, m = g[f"t{c}"], int(g[f"m{c}"])
        P, I = scan(t, m)
        assert np.array_equal(P, g[f"e_P{c}"]) and np.array_equal(I, g[f"e_I{c}"]), c
        for p in (1.0, 2.0, 3.0, 4.5):
            P, I = scan(t, m, PNORM, p)
            assert np.array_equal(P, g[f"p{p}_P{c}"]) and np.array_equal(I, g[f"p{p}_I{c}"]), (c, p)
        for tag, use_f in (("zf", True), ("zs", False)):
            _, P, I = oracle.scan(t, m, ZNORM, use_f=use_f)
            assert np.array_equal(P, g[f"{tag}_P{c}"]) and np.array_equal(I, g[f"{tag}_I{c}"]), (c, tag)


def test_refresh_runs_match_reference_bit_exact(golden):
    g = golden["exact"]
    for name in ("walk", "walk_excl", "walk_r1", "walk_r7"):
        t = g[f"{name}_t"]
        m, R, excl = (int(x) for x in g[f"{name}_meta"])
        for tag, fam, p in [("e", EUCLIDEAN, 2.0), ("p1", PNORM, 1.0), ("p3", PNORM, 3.0), ("p4", PNORM, 4.0)]:
            cmp, P, I = oracle.scan(t, m, fam, p, exclusion=excl, refresh=R)
            assert np.array_equal(cmp, g[f"{name}_{tag}_cmp"]), (name, tag)
            assert np.array_equal(I, g[f"{name}_{tag}_I"]), (name, tag)


# ---- (c) the reference library itself ---------------------------------------------------------

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("fam,p", [(EUCLIDEAN, 2.0), (PNORM, 1.0), (PNORM, 2.0), (PNORM, 3.0), (PNORM, 4.0),
                                   (PNORM, 2.5), (ZNORM, 2.0)])
def test_scan_bit_exact_against_reference(fam, p):
    r = np.random.default_rng(100 + int(p * 10) + fam)
    for c in range(8):
        n = int(40 + r.integers(0, 900))
        m = int(2 + r.integers(0, min(80, n // 3)))
        kind = c % 4
        t = (np.cumsum(r.standard_normal(n)) + (1000.0 if kind == 1 else 0.0) if kind < 2
             else r.uniform(-1, 1, n))
        if kind == 3 and fam == ZNORM:
            t[n // 4:n // 4 + 3 * m] = 7.0  # flat run
        excl = int([1, 1, m, max(1, (n - m) // 4)][kind])
        refresh = int([0, 64, 0, 17][kind])
        for use_f in ((True, False) if fam == ZNORM else (True,)):
            c1, P1, I1 = oracle.scan(t, m, fam, p, exclusion=excl, refresh=refresh, use_f=use_f, threads=3)
            c2, P2, I2 = oracle.ref_engine(t, m, fam, p, exclusion=excl, refresh=refresh, use_f=use_f, threads=2)
            assert np.array_equal(c1, c2), (c, n, m, excl, refresh)
            assert np.array_equal(P1, P2) and np.array_equal(I1, I2), (c, n, m, excl, refresh)


@needs_ref
def test_brute_bit_exact_against_reference():
    r = np.random.default_rng(77)
    for fam, p in [(EUCLIDEAN, 2.0), (PNORM, 3.0), (ZNORM, 2.0)]:
        t = r.standard_normal(150)
        P1, I1 = oracle.brute(t, 9, fam, p, exclusion=2)
        P2, I2 = oracle.ref_brute(t, 9, fam, p, exclusion=2)
        assert np.array_equal(P1, P2) and np.array_equal(I1, I2)


def test_exact_distance_is_well_conditioned():
    """d* agrees with the direct double evaluation and is 0 on exact affine copies."""
    r = np.random.default_rng(5)
    t = np.cumsum(r.standard_normal(400))
    burst = np.sin(np.arange(32) / 3.0)
    t[50:82] = 400 + burst
    t[250:282] = 400 + 2.5 * burst - 1
    d = oracle.dist_exact(t, [50], [250], 32, ZNORM)
    assert d[0] < 1e-7
    i = r.integers(0, 300, 50)
    j = r.integers(0, 300, 50)
    de = oracle.dist_exact(t, i, j, 32, EUCLIDEAN)
    dd = np.array([oracle.olib().or_dist(np.ascontiguousarray(t).ctypes.data, a, b, 32, 0, 2.0, 0.0)
                   for a, b in zip(i, j)])
    assert np.all(within(de, dd, 1e-12))
