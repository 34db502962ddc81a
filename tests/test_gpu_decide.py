"""The headline kernels where THEY decide the profile.

At exclusion 1 on a random walk nearly every nearest neighbour sits on diagonal 1, which the
direct first-diagonal pass (k_first_diag) evaluates before any tile runs, so full-size tests at
exclusion 1 cannot tell a correct sweep kernel from one that skips far diagonals. Here:

* C4 prefix (n = 2^18, m = 1024: >= 4e9 cells, the size at which the form probe runs, as in the
  bench) at exclusion = m and (n - m) / 4, AAMP and ACAMP, with every filter form forced through
  mprof_ctx_set_form (Cov, Wide, Alt) and the automatic choice; the policy that ran is asserted
  from mprof_run_info (Wide<EuclidCov>, EuclidCov, Euclid / Wide<Znorm<0>>, Znorm<0>, Znorm<1>)
  and at least 90 % of the entries must have their neighbour BEYOND the diagonal block next to
  the exclusion zone (the block the side-stream kernel sweeps), i.e. decided by that policy's
  tiles. Entry-wise parity against the oracle scan (bit-identical restatement of the reference,
  tests/test_oracle_pin.py) with the SURVEY 8(d) rules, plus 1024 rows through the GPU brute force.
* C5 prefix (n = 2^20, m = 512) at exclusion = m, ACAMP (the oracle scan is too slow there):
  4096 rows' full argmin through the GPU brute force plus the long-double distance of every
  reported pair.
* Small series with the forms forced, against the oracle (fast, many shapes).

References: /root/reference/proj/src/detail/diag_scan.hpp:197-199 (diagonal range
[exclusion, n - m]), tests/test_aamp.cpp:276-290 (wider exclusion zones).
"""
import functools

import numpy as np
import pytest

import oracle
from oracle import EUCLIDEAN, ZNORM
from oracle.parity import check, within
from paper_1901_05708_b200 import workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-9
ZN_ABS = 2e-6
K_BLOCK = 1024  # diagonals per tile block (kK); the block after `exclusion` runs the side kernel

FORMS = ("cov", "wide", "alt", "auto")
EXPECT = {
    (EUCLIDEAN, "cov"): {"EuclidCov"}, (EUCLIDEAN, "wide"): {"Wide<EuclidCov>"},
    (EUCLIDEAN, "alt"): {"Euclid"},
    (EUCLIDEAN, "auto"): {"Wide<EuclidCov>", "EuclidCov", "Euclid"},
    (ZNORM, "cov"): {"Znorm<0>"}, (ZNORM, "wide"): {"Wide<Znorm<0>>"}, (ZNORM, "alt"): {"Znorm<1>"},
    (ZNORM, "auto"): {"Wide<Znorm<0>>", "Znorm<0>", "Znorm<1>"},
    (EUCLIDEAN, "dense"): {"Dense<Euclid>"}, (ZNORM, "dense"): {"Dense<Znorm<1>>"},
}


def run(mp, ctx, t, m, fam, excl, form):
    ctx.set_form(getattr(mp.Form, form.capitalize()))
    ts = mp.make_time_series(t)
    kind = mp.DistanceKind.euclidean() if fam == EUCLIDEAN else mp.DistanceKind.znormalized()
    cfg = mp.ProfileConfig(m, kind)
    cfg.exclusion = excl
    r = mp.aamp(ts, cfg, ctx=ctx) if fam == EUCLIDEAN else mp.acamp(ts, cfg, ctx=ctx)
    ctx.set_form(mp.Form.Auto)
    return np.asarray(r.distances), np.asarray(r.nn_index), r.info


def decided_beyond_near_block(I, excl):
    d = np.abs(I - np.arange(I.size))
    return float(np.mean(d >= excl + 1 + K_BLOCK))


@functools.lru_cache(maxsize=None)
def c4_prefix():
    return W.c4()[: 1 << 18]


@functools.lru_cache(maxsize=None)
def c4_oracle(fam, excl):
    _, P, I = oracle.scan(c4_prefix(), 1024, fam, exclusion=excl)
    return P, I


@pytest.fixture(scope="module")
def ctx(mp):
    c = mp.Context(0)
    yield c
    c.close()


@pytest.mark.slow
@pytest.mark.parametrize("fam", [EUCLIDEAN, ZNORM], ids=["aamp", "acamp"])
@pytest.mark.parametrize("excl_kind", ["m", "quarter"])
def test_c4_prefix_kernels_decide(mp, ctx, fam, excl_kind):
    t = c4_prefix()
    m = 1024
    excl = m if excl_kind == "m" else (t.size - m) // 4
    Pr, Ir = c4_oracle(fam, excl)
    frac = decided_beyond_near_block(Ir, excl)
    assert frac >= 0.9, frac  # the reference's own neighbours: far from the exclusion zone
    rng = np.random.default_rng(excl + fam)
    rows = rng.choice(Pr.size, 1024, replace=False)
    kind = mp.DistanceKind.euclidean() if fam == EUCLIDEAN else mp.DistanceKind.znormalized()
    bcfg = mp.ProfileConfig(m, kind)
    bcfg.exclusion = excl
    Pb, Ib = mp.brute_rows(mp.make_time_series(t), bcfg, rows)
    bound = ZN_ABS if fam == ZNORM else 0.0
    for form in FORMS:
        P, I, info = run(mp, ctx, t, m, fam, excl, form)
        assert info.policy in EXPECT[(fam, form)], (form, info.policy)
        if form != "alt":
            assert info.hit_group == (8 if info.policy.startswith("Wide") else 2), info.hit_group
        rep = check(t, m, fam, P, I, Pr, Ir, tol=TOL, abs_bound=ZN_ABS if fam == ZNORM else None)
        assert rep.ok, (form, info.policy, rep.summary())
        assert np.all(np.abs(I - np.arange(I.size))[I >= 0] >= excl)
        assert decided_beyond_near_block(I, excl) >= 0.9
        # full argmin of 1024 rows, independent of the sweep
        assert np.all(within(P[rows], Pb, TOL) | (np.abs(P[rows] - Pb) <= bound)), form
        dg = oracle.dist_exact(t, rows, I[rows], m, fam)
        db = oracle.dist_exact(t, rows, Ib, m, fam)
        assert np.all(within(dg, db, TOL) | (np.abs(dg - db) <= bound)), form


@pytest.mark.slow
def test_c5_prefix_acamp_decides(mp, ctx):
    """C5-shaped series (regime-switching walk), n = 2^20, m = 512, exclusion = m: the z-norm
    kernels decide (neighbours beyond the near block); 4096 rows' full argmin through the GPU
    brute force and every sampled reported pair's long-double distance."""
    t = W.c5()[: 1 << 20]
    m = 512
    excl = m
    rng = np.random.default_rng(55)
    rows = rng.choice(t.size - m + 1, 4096, replace=False)
    bcfg = mp.ProfileConfig(m, mp.DistanceKind.znormalized())
    bcfg.exclusion = excl
    Pb, Ib = mp.brute_rows(mp.make_time_series(t), bcfg, rows)
    for form in ("auto", "cov", "wide"):
        P, I, info = run(mp, ctx, t, m, ZNORM, excl, form)
        assert info.policy in EXPECT[(ZNORM, form)], (form, info.policy)
        assert decided_beyond_near_block(I, excl) >= 0.9
        assert np.all(np.isfinite(P)) and np.all(np.abs(I - np.arange(I.size)) >= excl)
        assert np.all(within(P[rows], Pb, TOL) | (np.abs(P[rows] - Pb) <= ZN_ABS)), form
        dg = oracle.dist_exact(t, rows, I[rows], m, ZNORM)
        db = oracle.dist_exact(t, rows, Ib, m, ZNORM)
        assert np.all(within(dg, db, TOL) | (np.abs(dg - db) <= ZN_ABS)), form
        pick = rng.choice(P.size, 20000, replace=False)
        d = oracle.dist_exact(t, pick, I[pick], m, ZNORM)
        assert np.all(within(P[pick], d, TOL) | (np.abs(P[pick] - d) <= ZN_ABS)), form


@pytest.mark.parametrize("n,m,excl", [(20000, 256, 256), (20000, 256, 4000), (9000, 100, 1),
                                      (12000, 512, 700), (5000, 64, 2500)])
@pytest.mark.parametrize("fam", [EUCLIDEAN, ZNORM], ids=["aamp", "acamp"])
def test_forced_forms_small(mp, ctx, n, m, excl, fam):
    """Every filter form on small series (no probe: the forced form runs), against the oracle."""
    r = np.random.default_rng(n + m + excl)
    t = np.cumsum(r.standard_normal(n)) + 50.0
    _, Pr, Ir = oracle.scan(t, m, fam, exclusion=excl)
    for form in ("cov", "wide", "alt", "dense"):
        P, I, info = run(mp, ctx, t, m, fam, excl, form)
        assert info.policy in EXPECT[(fam, form)], (form, info.policy)
        rep = check(t, m, fam, P, I, Pr, Ir, tol=TOL, abs_bound=ZN_ABS if fam == ZNORM else None)
        assert rep.ok, (form, rep.summary())


@pytest.mark.parametrize("kind", ["uniform", "walk"])
@pytest.mark.parametrize("fam,p", [(EUCLIDEAN, 2.0), (ZNORM, 2.0), (1, 1.0), (1, 3.0)],
                         ids=["aamp", "acamp", "p1", "p3"])
def test_dense_form_noise(mp, ctx, kind, fam, p):
    """Dense<P> (no block filter, every cell compared exactly, shared-memory candidates flushed
    per stage) forced on noise-like series (uniform iid samples, the reference acceptance
    criterion 9 input) and on random walks, and the automatic (filtered) choice, all against the
    oracle."""
    r = np.random.default_rng(9001 + fam)
    t = r.uniform(-1, 1, 8192) if kind == "uniform" else np.cumsum(r.standard_normal(8192))
    m = 256
    kindobj = {EUCLIDEAN: mp.DistanceKind.euclidean(), ZNORM: mp.DistanceKind.znormalized(),
               1: mp.DistanceKind.pnorm(p)}[fam]
    _, Pr, Ir = oracle.scan(t, m, fam, p)
    for form in (mp.Form.Auto, mp.Form.Dense):
        ctx.set_form(form)
        fn = {EUCLIDEAN: mp.aamp, ZNORM: mp.acamp, 1: mp.aamp_pnorm}[fam]
        res = fn(mp.make_time_series(t), mp.ProfileConfig(m, kindobj), ctx=ctx)
        ctx.set_form(mp.Form.Auto)
        assert res.info.policy.startswith("Dense<") == (form == mp.Form.Dense), res.info.policy
        rep = check(t, m, fam, res.distances, res.nn_index, Pr, Ir, tol=TOL, p=p,
                    abs_bound=ZN_ABS if fam == ZNORM else None)
        assert rep.ok, (kind, form, rep.summary())


def test_run_info_reports_policy(mp):
    """Other families report their policy too (p-norm, exact mode, FP32)."""
    r = np.random.default_rng(3)
    t = np.cumsum(r.standard_normal(3000))
    ts = mp.make_time_series(t)
    info = mp.aamp_pnorm(ts, mp.ProfileConfig(64, mp.DistanceKind.pnorm(3.0))).info
    assert info.policy == "Pnorm<3>" and info.hit_group == 1
    cfg = mp.ProfileConfig(64, mp.DistanceKind.euclidean())
    cfg.exact, cfg.refresh_interval = True, 256
    assert mp.aamp(ts, cfg).info.policy == "Euclid<exact>"
    cfg = mp.ProfileConfig(64, mp.DistanceKind.znormalized())
    cfg.precision = mp.Precision.FP32
    assert mp.acamp(ts, cfg).info.policy.startswith("ZnormF32<")
