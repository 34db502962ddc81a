"""Constant-row sweep (csrc/sweep_rc.cu) against the legacy tile kernel: the two paths do the same
arithmetic per cell (same seeds on the same row grid, same slide order), so P and I must be
bit-identical; the run info says which path ran. Series: a C4 prefix (n = 2^18, m = 1024: large
enough for the form probe)."""
import numpy as np
import pytest

import paper_1901_05708_b200 as mp
from paper_1901_05708_b200 import workloads as W

pytestmark = pytest.mark.gpu

N, M = 1 << 18, 1024


@pytest.fixture(scope="module")
def series():
    return W.c4(n=N)


def run(series, family, form, excl, row_const, k_lo=0, k_hi=0):
    ctx = mp.Context(0)
    ctx.set_form(form)
    ctx.set_row_const(row_const)
    kind = mp.DistanceKind.euclidean() if family == "aamp" else mp.DistanceKind.znormalized()
    cfg = mp.ProfileConfig(M, kind)
    cfg.exclusion = excl
    fn = mp.aamp if family == "aamp" else mp.acamp
    r = fn(mp.make_time_series(series), cfg, ctx=ctx)
    ctx.close()
    return r


@pytest.mark.parametrize("family", ["aamp", "acamp"])
@pytest.mark.parametrize("form", [mp.Form.Wide, mp.Form.Cov])
@pytest.mark.parametrize("excl", [1, M])
def test_row_const_bit_identical_to_tile_kernel(series, family, form, excl):
    a = run(series, family, form, excl, True)
    b = run(series, family, form, excl, False)
    assert a.info.row_windows > 0 and b.info.row_windows == 0
    assert a.info.policy == b.info.policy
    assert a.info.rows_per_tile == b.info.rows_per_tile
    np.testing.assert_array_equal(a.nn_index, b.nn_index)
    np.testing.assert_array_equal(a.distances.view(np.uint64), b.distances.view(np.uint64))


def test_row_const_is_the_default_where_it_applies(series):
    ctx = mp.Context(0)
    cfg = mp.ProfileConfig(M, mp.DistanceKind.znormalized())
    r = mp.acamp(mp.make_time_series(series), cfg, ctx=ctx)
    assert r.info.policy in ("Wide<Znorm<0>>", "Znorm<0>") and r.info.row_windows > 0
    # column-scaled form, p-norm and small sweeps keep the tile kernel
    ctx.set_form(mp.Form.Alt)
    r = mp.acamp(mp.make_time_series(series), cfg, ctx=ctx)
    assert r.info.policy == "Znorm<1>" and r.info.row_windows == 0
    ctx.close()


def test_row_const_bands_merge_to_the_single_sweep(series):
    """Diagonal bands (the multi-GPU split) through the constant-row kernel merge to the profile of
    one sweep, bit-identically (band edges cut tiles: the guarded stage variant runs)."""
    cfg = mp.ProfileConfig(M, mp.DistanceKind.euclidean())
    whole = mp.profile_multi(mp.make_time_series(series), cfg, [0], "aamp")
    parts = mp.profile_multi(mp.make_time_series(series), cfg, [0, 0, 0], "aamp")
    assert whole.info.row_windows > 0
    np.testing.assert_array_equal(whole.nn_index, parts.nn_index)
    np.testing.assert_array_equal(whole.distances.view(np.uint64), parts.distances.view(np.uint64))


@pytest.mark.parametrize("family", ["aamp", "acamp"])
def test_row_const_replay_heavy_series_bit_identical(family):
    """A near-periodic series with a low noise floor (the C3 recipe): the covariance-only filters
    pass and replay a large share of their blocks, so the constant-row kernel's deferred replays
    (stash restart, fast-forward of the groups that did not pass, partial last stages) decide most
    entries; they must reproduce the tile kernel's in-place replays bit for bit."""
    t = W.c3(n=1 << 15)
    kind = mp.DistanceKind.euclidean() if family == "aamp" else mp.DistanceKind.znormalized()
    fn = mp.aamp if family == "aamp" else mp.acamp
    out = []
    for rc in (1, 0):
        ctx = mp.Context(0)
        ctx.set_form(mp.Form.Cov)
        ctx.set_row_const(rc)
        cfg = mp.ProfileConfig(256, kind)
        cfg.exclusion = 64
        out.append(fn(mp.make_time_series(t), cfg, ctx=ctx))
        ctx.close()
    a, b = out
    assert a.info.row_windows > 0 and b.info.row_windows == 0
    np.testing.assert_array_equal(a.nn_index, b.nn_index)
    np.testing.assert_array_equal(a.distances.view(np.uint64), b.distances.view(np.uint64))


def test_row_const_fp32_znorm_bit_identical(series):
    """FP32 mode, covariance-only z-norm kernel: the constant-row path (float accumulators, float
    row operands in the parameter space, float carry and stash) against the tile kernel."""
    out = []
    for rc in (1, 0):
        ctx = mp.Context(0)
        ctx.set_row_const(rc)
        cfg = mp.ProfileConfig(M, mp.DistanceKind.znormalized())
        cfg.precision = mp.Precision.FP32
        out.append(mp.acamp(mp.make_time_series(series), cfg, ctx=ctx))
        ctx.close()
    a, b = out
    assert a.info.policy == b.info.policy == "ZnormF32<0>"
    assert a.info.row_windows > 0 and b.info.row_windows == 0
    np.testing.assert_array_equal(a.nn_index, b.nn_index)
    np.testing.assert_array_equal(a.distances.view(np.uint64), b.distances.view(np.uint64))
