"""Results do not depend on how the diagonals are split.

The reference is bit-identical for any thread count and diagonal schedule
(/root/reference/proj/tests/test_aamp.cpp:245-274, tests/test_acamp.cpp:293-310). On the GPU the
default (fast) mode seeds every diagonal on one row grid chosen from the series alone (choose_R on
the whole diagonal range), cuts bands and anytime chunks along one global grid of diagonal blocks,
and takes the filter-form decision (and its probe) once per series, so the arithmetic of every cell
is the same whatever the split: one device, 2 / 3 / 8 bands, or band-granular progress chunks all
give bit-identical P and I.
"""
import numpy as np
import pytest

from paper_1901_05708_b200 import workloads as W

pytestmark = pytest.mark.gpu

ENGINES = [("aamp", "euclidean", None), ("aamp_pnorm", "pnorm", 3.0), ("acamp", "znormalized", None)]


def kind(mp, name, p):
    return mp.DistanceKind.pnorm(p) if name == "pnorm" else getattr(mp.DistanceKind, name)()


def series_cases():
    r = np.random.default_rng(77)
    walk = 20 + np.cumsum(r.standard_normal(30000))
    walk[12000:12600] = walk[12000]  # a flat run (z-norm flat rule)
    return [("walk30k", walk, 128, 1), ("walk30k_excl", walk, 128, 700),
            ("c4_prefix", W.c4()[: 1 << 18], 1024, 1)]  # >= 4e9 cells: the form probe runs


@pytest.mark.parametrize("case", series_cases(), ids=lambda c: c[0])
def test_band_split_bit_identical(mp, case):
    _, t, m, excl = case
    ts = mp.make_time_series(t)
    for engine, kname, p in ENGINES:
        if case[0] == "c4_prefix" and engine == "aamp_pnorm":
            continue
        cfg = mp.ProfileConfig(m, kind(mp, kname, p))
        cfg.exclusion = excl
        one = getattr(mp, engine)(ts, cfg)
        for k in (1, 2, 3, 8):
            multi = mp.profile_multi(ts, cfg, [0] * k, engine)
            assert np.array_equal(multi.nn_index, one.nn_index), (engine, k)
            assert np.array_equal(multi.distances, one.distances), (engine, k)


def test_anytime_chunks_bit_identical(mp):
    """Band-granular progress chunks (ascending, unaligned to the block grid) == one launch."""
    r = np.random.default_rng(78)
    t = np.cumsum(r.standard_normal(40000))
    ts = mp.make_time_series(t)
    ticks = []
    for engine, kname, p in ENGINES:
        cfg = mp.ProfileConfig(256, kind(mp, kname, p))
        one = getattr(mp, engine)(ts, cfg)
        ticks.clear()
        chunked = getattr(mp, engine)(ts, cfg, progress=lambda d, n: ticks.append(d) or True)
        assert len(ticks) > 100
        assert np.array_equal(chunked.nn_index, one.nn_index), engine
        assert np.array_equal(chunked.distances, one.distances), engine
