"""CPU-side checks of the C ABI (no compute without a GPU): the library loads, exports every
symbol include/mprof_gpu.h declares, applies the reference's validation order and error codes,
and the host-side partition math is right."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import oracle

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "mprof_gpu.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(mprof_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol(mp):
    L = mp.lib()
    syms = declared_symbols()
    assert len(syms) >= 19
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # and the Python binding binds exactly these
    assert set(mp.EXPORTS) == set(syms)


def test_abi_version_and_strings(mp):
    L = mp.lib()
    assert L.mprof_abi_version() == 3
    assert L.mprof_status_string(0) == b"ok"
    assert L.mprof_status_string(9) == b"BadKind"
    assert L.mprof_status_string(100) == b"Cuda"


def test_config_defaults_match_profileconfig(mp):
    c = mp._Config()
    mp.lib().mprof_config_init(C.byref(c), 100, 1, 3.0)
    # core.hpp:82-93 defaults
    assert (c.m, c.family, c.p, c.exclusion, c.order, c.order_seed, c.refresh_interval) == \
        (100, 1, 3.0, 1, 0, 0, 0)
    assert c.flat_threshold == 1e-12 * 100
    assert c.precision == 0 and c.exact == 0
    py = mp.ProfileConfig(100, mp.DistanceKind.pnorm(3.0))
    assert py.flat_threshold == c.flat_threshold and py.exclusion == 1


# (series, m, family, p, exclusion, flat, entry) -> reference error code (ErrorCode + 1)
BAD = [
    ([1.0, 2.0, float("nan"), 3.0], 2, 0, 2.0, 1, None, 0),     # NonFinite
    ([1.0], 1, 0, 2.0, 1, None, 0),                               # TooShort
    ([1.0, float("inf")], 1, 0, 2.0, 1, None, 0),                 # NonFinite before TooShort
    ([0, 1, 2, 3, 4], 0, 0, 2.0, 1, None, 0),                     # BadSubseqLen (m < 1)
    ([0, 1, 2, 3, 4], 5, 0, 2.0, 1, None, 0),                     # BadSubseqLen (m > n-1)
    ([0, 1, 2, 3, 4], 2, 1, 0.5, 1, None, 1),                     # BadP
    ([0, 1, 2, 3, 4], 2, 1, float("nan"), 1, None, 1),            # BadP (nan)
    ([0, 1, 2, 3, 4], 2, 0, 2.0, 0, None, 0),                     # BadExclusion (0)
    ([0, 1, 2, 3, 4], 2, 0, 2.0, 4, None, 0),                     # BadExclusion (> n-m)
    ([0, 1, 2, 3, 4], 2, 2, 2.0, 1, -1e-3, 2),                    # BadThreshold
    ([0, 1, 2, 3, 4], 2, 1, 3.0, 1, None, 0),                     # BadKind (pnorm -> aamp)
    ([0, 1, 2, 3, 4], 2, 2, 2.0, 1, None, 0),                     # BadKind (znorm -> aamp)
    ([0, 1, 2, 3, 4], 2, 0, 2.0, 1, None, 1),                     # BadKind (euclid -> pnorm)
    ([0, 1, 2, 3, 4], 2, 1, 2.0, 1, None, 2),                     # BadKind (pnorm -> acamp)
    ([0, 1, 2, 3, 4], 0, 1, 0.5, 0, None, 2),                     # BadSubseqLen first
    ([0, 1, 2, 3, 4], 2, 1, 0.5, 0, None, 1),                     # BadP before BadExclusion
]
EXPECTED = [1, 2, 1, 5, 5, 6, 6, 7, 7, 8, 9, 9, 9, 9, 5, 6]


def _call_entry(mp, t, m, fam, p, excl, flat, entry):
    t = np.ascontiguousarray(np.asarray(t, dtype=np.float64))
    c = mp._Config()
    mp.lib().mprof_config_init(C.byref(c), m, fam, p)
    c.p = p
    c.exclusion = excl
    if flat is not None:
        c.flat_threshold = flat
    L = max(t.size - m + 1, 1)
    P = np.empty(L)
    I = np.empty(L, dtype=np.int64)
    fn = [mp.lib().mprof_aamp, mp.lib().mprof_aamp_pnorm][entry] if entry < 2 else None
    if entry < 2:
        return fn(None, t.ctypes.data, t.size, C.byref(c), P.ctypes.data, I.ctypes.data, None)
    return mp.lib().mprof_acamp(None, t.ctypes.data, t.size, C.byref(c), 1, P.ctypes.data,
                                I.ctypes.data, None)


@pytest.mark.parametrize("case,expected", list(zip(BAD, EXPECTED)))
def test_error_codes_match_reference(mp, case, expected):
    got = _call_entry(mp, *case)
    assert got == expected, mp.lib().mprof_last_error()
    if oracle.ref_available():
        t, m, fam, p, excl, flat, entry = case
        assert oracle.ref_validate(t, m, fam, p, excl, flat, entry) == expected


def test_python_mirror_raises_reference_errors(mp):
    with pytest.raises(mp.Error) as e:
        mp.make_time_series([1.0, float("nan")])
    assert e.value.code == mp.ErrorCode.NonFinite
    with pytest.raises(mp.Error) as e:
        mp.make_time_series([1.0])
    assert e.value.code == mp.ErrorCode.TooShort
    ts = mp.make_time_series([0, 1, 2, 1, 0, 1, 2])
    with pytest.raises(mp.Error) as e:
        mp.aamp(ts, mp.ProfileConfig(3, mp.DistanceKind.pnorm(3.0)))
    assert e.value.code == mp.ErrorCode.BadKind
    with pytest.raises(mp.Error) as e:
        mp.acamp(ts, mp.ProfileConfig(9, mp.DistanceKind.znormalized()))
    assert e.value.code == mp.ErrorCode.BadSubseqLen
    cfg = mp.ProfileConfig(3, mp.DistanceKind.euclidean())
    cfg.exclusion = 0
    with pytest.raises(mp.Error) as e:
        mp.validate_config(ts, cfg)
    assert e.value.code == mp.ErrorCode.BadExclusion


def test_compute_without_gpu_fails_loudly(mp):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ts = mp.make_time_series(np.arange(20.0))
    with pytest.raises(mp.Error) as e:
        mp.aamp(ts, mp.ProfileConfig(4, mp.DistanceKind.euclidean()))
    assert e.value.code == mp.ErrorCode.Cuda


def test_band_cuts_equal_area(mp):
    n, m = 4194304, 512
    for parts in (1, 2, 4, 8):
        cuts = mp.band_cuts(n, m, 1, parts)
        assert cuts[0] == 1 and cuts[-1] == n - m + 1 and cuts == sorted(cuts)
        cells = [mp.band_cells(n, m, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
        total = mp.band_cells(n, m, 1, n - m + 1)
        assert sum(cells) == total == (n - m) * (n - m + 1) // 2
        # interior cuts sit on whole 1024-diagonal tile blocks (from exclusion + 1), so the
        # balance is within 512 diagonals per cut of perfect
        assert all((c - 2) % 1024 == 0 for c in cuts[1:-1])
        assert max(cells) - min(cells) <= 2 * 512 * n
    # SURVEY.md §8(e) C5 cuts at G=8 (the exact equal-area cut, rounded to a tile block)
    ref = [270858, 561861, 878308, 1228333, 1625629, 2096896, 2711062]
    got = mp.band_cuts(n, m, 1, 8)[1:-1]
    assert all(abs(a - b) <= 512 for a, b in zip(got, ref))


def test_header_documents_reference_interfaces():
    text = HEADER.read_text()
    for needle in ("aamp.hpp:59-60", "aamp.hpp:64-65", "acamp.hpp:100-102", "core.cpp:7-40",
                   "diag_scan.cpp:89-140"):
        assert needle in text
