"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the matrix-profile hot path.

* ``liboracle.so``: our plain-C restatement of the reference algorithm (mprof_oracle.c), each
  function citing the reference lines it follows. Bit-identical to the reference scan
  (pinned by tests/test_oracle_pin.py).
* ``_ref/libmprof_ref.so``: the reference library itself, compiled from /root/reference by
  oracle/Makefile (only where that tree exists; the prebuilt file travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may import
this package. The product (paper_1901_05708_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libmprof_ref.so"

EUCLIDEAN, PNORM, ZNORM = 0, 1, 2
DEFAULT_FLAT = -7.0e300  # ref_wrapper.cpp sentinel: keep ProfileConfig's default
_P = C.c_void_p
_U = C.c_uint64
_D = C.c_double

_olib = None
_rlib = None


def build() -> None:
    import subprocess
    r = subprocess.run(["make", "-C", str(HERE), "all"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stdout + r.stderr)


def olib() -> C.CDLL:
    global _olib
    if _olib is None:
        if not ORACLE_SO.exists():
            build()
        L = C.CDLL(str(ORACLE_SO))
        L.or_scan.argtypes = [_P, _U, _U, C.c_int, _D, _U, _U, _D, C.c_int, _U, _U, C.c_int, _P, _P, _P]
        L.or_scan.restype = None
        L.or_brute_profile.argtypes = [_P, _U, _U, C.c_int, _D, _U, _D, _P, _P]
        L.or_brute_profile.restype = None
        L.or_dist.argtypes = [_P, _U, _U, _U, C.c_int, _D, _D]
        L.or_dist.restype = _D
        L.or_dist_exact.argtypes = [_P, _U, _U, _U, C.c_int, _D, _D]
        L.or_dist_exact.restype = _D
        L.or_dist_exact_many.argtypes = [_P, _U, C.c_int, _D, _D, _P, _P, _U, _P]
        L.or_dist_exact_many.restype = None
        L.or_exact_rows.argtypes = [_P, _U, _U, C.c_int, _D, _U, _D, _P, _U, C.c_int, _P, _P]
        L.or_exact_rows.restype = None
        L.or_incremental_euclidean_step.argtypes = [_D] * 5
        L.or_incremental_euclidean_step.restype = _D
        L.or_incremental_pnorm_step.argtypes = [_D] * 6
        L.or_incremental_pnorm_step.restype = _D
        L.or_f_to_dz.argtypes = [_D, _U]
        L.or_f_to_dz.restype = _D
        L.or_abs_pow.argtypes = [_D, _D]
        L.or_abs_pow.restype = _D
        _olib = L
    return _olib


class Stats(C.Structure):
    _fields_ = [("sum_left", _D), ("sum_right", _D), ("sumsq_left", _D), ("sumsq_right", _D),
                ("dot", _D), ("offset", _U), ("pos", _U)]


def _stats_fns():
    L = olib()
    L.or_direct_stats.argtypes = [_P, _U, _U, _U]
    L.or_direct_stats.restype = Stats
    L.or_advance_stats.argtypes = [Stats, _D, _D, _D, _D]
    L.or_advance_stats.restype = Stats
    L.or_f_value.argtypes = [C.POINTER(Stats), _D, _D]
    L.or_f_value.restype = _D
    L.or_znorm_sq_from_stats.argtypes = [C.POINTER(Stats), _U, _D]
    L.or_znorm_sq_from_stats.restype = _D
    return L


def _arr(t) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(t, dtype=np.float64))


def default_flat(m: int) -> float:
    return 1e-12 * m


def scan(t, m, family=EUCLIDEAN, p=2.0, exclusion=1, refresh=0, flat=None, use_f=True,
         k_lo=0, k_hi=0, threads=None):
    """run_engine restated: returns (cmp, P, I)."""
    t = _arr(t)
    n = t.shape[0]
    L = n - m + 1
    cmp = np.empty(L)
    P = np.empty(L)
    I = np.empty(L, dtype=np.int64)
    flat = default_flat(m) if flat is None else flat
    threads = threads or min(os.cpu_count() or 1, 64)
    olib().or_scan(t.ctypes.data, n, m, family, p, exclusion, refresh, flat, 1 if use_f else 0,
                   k_lo, k_hi, threads, cmp.ctypes.data, P.ctypes.data, I.ctypes.data)
    return cmp, P, I


def brute(t, m, family=EUCLIDEAN, p=2.0, exclusion=1, flat=None):
    """brute_profile restated (oracle.cpp:95-132)."""
    t = _arr(t)
    n = t.shape[0]
    L = n - m + 1
    P = np.empty(L)
    I = np.empty(L, dtype=np.int64)
    flat = default_flat(m) if flat is None else flat
    olib().or_brute_profile(t.ctypes.data, n, m, family, p, exclusion, flat, P.ctypes.data,
                            I.ctypes.data)
    return P, I


def dist_exact(t, i, j, m, family=EUCLIDEAN, p=2.0, flat=None) -> np.ndarray:
    """Well-conditioned long-double d*(i, j) for arrays of pairs."""
    t = _arr(t)
    i = np.ascontiguousarray(np.asarray(i, dtype=np.int64).reshape(-1))
    j = np.ascontiguousarray(np.asarray(j, dtype=np.int64).reshape(-1))
    out = np.empty(i.shape[0])
    flat = default_flat(m) if flat is None else flat
    olib().or_dist_exact_many(t.ctypes.data, m, family, p, flat, i.ctypes.data, j.ctypes.data,
                              i.shape[0], out.ctypes.data)
    return out


def exact_rows(t, m, rows, family=EUCLIDEAN, p=2.0, exclusion=1, flat=None, threads=None):
    t = _arr(t)
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    best = np.empty(rows.shape[0])
    arg = np.empty(rows.shape[0], dtype=np.int64)
    flat = default_flat(m) if flat is None else flat
    threads = threads or min(os.cpu_count() or 1, 64)
    olib().or_exact_rows(t.ctypes.data, t.shape[0], m, family, p, exclusion, flat, rows.ctypes.data,
                         rows.shape[0], threads, best.ctypes.data, arg.ctypes.data)
    return best, arg


# --- the reference itself (oracle/_ref) ------------------------------------------------------

def ref_available() -> bool:
    return REF_SO.exists()


def rlib() -> C.CDLL:
    global _rlib
    if _rlib is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(str(REF_SO))
        L.ref_profile.argtypes = [_P, _U, _U, C.c_int, _D, _U, _U, _D, C.c_int, C.c_uint, _P, _P]
        L.ref_profile.restype = C.c_int
        L.ref_engine.argtypes = [_P, _U, _U, C.c_int, _D, _U, _U, _D, C.c_int, C.c_uint, _P, _P, _P]
        L.ref_engine.restype = C.c_int
        L.ref_brute.argtypes = [_P, _U, _U, C.c_int, _D, _U, _D, _P, _P]
        L.ref_brute.restype = C.c_int
        L.ref_validate.argtypes = [_P, _U, _U, C.c_int, _D, _U, _D, C.c_int]
        L.ref_validate.restype = C.c_int
        _rlib = L
    return _rlib


def ref_engine(t, m, family=EUCLIDEAN, p=2.0, exclusion=1, refresh=0, flat=None, use_f=True,
               threads=0):
    """mprof::detail::run_engine of the real reference: (cmp, P, I)."""
    t = _arr(t)
    n = t.shape[0]
    L = n - m + 1
    cmp = np.empty(L)
    P = np.empty(L)
    I = np.empty(L, dtype=np.int64)
    st = rlib().ref_engine(t.ctypes.data, n, m, family, p, exclusion, refresh,
                           DEFAULT_FLAT if flat is None else flat, 1 if use_f else 0, threads,
                           cmp.ctypes.data, P.ctypes.data, I.ctypes.data)
    if st != 0:
        raise RuntimeError(f"reference error code {st}")
    return cmp, P, I


def ref_profile(t, m, family=EUCLIDEAN, p=2.0, exclusion=1, refresh=0, flat=None, use_f=True,
                threads=0):
    """mprof::aamp / aamp_pnorm / acamp of the real reference: (P, I)."""
    t = _arr(t)
    n = t.shape[0]
    L = n - m + 1
    P = np.empty(L)
    I = np.empty(L, dtype=np.int64)
    st = rlib().ref_profile(t.ctypes.data, n, m, family, p, exclusion, refresh,
                            DEFAULT_FLAT if flat is None else flat, 1 if use_f else 0, threads,
                            P.ctypes.data, I.ctypes.data)
    if st != 0:
        raise RuntimeError(f"reference error code {st}")
    return P, I


def ref_brute(t, m, family=EUCLIDEAN, p=2.0, exclusion=1, flat=None):
    t = _arr(t)
    n = t.shape[0]
    L = n - m + 1
    P = np.empty(L)
    I = np.empty(L, dtype=np.int64)
    st = rlib().ref_brute(t.ctypes.data, n, m, family, p, exclusion, DEFAULT_FLAT if flat is None else flat,
                          P.ctypes.data, I.ctypes.data)
    if st != 0:
        raise RuntimeError(f"reference error code {st}")
    return P, I


def ref_validate(t, m, family=EUCLIDEAN, p=2.0, exclusion=1, flat=None, entry=0) -> int:
    """0 or mprof::ErrorCode + 1 thrown by the reference entry point `entry` (0 aamp,
    1 aamp_pnorm, 2 acamp)."""
    t = _arr(t)
    return int(rlib().ref_validate(t.ctypes.data, t.shape[0], m, family, p, exclusion,
                                   DEFAULT_FLAT if flat is None else flat, entry))
