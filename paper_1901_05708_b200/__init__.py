"""B200-native exact matrix profiles (AAMP, p-norm AAMP, ACAMP) — Python mirror of the
reference's ``mprof`` C++ API over the C ABI in ``include/mprof_gpu.h``.

Names, argument order, defaults and error codes follow the reference
(/root/reference/proj/include/mprof/{core,aamp,acamp}.hpp):

    ts  = make_time_series(samples)                       # NonFinite / TooShort
    cfg = ProfileConfig(m, DistanceKind.euclidean())      # exclusion=1, refresh_interval=0, ...
    mp  = aamp(ts, cfg)                                   # MatrixProfile(distances, nn_index)
    mp  = aamp_pnorm(ts, ProfileConfig(m, DistanceKind.pnorm(3.0)))
    mp  = acamp(ts, ProfileConfig(m, DistanceKind.znormalized()), AcampVariant.FScore)

All compute runs in ``libmprof_gpu.so`` on the GPU. There is no CPU fallback: importing works
without a GPU, every compute call raises ``Error(ErrorCode.Cuda)`` if no device is usable, and a
missing library raises ``ImportError`` at first use.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional, Sequence

import numpy as np

__all__ = [
    "ErrorCode", "Error", "DistanceFamily", "DistanceKind", "DiagonalOrder", "AcampVariant",
    "Precision", "Form", "ProfileConfig", "TimeSeries", "make_time_series", "validate_config",
    "profile_length", "default_flat_threshold", "MatrixProfile", "RunInfo", "aamp",
    "aamp_pnorm", "acamp", "sweep_device", "finalize_device", "merge_device", "band_cuts",
    "band_cells", "fp64_peak", "lib", "LIB_PATH", "Context", "EngineState",
    "build_engine_state", "extend_profile", "brute_profile", "ipc_alloc", "ipc_free",
    "ipc_open", "ipc_close", "merge_finalize_peers", "Plan",
]

LIB_PATH = Path(__file__).resolve().parent / "libmprof_gpu.so"
# experiments only: load a tile-parameter variant built by tools/build_variants.py
if __import__("os").environ.get("MPROF_GPU_LIB"):
    LIB_PATH = Path(__import__("os").environ["MPROF_GPU_LIB"])


class ErrorCode(enum.IntEnum):
    """mprof::ErrorCode (core.hpp:16-30) + device-side codes; value = C-ABI status."""
    NonFinite = 1
    TooShort = 2
    EmptyInput = 3
    ParseError = 4
    BadSubseqLen = 5
    BadP = 6
    BadExclusion = 7
    BadThreshold = 8
    BadKind = 9
    OutOfRange = 10
    Degenerate = 11
    IncompleteState = 12
    Io = 13
    Cuda = 100
    OutOfMemory = 101
    BadArgument = 102
    TooLarge = 103


class Error(RuntimeError):
    """mprof::Error (core.hpp:32-44)."""

    def __init__(self, code: ErrorCode, message: str, line: int = 0):
        super().__init__(message)
        self.code = code
        self.line = line


class DistanceFamily(enum.IntEnum):
    Euclidean = 0
    PNorm = 1
    ZNormalized = 2


@dataclass(frozen=True)
class DistanceKind:
    """mprof::DistanceKind (core.hpp:66-73)."""
    family: DistanceFamily = DistanceFamily.Euclidean
    p: float = 2.0

    @staticmethod
    def euclidean() -> "DistanceKind":
        return DistanceKind(DistanceFamily.Euclidean, 2.0)

    @staticmethod
    def pnorm(p: float) -> "DistanceKind":
        return DistanceKind(DistanceFamily.PNorm, float(p))

    @staticmethod
    def znormalized() -> "DistanceKind":
        return DistanceKind(DistanceFamily.ZNormalized, 2.0)


class DiagonalOrder(enum.IntEnum):
    Ascending = 0
    RandomPermutation = 1


class AcampVariant(enum.IntEnum):
    """mprof::AcampVariant (acamp.hpp:95)."""
    SquaredDistance = 0
    FScore = 1


class Precision(enum.IntEnum):
    FP64 = 0
    FP32 = 1


class Form(enum.IntEnum):
    """Filter form override (MPROF_FORM_*): which kernel decides a fast-mode FP64 sweep."""
    Auto = 0
    Cov = 1     # EuclidCov / Znorm<0>
    Wide = 2    # Wide<EuclidCov> / Wide<Znorm<0>>
    Alt = 3     # Euclid (delta, sigma) / Znorm<1> (column-scaled)
    Dense = 4   # no block filter (noise-like series; also p-norm p = 1, 2, 3)


def default_flat_threshold(m: int) -> float:
    """core.hpp:78-80."""
    return 1e-12 * float(m)


class ProfileConfig:
    """mprof::ProfileConfig (core.hpp:82-93) + GPU-only ``precision`` and ``exact``."""

    def __init__(self, m: int, kind: DistanceKind):
        self.m = int(m)
        self.kind = kind
        self.exclusion = 1
        self.order = DiagonalOrder.Ascending
        self.order_seed = 0
        self.refresh_interval = 0
        self.flat_threshold = default_flat_threshold(self.m)
        self.precision = Precision.FP64
        self.exact = False

    def copy(self) -> "ProfileConfig":
        c = ProfileConfig(self.m, self.kind)
        c.__dict__.update(self.__dict__)
        return c

    def __repr__(self) -> str:
        return f"ProfileConfig({self.__dict__})"


class TimeSeries:
    """Immutable validated series (core.hpp:47-59); build with make_time_series."""
    __slots__ = ("_v",)

    def __init__(self, values: np.ndarray, _token=None):
        if _token is not _TOKEN:
            raise TypeError("use make_time_series()")
        self._v = values

    def values(self) -> np.ndarray:
        return self._v

    def size(self) -> int:
        return int(self._v.shape[0])

    def __len__(self) -> int:
        return self.size()

    def __getitem__(self, i):
        return self._v[i]


_TOKEN = object()


def make_time_series(samples: Sequence[float]) -> TimeSeries:
    """core.cpp:7-19: NonFinite (first offending sample) is checked before TooShort."""
    v = np.ascontiguousarray(np.asarray(samples, dtype=np.float64).reshape(-1))
    bad = np.flatnonzero(~np.isfinite(v))
    if bad.size:
        raise Error(ErrorCode.NonFinite, f"sample {int(bad[0])} is not finite")
    if v.shape[0] < 2:
        raise Error(ErrorCode.TooShort, f"time series needs at least 2 samples, got {v.shape[0]}")
    v = v.copy()
    v.setflags(write=False)
    return TimeSeries(v, _TOKEN)


def profile_length(n: int, m: int) -> int:
    return n - m + 1


@dataclass
class MatrixProfile:
    """mprof::MatrixProfile (core.hpp:101-108)."""
    distances: np.ndarray
    nn_index: np.ndarray
    m: int = 0
    kind: DistanceKind = field(default_factory=DistanceKind)
    info: Optional["RunInfo"] = None

    def size(self) -> int:
        return int(self.distances.shape[0])

    def __len__(self) -> int:
        return self.size()


# --------------------------------------------------------------------------------------------
# ctypes binding

class _Config(C.Structure):
    _fields_ = [("m", C.c_uint64), ("family", C.c_int32), ("order", C.c_int32), ("p", C.c_double),
                ("exclusion", C.c_uint64), ("order_seed", C.c_uint64),
                ("refresh_interval", C.c_uint64), ("flat_threshold", C.c_double),
                ("precision", C.c_int32), ("exact", C.c_int32)]


class RunInfo(C.Structure):
    _fields_ = [("cells", C.c_uint64), ("diagonals", C.c_uint64), ("tiles", C.c_uint64),
                ("rows_per_tile", C.c_uint64), ("kernel_launches", C.c_uint32),
                ("sweep_ms", C.c_float), ("fp64_ops_per_cell", C.c_float),
                ("fp32_ops_per_cell", C.c_float), ("_policy", C.c_char * 32),
                ("hit_group", C.c_int32), ("probe_replays", C.c_uint32),
                ("probe_cells", C.c_uint64), ("row_windows", C.c_uint32),
                ("reserved", C.c_uint32)]

    @property
    def policy(self) -> str:
        """The sweep kernel's policy, e.g. "Wide<EuclidCov>", "Znorm<0>", "Pnorm<3>"."""
        return self._policy.decode()

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("_")}
        d["policy"] = self.policy
        return d


EXPORTS = {
    # name: (restype, argtypes)
    "mprof_abi_version": (C.c_int32, []),
    "mprof_status_string": (C.c_char_p, [C.c_int32]),
    "mprof_last_error": (C.c_char_p, []),
    "mprof_config_init": (None, [C.POINTER(_Config), C.c_uint64, C.c_int32, C.c_double]),
    "mprof_validate": (C.c_int32, [C.c_void_p, C.c_uint64, C.POINTER(_Config)]),
    "mprof_profile_length": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "mprof_ctx_create": (C.c_int32, [C.c_int32, C.POINTER(C.c_void_p)]),
    "mprof_ctx_destroy": (None, [C.c_void_p]),
    "mprof_ctx_set_stream": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "mprof_ctx_set_timing": (C.c_int32, [C.c_void_p, C.c_int32]),
    "mprof_aamp": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(_Config), C.c_void_p,
                               C.c_void_p, C.POINTER(RunInfo)]),
    "mprof_aamp_pnorm": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(_Config),
                                     C.c_void_p, C.c_void_p, C.POINTER(RunInfo)]),
    "mprof_acamp": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(_Config), C.c_int32,
                                C.c_void_p, C.c_void_p, C.POINTER(RunInfo)]),
    "mprof_sweep_device": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(_Config),
                                       C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                       C.POINTER(RunInfo)]),
    "mprof_finalize_device": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                          C.c_void_p, C.POINTER(_Config), C.c_void_p]),
    "mprof_merge_device": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_uint64]),
    "mprof_finalize_range_device": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                                C.c_void_p, C.POINTER(_Config), C.c_void_p,
                                                C.c_uint64, C.c_uint64]),
    "mprof_band_cuts": (C.c_int32, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                    C.POINTER(C.c_uint64)]),
    "mprof_band_cells": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]),
    "mprof_fp64_peak": (C.c_int32, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_float)]),
    "mprof_state_build": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(_Config),
                                      C.POINTER(C.c_void_p), C.POINTER(RunInfo)]),
    "mprof_state_extend": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(RunInfo)]),
    "mprof_state_clone": (C.c_int32, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "mprof_state_series_length": (C.c_uint64, [C.c_void_p]),
    "mprof_state_profile": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mprof_state_series": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "mprof_state_destroy": (None, [C.c_void_p]),
    "mprof_state_completed_diagonals": (C.c_uint64, [C.c_void_p]),
    "mprof_state_tail": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "mprof_ctx_set_progress": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "mprof_ctx_set_form": (C.c_int32, [C.c_void_p, C.c_int32]),
    "mprof_ctx_set_row_const": (C.c_int32, [C.c_void_p, C.c_int32]),
    "mprof_plan_create": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(_Config),
                                      C.c_uint64, C.c_uint64, C.POINTER(C.c_void_p)]),
    "mprof_plan_sweep": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(RunInfo)]),
    "mprof_plan_destroy": (None, [C.c_void_p]),
    "mprof_brute_profile": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(_Config),
                                        C.c_void_p, C.c_void_p]),
    "mprof_brute_rows": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(_Config),
                                     C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "mprof_profile_multi": (C.c_int32, [C.c_void_p, C.c_uint32, C.c_int32, C.c_void_p, C.c_uint64,
                                        C.POINTER(_Config), C.c_void_p, C.c_void_p, C.c_void_p]),
    "mprof_ipc_alloc": (C.c_int32, [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p), C.c_void_p]),
    "mprof_ipc_free": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "mprof_ipc_open": (C.c_int32, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "mprof_ipc_close": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "mprof_merge_finalize_peers": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64,
                                               C.POINTER(_Config), C.POINTER(C.c_void_p),
                                               C.POINTER(C.c_void_p), C.c_uint32,
                                               C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                               C.c_uint32, C.c_uint64, C.c_uint64]),
}
IPC_HANDLE_BYTES = 64
MAX_PEERS = 16
PROGRESS_FN = C.CFUNCTYPE(C.c_int32, C.c_uint64, C.c_uint64, C.c_void_p)

_lib = None


def lib() -> C.CDLL:
    """Loads the in-tree libmprof_gpu.so (raises ImportError if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (the CUDA extension is required; there is no fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _raise(status: int) -> None:
    if status != 0:
        msg = lib().mprof_last_error().decode(errors="replace")
        try:
            code = ErrorCode(status)
        except ValueError:
            code = ErrorCode.Cuda
        raise Error(code, msg)


def _to_c(cfg: ProfileConfig) -> _Config:
    c = _Config()
    c.m = cfg.m
    c.family = int(cfg.kind.family)
    c.order = int(cfg.order)
    c.p = float(cfg.kind.p)
    c.exclusion = int(cfg.exclusion)
    c.order_seed = int(cfg.order_seed)
    c.refresh_interval = int(cfg.refresh_interval)
    c.flat_threshold = float(cfg.flat_threshold)
    c.precision = int(cfg.precision)
    c.exact = 1 if cfg.exact else 0
    return c


def _check_int_fields(cfg: ProfileConfig) -> None:
    # size_t fields: negative values would wrap; the reference's validate_config rejects them
    if cfg.m < 1:
        raise Error(ErrorCode.BadSubseqLen, f"subsequence length {cfg.m} < 1")
    if cfg.exclusion < 1:
        raise Error(ErrorCode.BadExclusion, f"exclusion {cfg.exclusion} < 1")


def validate_config(ts: TimeSeries, cfg: ProfileConfig) -> ProfileConfig:
    """core.cpp:21-40 (same order and codes)."""
    _check_int_fields(cfg)
    c = _to_c(cfg)
    v = ts.values()
    _raise(lib().mprof_validate(v.ctypes.data, v.shape[0], C.byref(c)))
    return cfg


class Context:
    """One device's workspace + stream (mprof_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _raise(lib().mprof_ctx_create(int(device), C.byref(h)))
        self.handle = h

    def set_stream(self, stream_ptr: int) -> None:
        _raise(lib().mprof_ctx_set_stream(self.handle, C.c_void_p(stream_ptr)))

    def set_timing(self, on: bool) -> None:
        _raise(lib().mprof_ctx_set_timing(self.handle, 1 if on else 0))

    def set_form(self, form: "Form") -> None:
        """Filter form of FP64 fast-mode Euclidean / z-norm sweeps (mprof_ctx_set_form)."""
        _raise(lib().mprof_ctx_set_form(self.handle, int(form)))

    def set_row_const(self, on) -> None:
        """Constant-row sweep of the covariance-only forms (mprof_ctx_set_row_const): on by
        default; False / 0 selects the single-launch tile kernel."""
        _raise(lib().mprof_ctx_set_row_const(self.handle, int(on)))

    def close(self) -> None:
        if self.handle:
            lib().mprof_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def _ctx_handle(ctx: Optional[Context]):
    return None if ctx is None else ctx.handle


def _run(fn_name: str, ts: TimeSeries, cfg: ProfileConfig, extra, ctx, progress) -> MatrixProfile:
    _check_int_fields(cfg)
    v = ts.values()
    n = v.shape[0]
    L = max(n - cfg.m + 1, 0)
    P = np.empty(L, dtype=np.float64)
    I = np.empty(L, dtype=np.int64)
    info = RunInfo()
    c = _to_c(cfg)
    args = [_ctx_handle(ctx), v.ctypes.data, n, C.byref(c), *extra, P.ctypes.data, I.ctypes.data,
            C.byref(info)]
    cb = None
    if progress is not None:
        # anytime observer (ProgressFn): band-granular chunks, False cancels
        cb = PROGRESS_FN(lambda done, total, _u: 1 if progress(int(done), int(total)) else 0)
        _raise(lib().mprof_ctx_set_progress(_ctx_handle(ctx), C.cast(cb, C.c_void_p), None))
    try:
        _raise(getattr(lib(), fn_name)(*args))
    finally:
        if cb is not None:
            lib().mprof_ctx_set_progress(_ctx_handle(ctx), None, None)
    return MatrixProfile(P, I, cfg.m, cfg.kind, info)


def brute_profile(ts: TimeSeries, cfg: ProfileConfig, ctx: Optional[Context] = None) -> MatrixProfile:
    """mprof::brute_profile (/root/reference/proj/include/mprof/oracle.hpp:20) on the GPU."""
    _check_int_fields(cfg)
    v = ts.values()
    L = max(v.shape[0] - cfg.m + 1, 0)
    P = np.empty(L)
    I = np.empty(L, dtype=np.int64)
    c = _to_c(cfg)
    _raise(lib().mprof_brute_profile(_ctx_handle(ctx), v.ctypes.data, v.shape[0], C.byref(c),
                                     P.ctypes.data, I.ctypes.data))
    return MatrixProfile(P, I, cfg.m, cfg.kind)


ENGINES = {"aamp": 0, "aamp_pnorm": 1, "acamp": 2}


def profile_multi(ts: TimeSeries, cfg: ProfileConfig, devices, engine: str = "aamp") -> MatrixProfile:
    """One process, several GPUs (mprof_profile_multi): equal-area diagonal bands, one per entry
    of `devices` (a device may repeat), merged on devices[0]. engine: aamp | aamp_pnorm | acamp."""
    _check_int_fields(cfg)
    v = ts.values()
    n = v.shape[0]
    L = max(n - cfg.m + 1, 0)
    P = np.empty(L, dtype=np.float64)
    I = np.empty(L, dtype=np.int64)
    info = RunInfo()
    d = np.ascontiguousarray(devices, dtype=np.int32)
    c = _to_c(cfg)
    _raise(lib().mprof_profile_multi(d.ctypes.data, d.size, ENGINES[engine], v.ctypes.data, n,
                                     C.byref(c), P.ctypes.data, I.ctypes.data, C.byref(info)))
    return MatrixProfile(P, I, cfg.m, cfg.kind, info)


def brute_rows(ts: TimeSeries, cfg: ProfileConfig, rows, ctx: Optional[Context] = None):
    """Brute-force (distance, index) of the nearest neighbour of each of `rows` (GPU, the
    arithmetic of brute_profile). Returns (P, I) arrays of len(rows)."""
    _check_int_fields(cfg)
    v = ts.values()
    r = np.ascontiguousarray(rows, dtype=np.int64)
    P = np.empty(r.size)
    I = np.empty(r.size, dtype=np.int64)
    c = _to_c(cfg)
    _raise(lib().mprof_brute_rows(_ctx_handle(ctx), v.ctypes.data, v.shape[0], C.byref(c),
                                  r.ctypes.data, r.size, P.ctypes.data, I.ctypes.data))
    return P, I


def aamp(ts: TimeSeries, cfg: ProfileConfig, progress: Optional[Callable] = None, threads: int = 0,
         ctx: Optional[Context] = None) -> MatrixProfile:
    """mprof::aamp (aamp.hpp:59-60). `threads` is accepted for signature parity."""
    return _run("mprof_aamp", ts, cfg, [], ctx, progress)


def aamp_pnorm(ts: TimeSeries, cfg: ProfileConfig, progress: Optional[Callable] = None,
               threads: int = 0, ctx: Optional[Context] = None) -> MatrixProfile:
    """mprof::aamp_pnorm (aamp.hpp:64-65)."""
    return _run("mprof_aamp_pnorm", ts, cfg, [], ctx, progress)


def acamp(ts: TimeSeries, cfg: ProfileConfig, variant: AcampVariant = AcampVariant.FScore,
          progress: Optional[Callable] = None, threads: int = 0,
          ctx: Optional[Context] = None) -> MatrixProfile:
    """mprof::acamp (acamp.hpp:100-102)."""
    return _run("mprof_acamp", ts, cfg, [int(variant)], ctx, progress)


# --------------------------------------------------------------------------------------------
# device-resident pipeline (pointers are raw device addresses, e.g. torch tensor.data_ptr())

def sweep_device(d_t: int, n: int, cfg: ProfileConfig, k_lo: int, k_hi: int, d_cmp: int, d_idx: int,
                 ctx: Optional[Context] = None) -> RunInfo:
    info = RunInfo()
    c = _to_c(cfg)
    _raise(lib().mprof_sweep_device(_ctx_handle(ctx), C.c_void_p(d_t), n, C.byref(c), k_lo, k_hi,
                                    C.c_void_p(d_cmp), C.c_void_p(d_idx), C.byref(info)))
    return info


class Plan:
    """A planned band sweep of one device-resident series (mprof_plan_create): the per-series
    decisions are taken once; sweep() only enqueues kernels (no host synchronisation)."""

    def __init__(self, d_t: int, n: int, cfg: ProfileConfig, k_lo: int = 0, k_hi: int = 0,
                 ctx: Optional[Context] = None):
        self.cfg = cfg
        self._c = _to_c(cfg)
        self._ctx = ctx  # the plan borrows the context: keep it alive as long as the plan
        h = C.c_void_p()
        _raise(lib().mprof_plan_create(_ctx_handle(ctx), C.c_void_p(d_t), n, C.byref(self._c),
                                       k_lo, k_hi, C.byref(h)))
        self.handle = h

    def sweep(self, d_cmp: int, d_idx: int) -> RunInfo:
        info = RunInfo()
        _raise(lib().mprof_plan_sweep(self.handle, C.c_void_p(d_cmp), C.c_void_p(d_idx), C.byref(info)))
        return info

    def close(self) -> None:
        if self.handle:
            lib().mprof_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def finalize_device(d_t: int, n: int, d_cmp: int, d_idx: int, cfg: ProfileConfig, d_P: int,
                    ctx: Optional[Context] = None) -> None:
    c = _to_c(cfg)
    _raise(lib().mprof_finalize_device(_ctx_handle(ctx), C.c_void_p(d_t), n, C.c_void_p(d_cmp),
                                       C.c_void_p(d_idx), C.byref(c), C.c_void_p(d_P)))


def finalize_range_device(d_t: int, n: int, d_cmp: int, d_idx: int, cfg: ProfileConfig, d_P: int,
                          lo: int, hi: int, ctx: Optional[Context] = None) -> None:
    c = _to_c(cfg)
    _raise(lib().mprof_finalize_range_device(_ctx_handle(ctx), C.c_void_p(d_t), n, C.c_void_p(d_cmp),
                                             C.c_void_p(d_idx), C.byref(c), C.c_void_p(d_P), lo, hi))


def merge_device(d_cmp: int, d_idx: int, d_ocmp: int, d_oidx: int, L: int,
                 ctx: Optional[Context] = None) -> None:
    _raise(lib().mprof_merge_device(_ctx_handle(ctx), C.c_void_p(d_cmp), C.c_void_p(d_idx),
                                    C.c_void_p(d_ocmp), C.c_void_p(d_oidx), L))


def ipc_alloc(nbytes: int, ctx: Optional[Context] = None) -> tuple[int, bytes]:
    """Device buffer (zero-filled) that other processes can map: (pointer, 64-byte handle)."""
    ptr = C.c_void_p()
    h = (C.c_ubyte * IPC_HANDLE_BYTES)()
    _raise(lib().mprof_ipc_alloc(_ctx_handle(ctx), nbytes, C.byref(ptr), h))
    return int(ptr.value), bytes(h)


def ipc_free(ptr: int, ctx: Optional[Context] = None) -> None:
    _raise(lib().mprof_ipc_free(_ctx_handle(ctx), C.c_void_p(ptr)))


def ipc_open(handle: bytes, ctx: Optional[Context] = None) -> int:
    """Maps another process's ipc_alloc buffer (NVLink peer memory) into this process."""
    if len(handle) != IPC_HANDLE_BYTES:
        raise Error(ErrorCode.BadArgument, "IPC handles are 64 bytes")
    h = (C.c_ubyte * IPC_HANDLE_BYTES).from_buffer_copy(handle)
    ptr = C.c_void_p()
    _raise(lib().mprof_ipc_open(_ctx_handle(ctx), h, C.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int, ctx: Optional[Context] = None) -> None:
    _raise(lib().mprof_ipc_close(_ctx_handle(ctx), C.c_void_p(ptr)))


def merge_finalize_peers(d_t: int, n: int, cfg: ProfileConfig, peer_cmp: Sequence[int],
                         peer_idx: Sequence[int], out_P: Sequence[int], out_I: Sequence[int],
                         lo: int, hi: int, ctx: Optional[Context] = None) -> None:
    """Entries [lo, hi) of the merged + finalized profile of the partials (peer_cmp[r],
    peer_idx[r]) stored into every (out_P[r], out_I[r]) (peer pointers; one fused kernel)."""
    c = _to_c(cfg)
    arr = lambda xs: (C.c_void_p * max(1, len(xs)))(*[C.c_void_p(x) for x in xs])  # noqa: E731
    _raise(lib().mprof_merge_finalize_peers(_ctx_handle(ctx), C.c_void_p(d_t), n, C.byref(c),
                                            arr(peer_cmp), arr(peer_idx), len(peer_cmp),
                                            arr(out_P), arr(out_I), len(out_P), lo, hi))


def band_cuts(n: int, m: int, exclusion: int, parts: int) -> list:
    """Equal-area diagonal bands [cuts[g], cuts[g+1]) for `parts` GPUs (host math only)."""
    out = (C.c_uint64 * (parts + 1))()
    _raise(lib().mprof_band_cuts(n, m, exclusion, parts, out))
    return [int(x) for x in out]


def band_cells(n: int, m: int, k_lo: int, k_hi: int) -> int:
    return int(lib().mprof_band_cells(n, m, k_lo, k_hi))


def fp64_peak(ctx: Optional[Context] = None) -> tuple:
    """Measured DFMA-chain FP64 throughput of the current device: (GFLOP/s, ms)."""
    g = C.c_double()
    ms = C.c_float()
    _raise(lib().mprof_fp64_peak(_ctx_handle(ctx), C.byref(g), C.byref(ms)))
    return float(g.value), float(ms.value)


# --------------------------------------------------------------------------------------------
# streaming extension: mprof::EngineState / build_engine_state / extend_profile
# (/root/reference/proj/include/mprof/engine_state.hpp:26-52)

class EngineState:
    """A computed profile plus what is needed to grow it: here the series and the
    comparison-space profile held on the GPU (the reference keeps per-diagonal tail cursors;
    the GPU re-derives the new cells from the series instead)."""

    def __init__(self, handle, cfg: ProfileConfig, info: Optional[RunInfo] = None):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self.cfg = cfg
        self.info = info
        self._cache = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            if self._h:
                lib().mprof_state_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def _load(self):
        if self._cache is None:
            n = int(lib().mprof_state_series_length(self._h))
            L = n - self.cfg.m + 1
            t = np.empty(n)
            P = np.empty(L)
            I = np.empty(L, dtype=np.int64)
            cmp = np.empty(L)
            _raise(lib().mprof_state_series(self._h, t.ctypes.data))
            _raise(lib().mprof_state_profile(self._h, P.ctypes.data, I.ctypes.data, cmp.ctypes.data))
            self._cache = (t, MatrixProfile(P, I, self.cfg.m, self.cfg.kind, self.info), cmp)
        return self._cache

    @property
    def ts(self) -> TimeSeries:
        return make_time_series(self._load()[0])

    @property
    def profile(self) -> MatrixProfile:
        return self._load()[1]

    @property
    def comparison(self) -> np.ndarray:
        return self._load()[2]

    @property
    def completed_diagonals(self) -> np.ndarray:
        """Ascending offsets k of the diagonals the build completed (engine_state.hpp:33)."""
        done = int(lib().mprof_state_completed_diagonals(self._h))
        return np.arange(self.cfg.exclusion, self.cfg.exclusion + done, dtype=np.int64)

    def tail(self) -> np.ndarray:
        """Tail accumulators per completed diagonal (mprof_state_tail): shape (done,) or
        (done, 5) for z-normalized states (the five DiagStats sums)."""
        done = int(lib().mprof_state_completed_diagonals(self._h))
        five = self.cfg.kind.family == DistanceFamily.ZNormalized
        out = np.empty((done, 5) if five else done)
        _raise(lib().mprof_state_tail(self._h, out.ctypes.data))
        return out

    def complete(self) -> bool:
        """True when every diagonal of the build ran (engine_state.hpp:37-39); a build cancelled
        by its progress observer is incomplete and extend_profile refuses it."""
        n = int(lib().mprof_state_series_length(self._h))
        total = n - self.cfg.m - self.cfg.exclusion + 1
        return int(lib().mprof_state_completed_diagonals(self._h)) == total


def build_engine_state(ts: TimeSeries, cfg: ProfileConfig, progress: Optional[Callable] = None,
                       threads: int = 0, ctx: Optional[Context] = None) -> EngineState:
    """engine_state.hpp:44-45 (any distance family)."""
    _check_int_fields(cfg)
    v = ts.values()
    h = C.c_void_p()
    info = RunInfo()
    c = _to_c(cfg)
    cb = None
    if progress is not None:
        # anytime observer: band-granular chunks; False cancels -> an incomplete state
        cb = PROGRESS_FN(lambda done, total, _u: 1 if progress(int(done), int(total)) else 0)
        _raise(lib().mprof_ctx_set_progress(_ctx_handle(ctx), C.cast(cb, C.c_void_p), None))
    try:
        _raise(lib().mprof_state_build(_ctx_handle(ctx), v.ctypes.data, v.shape[0], C.byref(c),
                                       C.byref(h), C.byref(info)))
    finally:
        if cb is not None:
            lib().mprof_ctx_set_progress(_ctx_handle(ctx), None, None)
    return EngineState(h, cfg.copy(), info)


def extend_profile(state: EngineState, new_samples: Sequence[float]) -> EngineState:
    """engine_state.hpp:52: a NEW state for the extended series (the input is unchanged).
    NonFinite for a bad sample; an empty span returns an equal state."""
    s = np.ascontiguousarray(np.asarray(new_samples, dtype=np.float64).reshape(-1))
    if not state.complete():  # engine_state.cpp:56-58: before the sample checks
        done = int(lib().mprof_state_completed_diagonals(state._h))
        raise Error(ErrorCode.IncompleteState,
                    f"cannot extend a partially computed profile ({done} diagonals done)")
    bad = np.flatnonzero(~np.isfinite(s))
    if bad.size:
        raise Error(ErrorCode.NonFinite, f"appended sample {int(bad[0])} is not finite")
    h = C.c_void_p()
    _raise(lib().mprof_state_clone(state._h, C.byref(h)))
    out = EngineState(h, state.cfg.copy())
    info = RunInfo()
    _raise(lib().mprof_state_extend(out._h, s.ctypes.data if s.size else None, s.shape[0],
                                    C.byref(info)))
    out.info = info
    return out
