"""Wall time of single small host-API calls through the C ABI (the reference acceptance criteria 8
and 9 time such calls), for any build of libmprof_gpu.so (experiments only):

    python tools/call_latency.py [path/to/libmprof_gpu.so ...]

Binds only mprof_config_init / mprof_aamp / mprof_brute_profile (present in every ABI version)."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


class Cfg(C.Structure):
    _fields_ = [("m", C.c_uint64), ("family", C.c_int32), ("order", C.c_int32), ("p", C.c_double),
                ("exclusion", C.c_uint64), ("order_seed", C.c_uint64),
                ("refresh_interval", C.c_uint64), ("flat_threshold", C.c_double),
                ("precision", C.c_int32), ("exact", C.c_int32)]


def bench(libpath):
    L = C.CDLL(str(libpath))
    L.mprof_config_init.argtypes = [C.POINTER(Cfg), C.c_uint64, C.c_int32, C.c_double]
    L.mprof_aamp.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(Cfg), C.c_void_p, C.c_void_p, C.c_void_p]
    L.mprof_acamp.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(Cfg), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
    L.mprof_brute_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(Cfg), C.c_void_p, C.c_void_p]
    info = (C.c_char * 256)()
    r = np.random.default_rng(9001)
    print(f"== {libpath}")
    for kind, gen in (("uniform", lambda n: r.uniform(-1, 1, n)), ("walk", lambda n: np.cumsum(r.standard_normal(n)))):
        for fam in (0, 2):
            for n in (8192, 1 << 14, 1 << 15, 1 << 16):
                t = np.ascontiguousarray(gen(n))
                cfg = Cfg()
                L.mprof_config_init(C.byref(cfg), 256, fam, 2.0)
                P = np.empty(n - 255)
                I = np.empty(n - 255, dtype=np.int64)
                ts = []
                for _ in range(7):
                    t0 = time.perf_counter()
                    if fam == 0:
                        st = L.mprof_aamp(None, t.ctypes.data, n, C.byref(cfg), P.ctypes.data, I.ctypes.data, info)
                    else:
                        st = L.mprof_acamp(None, t.ctypes.data, n, C.byref(cfg), 1, P.ctypes.data, I.ctypes.data, info)
                    ts.append(time.perf_counter() - t0)
                    assert st == 0, st
                print(f"{kind:8s} {'aamp' if fam == 0 else 'acamp'} n={n:6d} m=256: min {min(ts)*1e3:8.3f} ms "
                      f"median {np.median(ts)*1e3:8.3f} ms", flush=True)
    t = np.ascontiguousarray(r.uniform(-1, 1, 8192))
    cfg = Cfg()
    L.mprof_config_init(C.byref(cfg), 256, 0, 2.0)
    P = np.empty(8192 - 255)
    I = np.empty(8192 - 255, dtype=np.int64)
    t0 = time.perf_counter()
    L.mprof_brute_profile(None, t.ctypes.data, 8192, C.byref(cfg), P.ctypes.data, I.ctypes.data)
    print(f"brute n=8192 m=256: {(time.perf_counter() - t0)*1e3:.3f} ms")


for lib in sys.argv[1:] or [ROOT / "paper_1901_05708_b200" / "libmprof_gpu.so"]:
    bench(lib)
