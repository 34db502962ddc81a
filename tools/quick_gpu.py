"""First-trip GPU check: FP64 peak, small parity vs numpy brute force, C4/C2-size timing."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1901_05708_b200 as mp

def windows(t, m):
    return np.lib.stride_tricks.sliding_window_view(t, m)

def brute(t, m, kind, excl=1, p=2.0):
    W = windows(t, m); L = W.shape[0]
    P = np.full(L, np.inf); I = np.full(L, -1)
    if kind == 'z':
        mu = W.mean(1, keepdims=True); sd = W.std(1, keepdims=True)
        Z = (W - mu) / sd
    for i in range(L):
        if kind == 'e':
            d = np.sqrt(((W - W[i])**2).sum(1))
        elif kind == 'p':
            d = (np.abs(W - W[i])**p).sum(1) ** (1.0/p)
        else:
            d = np.sqrt(((Z - Z[i])**2).sum(1))
        j = np.arange(L); d[np.abs(j - i) < excl] = np.inf
        k = int(np.argmin(d)); P[i] = d[k]; I[i] = k if np.isfinite(d[k]) else -1
    return P, I

def check(name, got, want, tol):
    P, I = got; Pw, Iw = want
    rel = np.abs(P - Pw) / np.maximum(1, np.maximum(np.abs(P), np.abs(Pw)))
    ok = np.isfinite(rel).all() and rel.max() <= tol
    print(f"{name}: max rel {rel.max():.3e} idx_mismatch {(I != Iw).sum()} {'OK' if ok else 'FAIL'}", flush=True)

g, ms = mp.fp64_peak(); print(f"fp64 peak {g/1e3:.2f} TFLOP/s ({ms:.1f} ms)", flush=True)
rng = np.random.default_rng(1)
for n, m, excl in [(3000, 64, 1), (3000, 64, 64), (1500, 100, 700), (2500, 7, 1)]:
    t = np.cumsum(rng.standard_normal(n))
    ts = mp.make_time_series(t)
    cfg = mp.ProfileConfig(m, mp.DistanceKind.euclidean()); cfg.exclusion = excl
    r = mp.aamp(ts, cfg); check(f"aamp n={n} m={m} excl={excl}", (r.distances, r.nn_index), brute(t, m, 'e', excl), 1e-9)
    cfg = mp.ProfileConfig(m, mp.DistanceKind.znormalized()); cfg.exclusion = excl
    r = mp.acamp(ts, cfg); check(f"acamp n={n} m={m} excl={excl}", (r.distances, r.nn_index), brute(t, m, 'z', excl), 1e-6)
    for p in (1.0, 3.0, 2.5):
        cfg = mp.ProfileConfig(m, mp.DistanceKind.pnorm(p)); cfg.exclusion = excl
        r = mp.aamp_pnorm(ts, cfg); check(f"pnorm p={p} n={n} m={m} excl={excl}", (r.distances, r.nn_index), brute(t, m, 'p', excl, p), 1e-9)

ctx = mp.Context(0); ctx.set_timing(True)
def timed(fn, name, t, cfg, reps=3):
    ts = mp.make_time_series(t)
    for r in range(reps):
        t0 = time.perf_counter(); res = fn(ts, cfg, ctx=ctx); wall = time.perf_counter() - t0
        info = res.info
        print(f"{name}: sweep {info.sweep_ms:.2f} ms wall {wall*1e3:.1f} ms cells {info.cells:.3e} "
              f"-> {info.cells/(info.sweep_ms*1e-3):.3e} cells/s tiles {info.tiles} R {info.rows_per_tile}", flush=True)
    return res
t = np.cumsum(rng.standard_normal(1 << 20))
timed(mp.aamp, "C4 aamp", t, mp.ProfileConfig(1024, mp.DistanceKind.euclidean()))
timed(mp.acamp, "C4 acamp", t, mp.ProfileConfig(1024, mp.DistanceKind.znormalized()))
t2 = np.cumsum(rng.standard_normal(1 << 17))
timed(mp.acamp, "C2 acamp", t2, mp.ProfileConfig(256, mp.DistanceKind.znormalized()))
i = np.arange(1 << 18)
t3 = np.sin(2*np.pi*i/97)+np.sin(2*np.pi*i/503)+np.sin(2*np.pi*i/2011) + 0.1*rng.standard_normal(i.size)
timed(mp.aamp_pnorm, "C3 p1", t3, mp.ProfileConfig(128, mp.DistanceKind.pnorm(1.0)))
timed(mp.aamp_pnorm, "C3 p3", t3, mp.ProfileConfig(128, mp.DistanceKind.pnorm(3.0)))
