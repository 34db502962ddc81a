"""Measured FP32-mode bound: relative excess of P32 (exact distance of the FP32-chosen neighbour)
over P64, per workload / family / exclusion / refresh_interval. Run on the GPU box."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import paper_1901_05708_b200 as mp  # noqa: E402
from paper_1901_05708_b200 import workloads as W  # noqa: E402


def run(t, m, kind, fn, excl, prec, refresh=0):
    cfg = mp.ProfileConfig(m, kind)
    cfg.exclusion = excl
    cfg.precision = prec
    cfg.refresh_interval = refresh
    r = fn(mp.make_time_series(t), cfg)
    return r.distances


cases = [("C1", W.c1(), 100), ("C3", W.c3(), 128), ("C2", W.c2(), 256), ("C4", W.c4(), 1024),
         ("rw500", 500.0 + W.random_walk(20000, 11), 128)]
fams = [("e", mp.DistanceKind.euclidean(), mp.aamp), ("p1", mp.DistanceKind.pnorm(1.0), mp.aamp_pnorm),
        ("p3", mp.DistanceKind.pnorm(3.0), mp.aamp_pnorm), ("z", mp.DistanceKind.znormalized(), mp.acamp)]
out = []
for name, t, m in cases:
    for fname, kind, fn in fams:
        if name == "C4" and fname in ("p1", "p3"):
            continue
        for excl in (1, m):
            for refresh in (0, 4 * m):
                P64 = run(t, m, kind, fn, excl, mp.Precision.FP64)
                P32 = run(t, m, kind, fn, excl, mp.Precision.FP32, refresh)
                e = (P32 - P64) / np.maximum(1.0, np.maximum(np.abs(P32), np.abs(P64)))
                out.append({"case": name, "fam": fname, "excl": excl, "refresh": refresh,
                            "max_excess": float(e.max()), "min_excess": float(e.min()),
                            "frac_changed": float(np.mean(e > 1e-12))})
                print(json.dumps(out[-1]), flush=True)
