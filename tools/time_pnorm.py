"""C3-series p-norm sweep times for several p (experiments only)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402
from paper_1901_05708_b200 import workloads as W  # noqa: E402

ctx = mp.Context(0)
ctx.set_timing(True)
ts = mp.make_time_series(W.c3())
out = {}
for p in [float(x) for x in (sys.argv[1:] or ["1", "3", "2.5", "1.5", "2.7"])]:
    cfg = mp.ProfileConfig(128, mp.DistanceKind.pnorm(p))
    ms = []
    for _ in range(3):
        r = mp.aamp_pnorm(ts, cfg, ctx=ctx)
        ms.append(r.info.sweep_ms)
    out[str(p)] = {"sweep_ms": round(min(ms[1:]), 3), "policy": r.info.policy,
                   "cells_per_s": f"{r.info.cells / (min(ms[1:]) * 1e-3):.3e}"}
print(json.dumps(out))
