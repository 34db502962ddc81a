"""Sweep-kernel timings of the C4 engines (and optional C2/C3/C5), experiments only."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402
from paper_1901_05708_b200 import workloads as W  # noqa: E402

args = [a for a in sys.argv[1:] if a not in ("norc", "rcall")]
names = args or ["C4aamp", "C4acamp"]
ctx = mp.Context(0)
ctx.set_timing(True)
if "norc" in sys.argv[1:]:
    ctx.set_row_const(False)  # the legacy single-launch tile kernel
if "rcall" in sys.argv[1:]:
    ctx.set_row_const(2)      # the constant-row kernel for every covariance-only form
out = {}
for name in names:
    c = W.CONFIGS[name]
    t = c.gen()
    kind = {"euclidean": mp.DistanceKind.euclidean(), "pnorm": mp.DistanceKind.pnorm(c.p),
            "znorm": mp.DistanceKind.znormalized()}[c.family]
    fn = {"euclidean": mp.aamp, "pnorm": mp.aamp_pnorm, "znorm": mp.acamp}[c.family]
    cfg = mp.ProfileConfig(c.m, kind)
    ts = mp.make_time_series(t)
    ms = []
    for r in range(4):
        res = fn(ts, cfg, ctx=ctx)
        ms.append(res.info.sweep_ms)
    best = min(ms[1:])
    out[name] = {"sweep_ms": round(best, 3), "cells_per_s": f"{res.info.cells / (best * 1e-3):.4e}",
                 "tiles": res.info.tiles, "R": res.info.rows_per_tile,
                 "policy": getattr(res.info, "policy", "?"), "row_windows": res.info.row_windows, "hg": getattr(res.info, "hit_group", 0),
                 "probe": [getattr(res.info, "probe_replays", 0), getattr(res.info, "probe_cells", 0)]}
print(json.dumps(out))
