"""Ad-hoc sweep timing: python tools/time_cfg.py GEN N M FAMILY [P]   (GEN: c1..c5 | rw)"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os  # noqa: E402
import numpy as np  # noqa: E402
import paper_1901_05708_b200 as mp  # noqa: E402
from paper_1901_05708_b200 import workloads as W  # noqa: E402

gen, n, m, fam = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
p = float(sys.argv[5]) if len(sys.argv) > 5 else 2.0
t = W.random_walk(n, 7) if gen == "rw" else getattr(W, gen)(n=n)
kind = {"e": mp.DistanceKind.euclidean(), "p": mp.DistanceKind.pnorm(p), "z": mp.DistanceKind.znormalized()}[fam]
fn = {"e": mp.aamp, "p": mp.aamp_pnorm, "z": mp.acamp}[fam]
ctx = mp.Context(0)
ctx.set_timing(True)
if os.environ.get("MPROF_RC") is not None:  # 0: tile kernel, 1: constant-row for Wide<>, 2: for all
    ctx.set_row_const(int(os.environ["MPROF_RC"]))
cfg = mp.ProfileConfig(m, kind)
if os.environ.get("MPROF_PRECISION") == "fp32":
    cfg.precision = mp.Precision.FP32
ts = mp.make_time_series(t)
ms = []
for r in range(4):
    res = fn(ts, cfg, ctx=ctx)
    ms.append(res.info.sweep_ms)
b = min(ms[1:])
print(json.dumps({"prec": os.environ.get("MPROF_PRECISION", "fp64"), "gen": gen, "n": n, "m": m, "fam": fam, "sweep_ms": round(b, 3),
                  "cells_per_s": f"{res.info.cells / (b * 1e-3):.3e}", "tiles": res.info.tiles,
                  "R": res.info.rows_per_tile, "policy": res.info.policy,
                  "row_windows": res.info.row_windows, "probe": res.info.probe_replays}))
