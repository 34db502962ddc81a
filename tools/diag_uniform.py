"""Diagnose slow sweeps on noise-like series (experiments only): sweep time, policy, replays."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402

r = np.random.default_rng(9001)
ctx = mp.Context(0)
ctx.set_timing(True)
for kind in ("uniform", "walk"):
    for n in (16384, 65536):
        t = r.uniform(-1, 1, n) if kind == "uniform" else np.cumsum(r.standard_normal(n))
        ts = mp.make_time_series(t)
        for fam in ("aamp", "acamp"):
            for form in (mp.Form.Auto, mp.Form.Alt, mp.Form.Cov):
                ctx.set_form(form)
                cfg = mp.ProfileConfig(256, mp.DistanceKind.euclidean() if fam == "aamp" else mp.DistanceKind.znormalized())
                fn = mp.aamp if fam == "aamp" else mp.acamp
                fn(ts, cfg, ctx=ctx)
                t0 = time.perf_counter()
                res = fn(ts, cfg, ctx=ctx)
                wall = time.perf_counter() - t0
                print(f"{kind:7s} n={n:6d} {fam:5s} form={form.name:4s} policy={res.info.policy:16s} "
                      f"sweep {res.info.sweep_ms:8.3f} ms wall {wall*1e3:8.3f} ms tiles {res.info.tiles}",
                      file=sys.stderr, flush=True)
