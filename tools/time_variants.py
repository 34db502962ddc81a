"""Time C4 AAMP / ACAMP sweeps for each variant library (experiments only; run on the GPU box).

    python tools/time_variants.py build/variants/*.so
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1901_05708_b200 as mp
from paper_1901_05708_b200 import workloads as W
import oracle
from oracle.parity import check
ctx = mp.Context(0); ctx.set_timing(True)
out = {"lib": mp.LIB_PATH.name}
t = W.c4()
for name, kind in [("aamp", mp.DistanceKind.euclidean()), ("acamp", mp.DistanceKind.znormalized())]:
    cfg = mp.ProfileConfig(1024, kind)
    fn = mp.aamp if name == "aamp" else mp.acamp
    ts = mp.make_time_series(t)
    ms = []
    for r in range(4):
        res = fn(ts, cfg, ctx=ctx)
        ms.append(res.info.sweep_ms)
    out[name] = {"sweep_ms": min(ms[1:]), "cells_per_s": res.info.cells / (min(ms[1:]) * 1e-3)}
# quick correctness: small case vs oracle
tt = np.cumsum(np.random.default_rng(3).standard_normal(6000))
for fam, kind in [(0, mp.DistanceKind.euclidean()), (2, mp.DistanceKind.znormalized())]:
    for excl in (1, 200):
        cfg = mp.ProfileConfig(128, kind); cfg.exclusion = excl
        r = (mp.aamp if fam == 0 else mp.acamp)(mp.make_time_series(tt), cfg, ctx=ctx)
        _, Pr, Ir = oracle.scan(tt, 128, fam, exclusion=excl)
        rep = check(tt, 128, fam, r.distances, r.nn_index, Pr, Ir, abs_bound=2e-6 if fam == 2 else None)
        out[f"parity_{fam}_{excl}"] = rep.ok
print(json.dumps(out))
'''

if __name__ == "__main__":
    for lib in sys.argv[1:]:
        env = dict(os.environ, MPROF_GPU_LIB=str(Path(lib).resolve()))
        r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)
