"""Replay/offer statistics of the sweep filter on the BASELINE workloads (MPROF_STATS=1)."""
import os
import sys
from pathlib import Path

os.environ["MPROF_STATS"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402
from paper_1901_05708_b200 import workloads as W  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2", "C3p1", "C3p3", "C4aamp", "C4acamp"]:
    c = W.CONFIGS[name]
    t = c.gen()
    kind = {"euclidean": mp.DistanceKind.euclidean(), "pnorm": mp.DistanceKind.pnorm(c.p),
            "znorm": mp.DistanceKind.znormalized()}[c.family]
    cfg = mp.ProfileConfig(c.m, kind)
    fn = {"euclidean": mp.aamp, "pnorm": mp.aamp_pnorm, "znorm": mp.acamp}[c.family]
    print(name, file=sys.stderr, flush=True)
    for excl in (1, c.m):
        cfg.exclusion = excl
        r = fn(mp.make_time_series(t), cfg)
        blocks = r.info.cells / 64
        print(f"  excl={excl}: cells {r.info.cells:.3e} (~{blocks:.3e} thread-blocks of 64 cells)",
              file=sys.stderr, flush=True)
