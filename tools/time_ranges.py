"""Sweep time of arbitrary C4 diagonal ranges under several rows-per-tile settings (experiments).
usage: time_ranges.py FAMILY R1,R2,.. lo:hi [lo:hi ...]   (R=0 -> library's choice)
The library reads MPROF_ROWS_PER_TILE once per process, so each R runs in its own process."""
import os
import subprocess
import sys
from pathlib import Path

if len(sys.argv[2].split(",")) > 1:
    for R in sys.argv[2].split(","):
        subprocess.run([sys.executable, __file__, sys.argv[1], R, *sys.argv[3:]], check=True)
    sys.exit(0)

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402
from paper_1901_05708_b200 import workloads as W  # noqa: E402

fam = sys.argv[1]
Rs = [int(x) for x in sys.argv[2].split(",")]
ranges = [tuple(int(v) for v in a.split(":")) for a in sys.argv[3:]]
ctx = mp.Context(0)
ctx.set_timing(True)
t = W.c4()
n, m = t.size, 1024
L = n - m + 1
kind = mp.DistanceKind.euclidean() if fam == "aamp" else mp.DistanceKind.znormalized()
cfg = mp.ProfileConfig(m, kind)
d_t = torch.tensor(t, dtype=torch.float64, device="cuda")
cmp = torch.empty(L, dtype=torch.float64, device="cuda")
idx = torch.empty(L, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
for R in Rs:
    if R:
        os.environ["MPROF_ROWS_PER_TILE"] = str(R)
    else:
        os.environ.pop("MPROF_ROWS_PER_TILE", None)
    for lo, hi in ranges:
        best, info = 1e30, None
        for _ in range(3):
            info = mp.sweep_device(d_t.data_ptr(), n, cfg, lo, hi, cmp.data_ptr(), idx.data_ptr(), ctx=ctx)
            best = min(best, info.sweep_ms)
        print(f"{fam} R={R or info.rows_per_tile} [{lo},{hi}) tiles {info.tiles} ms {best:.3f} "
              f"Gcells/s {info.cells / best / 1e6:.1f}", flush=True)
