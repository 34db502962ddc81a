"""Host-side enqueue time of a planned band sweep against its device time (experiments only):
how launch-bound the constant-row window chain is when a GPU sweeps 1/world of the diagonals."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402
from paper_1901_05708_b200 import workloads as W  # noqa: E402

t = W.c4()
n, m = t.size, 1024
L = n - m + 1
ctx = mp.Context(0)
d_t = torch.tensor(t, dtype=torch.float64, device="cuda")
cmp = torch.empty(L, dtype=torch.float64, device="cuda")
idx = torch.empty(L, dtype=torch.int64, device="cuda")
for world in (1, 8):
    cuts = mp.band_cuts(n, m, 1, world)
    for fam, kind in (("aamp", mp.DistanceKind.euclidean()), ("acamp", mp.DistanceKind.znormalized())):
        cfg = mp.ProfileConfig(m, kind)
        plan = mp.Plan(d_t.data_ptr(), n, cfg, cuts[0], cuts[1], ctx=ctx)
        plan.sweep(cmp.data_ptr(), idx.data_ptr())
        torch.cuda.synchronize()
        best = (1e9, 1e9)
        for _ in range(3):
            t0 = time.perf_counter()
            info = plan.sweep(cmp.data_ptr(), idx.data_ptr())
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            best = min(best, ((t1 - t0) * 1e3, (t2 - t0) * 1e3))
        print(f"world {world} band 0 {fam}: enqueue {best[0]:.2f} ms, total {best[1]:.2f} ms, "
              f"windows {info.row_windows}, launches {info.kernel_launches}", flush=True)
        plan.close()
