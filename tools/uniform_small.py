"""The reference acceptance criterion 9 shape (uniform noise, n = 8192, m = 256, AAMP) through the
host entry point: wall time per call and the sweep's own time (experiments only).
argv[1]: form (auto|cov|alt|dense), argv[2]: n."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402

form = sys.argv[1] if len(sys.argv) > 1 else "auto"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
ctx = mp.Context(0)
ctx.set_form(getattr(mp.Form, form.capitalize()))
ctx.set_timing(True)
t = np.random.default_rng(9001).uniform(-1, 1, n)
cfg = mp.ProfileConfig(256, mp.DistanceKind.euclidean())
ts = mp.make_time_series(t)
for _ in range(3):
    t0 = time.perf_counter()
    r = mp.aamp(ts, cfg, ctx=ctx)
    wall = time.perf_counter() - t0
print(form, n, r.info.policy, "tiles", r.info.tiles, "R", r.info.rows_per_tile, "sweep_ms",
      round(r.info.sweep_ms, 3), "wall_ms", round(wall * 1e3, 3), "launches", r.info.kernel_launches)
