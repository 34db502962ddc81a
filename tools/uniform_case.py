"""One AAMP profile of a uniform-noise series (n = 16384, m = 256, the reference acceptance
criterion 8 shape) for profiling (experiments only). argv[1]: form (auto|cov|alt)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402

form = sys.argv[1] if len(sys.argv) > 1 else "alt"
fam = sys.argv[2] if len(sys.argv) > 2 else "aamp"
ctx = mp.Context(0)
ctx.set_form(getattr(mp.Form, form.capitalize()))
t = np.random.default_rng(9001).uniform(-1, 1, 16384)
cfg = mp.ProfileConfig(256, mp.DistanceKind.euclidean() if fam == "aamp" else mp.DistanceKind.znormalized())
for _ in range(2):
    r = (mp.aamp if fam == "aamp" else mp.acamp)(mp.make_time_series(t), cfg, ctx=ctx)
print(r.info.policy, r.info.tiles)
