"""Workload for compute-sanitizer runs (racecheck / synccheck / memcheck; experiments and
evidence, not a test): every sweep kernel family on a C1-sized series (n = 16384, m = 100) and an
n = 20000, m = 1024 series, with the filter forms forced so that Wide<EuclidCov>, EuclidCov,
Euclid, Wide<Znorm<0>>, Znorm<0>, Znorm<1>, Pnorm<1> and Pnorm<3> all run, plus the exact mode,
FP32 mode and an EngineState extension. Prints the policy of every call.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py [small]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402
from paper_1901_05708_b200 import workloads as W  # noqa: E402

small = len(sys.argv) > 1 and sys.argv[1] == "small"
ctx = mp.Context(0)
ctx.set_row_const(1)  # the constant-row kernels (default)
r = np.random.default_rng(11)
cases = [("C1", W.c1(), 100)]
if not small:
    cases.append(("walk20000", np.cumsum(r.standard_normal(20000)), 1024))
for name, t, m in cases:
    ts = mp.make_time_series(t)
    for fam, kind in (("aamp", mp.DistanceKind.euclidean()), ("acamp", mp.DistanceKind.znormalized())):
        for form in (mp.Form.Wide, mp.Form.Cov, mp.Form.Alt):
            ctx.set_form(form)
            for excl in (1, m):
                cfg = mp.ProfileConfig(m, kind)
                cfg.exclusion = excl
                res = (mp.aamp if fam == "aamp" else mp.acamp)(ts, cfg, ctx=ctx)
                print(name, fam, form.name, excl, res.info.policy, flush=True)
    ctx.set_form(mp.Form.Auto)
    for p in (1.0, 3.0, 2.5):
        res = mp.aamp_pnorm(ts, mp.ProfileConfig(m, mp.DistanceKind.pnorm(p)), ctx=ctx)
        print(name, "pnorm", p, res.info.policy, flush=True)
    cfg = mp.ProfileConfig(m, mp.DistanceKind.euclidean())
    cfg.exact, cfg.refresh_interval = True, 512
    print(name, "exact", mp.aamp(ts, cfg, ctx=ctx).info.policy, flush=True)
    cfg = mp.ProfileConfig(m, mp.DistanceKind.znormalized())
    cfg.precision = mp.Precision.FP32
    print(name, "fp32", mp.acamp(ts, cfg, ctx=ctx).info.policy, flush=True)
    st = mp.build_engine_state(mp.make_time_series(t[:-500]), mp.ProfileConfig(m, mp.DistanceKind.euclidean()))
    g = mp.extend_profile(st, t[-500:])
    print(name, "extend", g.info.policy, flush=True)
print("sanitize case done")
