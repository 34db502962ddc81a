"""Planned sweeps (mprof_plan_create / mprof_plan_sweep): every per-series decision taken once,
the sweep itself only kernel launches (no host synchronisation: capturable in a CUDA graph). The
results must equal mprof_sweep_device's bit for bit, for every family, mode and band."""
import numpy as np
import pytest

from paper_1901_05708_b200 import workloads as W

pytestmark = pytest.mark.gpu


def cases(mp):
    r = np.random.default_rng(41)
    walk = 30 + np.cumsum(r.standard_normal(20000))
    walk[9000:9500] = walk[9000]
    yield "aamp", walk, 256, mp.DistanceKind.euclidean(), {}
    yield "pnorm3", walk, 128, mp.DistanceKind.pnorm(3.0), {}
    yield "pnorm2.5", walk, 128, mp.DistanceKind.pnorm(2.5), {}
    yield "acamp", walk, 200, mp.DistanceKind.znormalized(), {}
    yield "exact", walk, 64, mp.DistanceKind.euclidean(), {"exact": True, "refresh_interval": 512}
    yield "fp32", walk, 256, mp.DistanceKind.znormalized(), {"precision": mp.Precision.FP32}
    yield "c4prefix", W.c4()[: 1 << 18], 1024, mp.DistanceKind.znormalized(), {}  # probe runs


def test_plan_equals_sweep_device(mp):
    torch = pytest.importorskip("torch")
    for name, t, m, kind, extra in cases(mp):
        cfg = mp.ProfileConfig(m, kind)
        for k, v in extra.items():
            setattr(cfg, k, v)
        n, L = t.size, t.size - m + 1
        d_t = torch.tensor(t, device="cuda")
        cuts = mp.band_cuts(n, m, 1, 3)
        for band in [(0, 0), (cuts[1], cuts[2])]:
            ref_c = torch.empty(L, dtype=torch.float64, device="cuda")
            ref_i = torch.empty(L, dtype=torch.int64, device="cuda")
            torch.cuda.synchronize()
            mp.sweep_device(d_t.data_ptr(), n, cfg, band[0], band[1], ref_c.data_ptr(), ref_i.data_ptr())
            plan = mp.Plan(d_t.data_ptr(), n, cfg, band[0], band[1])
            for _ in range(2):  # repeated sweeps of one plan
                c = torch.full((L,), -1.0, dtype=torch.float64, device="cuda")
                i = torch.full((L,), -7, dtype=torch.int64, device="cuda")
                torch.cuda.synchronize()
                info = plan.sweep(c.data_ptr(), i.data_ptr())
                torch.cuda.synchronize()
                assert torch.equal(c, ref_c) and torch.equal(i, ref_i), (name, band)
                assert info.cells > 0 and info.policy
            plan.close()
