"""Per-band sweep times of the C4 engines when the diagonals are split into `world` equal-area
bands (what each rank of a world-GPU run sweeps), timed one band at a time on one GPU.
max over bands ~ the multi-GPU sweep time; experiments only."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_05708_b200 as mp  # noqa: E402
from paper_1901_05708_b200 import workloads as W  # noqa: E402

args = sys.argv[1:]
cfg_name = args.pop(0) if args and not args[0].isdigit() else "C4"  # C4 (both engines) or C5
worlds = [int(x) for x in (args or ["1", "2", "4", "8"])]
ctx = mp.Context(0)
ctx.set_timing(True)
c = W.CONFIGS["C4aamp" if cfg_name == "C4" else cfg_name]
t = c.gen()
n, m = t.size, c.m
L = n - m + 1
d_t = torch.tensor(t, dtype=torch.float64, device="cuda")
cmp = torch.empty(L, dtype=torch.float64, device="cuda")
idx = torch.empty(L, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
out = {}
engines = (("aamp", mp.DistanceKind.euclidean()), ("acamp", mp.DistanceKind.znormalized()))
if cfg_name != "C4":
    engines = engines[1:]  # C5: ACAMP
for fam, kind in engines:
    cfg = mp.ProfileConfig(m, kind)
    for world in worlds:
        cuts = mp.band_cuts(n, m, 1, world)
        ms, Rs = [], []
        for a, b in zip(cuts[:-1], cuts[1:]):
            best = 1e30
            for _ in range(3 if cfg_name == "C4" else 1):
                info = mp.sweep_device(d_t.data_ptr(), n, cfg, a, b, cmp.data_ptr(), idx.data_ptr(),
                                       ctx=ctx)
                best = min(best, info.sweep_ms)
            ms.append(round(best, 3))
            Rs.append(info.rows_per_tile)
        out[f"{fam}_w{world}"] = {"band_ms": ms, "max": max(ms), "sum": round(sum(ms), 3), "R": Rs}
        # fused merge + finalize + all-gather of rank r's slice (mprof_merge_finalize_peers),
        # with every partial local here: per-rank cost of the peer-memory merge step
        if world > 1:
            import time
            from paper_1901_05708_b200.distributed import shard_range
            parts = []
            for a, b in zip(cuts[:-1], cuts[1:]):
                c_r = torch.empty(L, dtype=torch.float64, device="cuda")
                i_r = torch.empty(L, dtype=torch.int64, device="cuda")
                mp.sweep_device(d_t.data_ptr(), n, cfg, a, b, c_r.data_ptr(), i_r.data_ptr(), ctx=ctx)
                parts.append((c_r, i_r))
            outs = [(torch.empty(L, dtype=torch.float64, device="cuda"),
                     torch.empty(L, dtype=torch.int64, device="cuda")) for _ in range(world)]
            mms = []
            for r in range(world):
                lo, hi = shard_range(L, r, world)
                best = 1e30
                for _ in range(3):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    mp.merge_finalize_peers(d_t.data_ptr(), n, cfg, [x[0].data_ptr() for x in parts],
                                            [x[1].data_ptr() for x in parts],
                                            [x[0].data_ptr() for x in outs],
                                            [x[1].data_ptr() for x in outs], lo, hi, ctx=ctx)
                    torch.cuda.synchronize()
                    best = min(best, (time.perf_counter() - t0) * 1e3)
                mms.append(round(best, 3))
            out[f"{fam}_w{world}"]["merge_finalize_ms"] = mms
            del parts, outs
        print(fam, world, out[f"{fam}_w{world}"], flush=True)
print(json.dumps(out))
