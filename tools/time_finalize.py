import sys, time
sys.path.insert(0, '.')
import torch
import paper_1901_05708_b200 as mp
from paper_1901_05708_b200 import workloads as W
t = W.c4(); n = t.size; m = 1024; L = n - m + 1
d_t = torch.tensor(t, dtype=torch.float64, device="cuda")
cmp = torch.empty(L, dtype=torch.float64, device="cuda"); idx = torch.empty(L, dtype=torch.int64, device="cuda")
P = torch.empty(L, dtype=torch.float64, device="cuda")
for fam in (mp.DistanceKind.euclidean(), mp.DistanceKind.znormalized()):
    cfg = mp.ProfileConfig(m, fam)
    torch.cuda.synchronize()
    mp.sweep_device(d_t.data_ptr(), n, cfg, 0, 0, cmp.data_ptr(), idx.data_ptr())
    torch.cuda.synchronize()
    for r in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        mp.finalize_device(d_t.data_ptr(), n, cmp.data_ptr(), idx.data_ptr(), cfg, P.data_ptr())
        torch.cuda.synchronize(); el = time.perf_counter() - t0
    print(fam, "finalize ms", round(el * 1e3, 3))
