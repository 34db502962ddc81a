"""Bitwise comparison of two builds of libmprof_gpu.so on the C1/C2/C4 series (experiments only).
    MPROF_GPU_LIB=<lib> python tools/cmp_libs.py dump <out.npz>;  python tools/cmp_libs.py cmp a.npz b.npz"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

if sys.argv[1] == "dump":
    import paper_1901_05708_b200 as mp
    from paper_1901_05708_b200 import workloads as W
    out = {}
    cases = [("c1e", W.c1(), 100, "e"), ("c2z", W.c2(), 256, "z"), ("c4e", W.c4(n=1 << 18), 1024, "e"),
             ("c4z", W.c4(n=1 << 18), 1024, "z"), ("lvl", W.random_walk(50000, 3) + 1e6, 300, "z"),
             ("lvle", W.random_walk(50000, 3) + 1e6, 300, "e")]
    for name, t, m, fam in cases:
        kind = mp.DistanceKind.euclidean() if fam == "e" else mp.DistanceKind.znormalized()
        fn = mp.aamp if fam == "e" else mp.acamp
        r = fn(mp.make_time_series(t), mp.ProfileConfig(m, kind))
        out[name + "_P"] = np.asarray(r.distances)
        out[name + "_I"] = np.asarray(r.nn_index)
    np.savez(sys.argv[2], **out)
else:
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        same = np.array_equal(a[k].view(np.uint64) if a[k].dtype == np.float64 else a[k],
                              b[k].view(np.uint64) if b[k].dtype == np.float64 else b[k])
        print(k, "identical" if same else f"DIFFER ({np.count_nonzero(a[k] != b[k])} entries)")
