for c in "c4 1048576 1024 e" "c1 16384 100 e" "rw 262144 256 e" "rw 262144 128 e" "c4 1048576 1024 z"; do echo -n "cov=1 "; MPROF_AAMP_COV=1 python tools/time_cfg.py $c; echo -n "auto "; python tools/time_cfg.py $c; done > gpurun_out/cov.log 2>&1
python - >> gpurun_out/cov.log 2>&1 <<'PY'
import numpy as np, paper_1901_05708_b200 as mp
from paper_1901_05708_b200 import workloads as W
for name, t, m in [("c1", W.c1(), 100), ("c4", W.c4(), 1024), ("rw256", W.random_walk(262144, 7), 256), ("c3", W.c3(), 128)]:
    r = mp.aamp(mp.make_time_series(t), mp.ProfileConfig(m, mp.DistanceKind.euclidean()))
    print(name, "fp64 ops/cell", r.info.fp64_ops_per_cell)
PY
MPROF_AAMP_COV=1 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_cov.log 2>&1
tail -15 gpurun_out/pytest_gpu_cov.log
