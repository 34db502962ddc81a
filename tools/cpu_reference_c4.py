"""One-off timing of the REFERENCE's own CPU implementation (oracle/_ref, compiled from
/root/reference/proj/src with its Release flags) on the full C4 workload (n = 2^20, m = 1024,
AAMP and ACAMP F-score) with every host thread, plus threads = 1 on the first 2^17 samples
(full C4 at one thread would take ~2.5 h), and the host CPU model. Writes
gpurun_out/r02_cpu_reference_c4.json (copied to profiles/). Run on the GPU box's host:

    python tools/cpu_reference_c4.py
"""
import json
import os
import platform
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402  (test infrastructure: the reference library itself)
from paper_1901_05708_b200 import workloads as W  # noqa: E402


def cells(n, m):
    return (n - m) * (n - m + 1) // 2


def lscpu():
    try:
        return subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    except OSError:
        return ""


t = W.c4()
m = 1024
threads = os.cpu_count() or 1
out = {"host": platform.node(), "nproc": threads, "lscpu": lscpu(),
       "library": "oracle/_ref/libmprof_ref.so (reference src/*.cpp, g++ -O3 -DNDEBUG)", "runs": []}
for fam, name in ((oracle.EUCLIDEAN, "aamp"), (oracle.ZNORM, "acamp_f")):
    for thr, n in ((threads, t.size), (1, 1 << 17)):
        x = t[:n]
        t0 = time.perf_counter()
        oracle.ref_profile(x, m, fam, threads=thr)
        s = time.perf_counter() - t0
        run = {"engine": name, "threads": thr, "n": n, "m": m, "seconds": s,
               "cells": cells(n, m), "cells_per_s": cells(n, m) / s}
        out["runs"].append(run)
        print(json.dumps(run), flush=True)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "r02_cpu_reference_c4.json").write_text(json.dumps(out, indent=1))
