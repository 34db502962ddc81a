"""bench.py's N > 1 path: two ranks under torchrun on the one GPU of the
box (--share-gpu: both ranks on cuda:0, gloo + host barriers, since NCCL cannot run two ranks on
one device), equal-area bands, the fused peer-memory merge + finalize over CUDA-IPC buffers, the
max-over-ranks device timing and the end-to-end leg. The driver's 8-GPU runs use the same code
with NCCL stream-ordered barriers."""
import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_on_one_gpu():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--share-gpu", "--steps", "2", "--warmup", "1", "--series-len", "65536",
           "--window", "256", "--no-cpu-baseline", "--no-configs"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-5000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["ms_per_step"] > 0
    assert "fused peer-memory merge" in d["config"]["parallelism"]
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
