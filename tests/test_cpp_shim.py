"""The C++ drop-in (include/mprof/*.hpp): reference-style code compiles and links against
libmprof_gpu.so; on a GPU it reproduces the reference's known answers and exercises ProgressFn
(ticks + cancellation), build_engine_state / extend_profile, brute_profile and the multi-device
entry point (tests/cpp/shim_demo.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1901_05708_b200"


def build_demo(tmp_path):
    exe = tmp_path / "shim_demo"
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                        str(ROOT / "tests" / "cpp" / "shim_demo.cpp"), "-L", str(PKG),
                        "-lmprof_gpu", f"-Wl,-rpath,{PKG}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_shim_compiles_links_and_reports_no_device(mp, tmp_path):
    exe = build_demo(tmp_path)
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 3, r.stdout + r.stderr


@pytest.mark.gpu
def test_shim_reproduces_known_answers_on_gpu(mp, tmp_path):
    exe = build_demo(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
