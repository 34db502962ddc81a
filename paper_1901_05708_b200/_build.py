"""In-tree build of the native libraries (sm_100a only).

* ``paper_1901_05708_b200/libmprof_gpu.so`` — CUDA kernels + the C ABI (include/mprof_gpu.h)
  + the C++ drop-in shim (include/mprof/*.hpp, namespace mprof).
* ``oracle/liboracle.so`` — the CPU restatement used ONLY by tests / smoke / bench baselines.
* ``oracle/_ref/libmprof_ref.so`` — the reference library itself, compiled from
  /root/reference/proj/src when that tree exists (this container; never on the GPU box).
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_1901_05708_b200"
CSRC = PKG / "csrc"
LIB = PKG / "libmprof_gpu.so"
CLI = PKG / "bin" / "mprof"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
           "--expt-relaxed-constexpr"]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))  # csrc/cli is the executable


def _deps():
    return _sources() + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted(
        (ROOT / "include").rglob("*.h*"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd, cwd=ROOT):
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(map(str, cmd))}\n{r.stdout}\n{r.stderr}")
    return r


def build_gpu(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale(LIB, _deps()):
        return LIB
    objdir = ROOT / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    jobs = []
    for src in _sources():
        obj = objdir / (src.name + ".o")
        cmd = [NVCC, *NVFLAGS, *ARCH, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        jobs.append(cmd)
        objs.append(str(obj))
    # the translation units are independent: compile them side by side
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(4, len(jobs))) as pool:
        for r in pool.map(_run, jobs):
            if verbose:
                print(r.stderr)
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart"])
    os.replace(tmp, LIB)
    return LIB


def build_cli(force: bool = False) -> Path:
    """The `mprof` command line front end (C++, links libmprof_gpu.so via rpath)."""
    src = CSRC / "cli" / "mprof_main.cpp"
    deps = [src, LIB] + sorted((ROOT / "include").rglob("*.h*"))
    if not force and not _stale(CLI, deps):
        return CLI
    CLI.parent.mkdir(parents=True, exist_ok=True)
    _run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), str(src), "-L", str(PKG),
          "-lmprof_gpu", "-Wl,-rpath,$ORIGIN/..", "-o", str(CLI)])
    return CLI


def build_oracle(force: bool = False) -> None:
    """Builds oracle/liboracle.so (always) and oracle/_ref (when /root/reference exists)."""
    _run(["make", "-C", str(ROOT / "oracle"), "all"])


def build(force: bool = False, verbose: bool = False) -> None:
    build_gpu(force=force, verbose=verbose)
    build_cli(force=force)
    build_oracle(force=force)


if __name__ == "__main__":
    import sys
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built", LIB)
