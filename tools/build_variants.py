"""Build tile-parameter variants of libmprof_gpu.so into build/variants/ (experiments only).

    python tools/build_variants.py D,T,S,MINB [D,T,S,MINB ...]
"""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1901_05708_b200 import _build as B  # noqa: E402

OUT = ROOT / "build" / "variants"


def one(spec):
    D, T, S, MB, *extra = spec.split(",")
    tag = f"d{D}_t{T}_s{S}_b{MB}" + "".join("_" + e.replace("=", "").replace("MPROF_", "").lower() for e in extra)
    objdir = OUT / tag
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in B._sources():
        obj = objdir / (src.name + ".o")
        B._run([B.NVCC, *B.NVFLAGS, *B.ARCH, "-I", str(ROOT / "include"), f"-DMPROF_TILE_D={D}",
                f"-DMPROF_TILE_T={T}", f"-DMPROF_TILE_S={S}", f"-DMPROF_MIN_BLOCKS={MB}",
                *[f"-D{e}" for e in extra],
                "-c", str(src), "-o", str(obj)])
        objs.append(str(obj))
    lib = OUT / f"libmprof_gpu_{tag}.so"
    B._run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *objs, "-lcudart"])
    return str(lib)


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for lib in ex.map(one, sys.argv[1:]):
            print(lib)
