"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libmprof_ref.so, built from
/root/reference/proj/src by oracle/Makefile). Run here (where /root/reference exists):

    python tests/golden/make_golden.py

The GPU box never reads /root/reference: the tests there use these committed vectors.

Contents
* fixtures.npz — the reference's committed n=1000 fixtures (/root/reference/proj/data/*.csv,
  read at generation time) with the reference engines' profiles at m=50 (the CLI acceptance
  setting, /root/reference/proj/tests/acceptance.cpp:382-412) and the brute-force oracle.
* corpus.npz — 60 seeded series shaped like the acceptance corpus (n in [16,512], m in
  [2, n/2], alternating uniform(-1,1) / N(0,1); acceptance.cpp:59-71) with the reference's
  aamp, aamp_pnorm (p = 1, 2, 3, 4.5) and acamp (FScore, SquaredDistance) profiles.
* exact.npz — random walks at level 1000 run by the reference with refresh_interval = R:
  comparison values for the bit-exact GPU parity build (SURVEY.md §7 hard part 5).
"""
from __future__ import annotations

import sys
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent
REF_DATA = Path("/root/reference/proj/data")


def read_csv(p: Path) -> np.ndarray:
    lines = p.read_text().splitlines()[1:]
    return np.array([float(x.split(",")[0]) for x in lines if x.strip()])


def fixtures():
    out = {}
    for name, fam, p in [("euclidean", oracle.EUCLIDEAN, 2.0), ("pnorm", oracle.PNORM, 3.0),
                         ("znorm", oracle.ZNORM, 2.0)]:
        t = read_csv(REF_DATA / f"fixture_{name}.csv")
        out[f"{name}_t"] = t
        P, I = oracle.ref_profile(t, 50, fam, p)
        out[f"{name}_P"], out[f"{name}_I"] = P, I
        if fam == oracle.ZNORM:
            P2, I2 = oracle.ref_profile(t, 50, fam, p, use_f=False)
            out[f"{name}_Psq"], out[f"{name}_Isq"] = P2, I2
        Pb, Ib = oracle.ref_brute(t, 50, fam, p)
        out[f"{name}_Pbrute"], out[f"{name}_Ibrute"] = Pb, Ib
    np.savez_compressed(OUT / "fixtures.npz", **out)


def corpus(count=60, seed=1001):
    r = np.random.Generator(np.random.PCG64(seed))
    out = {"count": np.array(count)}
    for c in range(count):
        n = int(16 + r.integers(0, 497))
        m = int(2 + r.integers(0, n // 2 - 1))
        t = r.uniform(-1, 1, n) if c % 2 == 0 else r.standard_normal(n)
        out[f"t{c}"] = t
        out[f"m{c}"] = np.array(m)
        P, I = oracle.ref_profile(t, m, oracle.EUCLIDEAN)
        out[f"e_P{c}"], out[f"e_I{c}"] = P, I
        for p in (1.0, 2.0, 3.0, 4.5):
            P, I = oracle.ref_profile(t, m, oracle.PNORM, p)
            out[f"p{p}_P{c}"], out[f"p{p}_I{c}"] = P, I
        P, I = oracle.ref_profile(t, m, oracle.ZNORM, use_f=True)
        out[f"zf_P{c}"], out[f"zf_I{c}"] = P, I
        P, I = oracle.ref_profile(t, m, oracle.ZNORM, use_f=False)
        out[f"zs_P{c}"], out[f"zs_I{c}"] = P, I
    np.savez_compressed(OUT / "corpus.npz", **out)


def exact():
    out = {}
    cases = [("walk", 3000, 64, 256, 1), ("walk_excl", 2500, 48, 128, 48), ("walk_r1", 600, 16, 1, 1),
             ("walk_r7", 900, 20, 7, 3)]
    for name, n, m, R, excl in cases:
        r = np.random.Generator(np.random.PCG64(zlib.crc32(name.encode())))
        t = 1000.0 + np.cumsum(r.standard_normal(n))
        out[f"{name}_t"] = t
        out[f"{name}_meta"] = np.array([m, R, excl])
        for tag, fam, p in [("e", oracle.EUCLIDEAN, 2.0), ("p1", oracle.PNORM, 1.0),
                            ("p3", oracle.PNORM, 3.0), ("p4", oracle.PNORM, 4.0)]:
            cmp, P, I = oracle.ref_engine(t, m, fam, p, exclusion=excl, refresh=R)
            out[f"{name}_{tag}_cmp"], out[f"{name}_{tag}_P"], out[f"{name}_{tag}_I"] = cmp, P, I
    np.savez_compressed(OUT / "exact.npz", **out)


if __name__ == "__main__":
    if not oracle.ref_available():
        oracle.build()
    fixtures()
    corpus()
    exact()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
