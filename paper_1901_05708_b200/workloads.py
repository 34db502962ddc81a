"""Seeded synthetic series for the five BASELINE.json configurations.

No public dataset is involved: the reference benchmarks seeded uniform data
(/root/reference/proj/src/bench.cpp:25-31) and the paper uniform random data
(/root/reference/PAPER.md:474). These generators follow BASELINE.json's recipes with NumPy's
PCG64; every call with the same arguments yields the same bytes (sha256 reported by
``fingerprint``).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

SEED_BASE = 20261001


def _rng(cfg_index: int, seed: int | None = None) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + cfg_index if seed is None else seed))


def random_walk(n: int, seed: int) -> np.ndarray:
    r = np.random.Generator(np.random.PCG64(seed))
    return np.cumsum(r.standard_normal(n))


def c1(n: int = 16384, seed: int | None = None) -> np.ndarray:
    """C1: Gaussian random walk, unit-variance steps (AAMP, m=100)."""
    r = _rng(1, seed)
    t = np.empty(n)
    t[0] = 0.0
    t[1:] = np.cumsum(r.standard_normal(n - 1))
    return t


def _slots(r, n, count, width):
    """`count` non-overlapping start offsets for windows of `width` samples."""
    nslots = n // width
    chosen = np.sort(r.choice(nslots, size=count, replace=False))
    return [int(s * width) for s in chosen]


def c2(n: int = 131072, seed: int | None = None, motifs: int = 20, flats: int = 5,
       motif_len: int = 256, flat_len: int = 512) -> np.ndarray:
    """C2: random walk; 20 windows replaced by t[s] + 3 sin(2 pi l/32) hann(l) (exact affine
    copies of one sine burst, amplitude 3, length 256) and 5 runs of 512 samples set to the
    run's first value (flat, zero-sigma windows)."""
    r = _rng(2, seed)
    t = np.cumsum(r.standard_normal(n))
    l = np.arange(motif_len)
    burst = 3.0 * np.sin(2 * np.pi * l / 32.0) * np.hanning(motif_len)
    # one slot grid for both kinds so nothing overlaps
    width = max(2 * motif_len, 2 * flat_len)
    starts = _slots(r, n - width, motifs + flats, width)
    kinds = r.permutation(np.array([0] * motifs + [1] * flats))
    for s, k in zip(starts, kinds):
        off = s + int(r.integers(0, width // 4))
        if k == 0:
            t[off:off + motif_len] = t[off] + burst
        else:
            t[off:off + flat_len] = t[off]
    return t


def c3(n: int = 262144, seed: int | None = None) -> np.ndarray:
    """C3: sin(2 pi i/97) + sin(2 pi i/503) + sin(2 pi i/2011) + N(0, 0.1)."""
    r = _rng(3, seed)
    i = np.arange(n, dtype=np.float64)
    return (np.sin(2 * np.pi * i / 97.0) + np.sin(2 * np.pi * i / 503.0)
            + np.sin(2 * np.pi * i / 2011.0) + 0.1 * r.standard_normal(n))


def c4(n: int = 1 << 20, seed: int | None = None, anomaly: int = 500) -> np.ndarray:
    """C4: random walk N(0,1) with one 500-step window of 5x step variance at a random offset."""
    r = _rng(4, seed)
    steps = r.standard_normal(n)
    a = int(r.integers(0, n - anomaly))
    steps[a:a + anomaly] *= np.sqrt(5.0)
    return np.cumsum(steps)


def c5(n: int = 1 << 22, seed: int | None = None, regime: int = 65536) -> np.ndarray:
    """C5: piecewise random walk, regime shifts every 65536 samples, step sigma ~ U[0.5, 2]."""
    r = _rng(5, seed)
    steps = r.standard_normal(n)
    nreg = (n + regime - 1) // regime
    sig = r.uniform(0.5, 2.0, size=nreg)
    steps *= np.repeat(sig, regime)[:n]
    return np.cumsum(steps)


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    m: int
    family: str          # "euclidean" | "pnorm" | "znorm"
    p: float = 2.0
    gen: object = None


CONFIGS = {
    "C1": Config("C1", 16384, 100, "euclidean", gen=c1),
    "C2": Config("C2", 131072, 256, "znorm", gen=c2),
    "C3p1": Config("C3p1", 262144, 128, "pnorm", 1.0, gen=c3),
    "C3p3": Config("C3p3", 262144, 128, "pnorm", 3.0, gen=c3),
    "C4aamp": Config("C4aamp", 1 << 20, 1024, "euclidean", gen=c4),
    "C4acamp": Config("C4acamp", 1 << 20, 1024, "znorm", gen=c4),
    "C5": Config("C5", 1 << 22, 512, "znorm", gen=c5),
}


def fingerprint(t: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(t, dtype=np.float64).tobytes()).hexdigest()[:16]


def cells(n: int, m: int, exclusion: int = 1) -> int:
    """Admissible cells: sum_{k=exclusion}^{n-m} (L - k); (n-m)(n-m+1)/2 at exclusion 1
    (/root/reference/proj/src/bench.cpp:110)."""
    L = n - m + 1
    c = L - exclusion
    return c * (c + 1) // 2 if c > 0 else 0
