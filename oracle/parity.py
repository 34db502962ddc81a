"""TEST INFRASTRUCTURE ONLY — parity rules of SURVEY.md §8(d) for comparing a GPU profile with
the reference (or its restatement) on the same input.

within(a, b, tol) is testutil::within (/root/reference/proj/tests/helpers.hpp:27-31).

Per entry i:
  1. identical +inf / -1 pattern;
  2. pass if within(P_gpu, P_ref, tol);
  3. otherwise d*(i, j) is evaluated in long double (oracle.dist_exact) for j in {I_gpu, I_ref};
     pass ("reference drift") if within(P_gpu, d*(i, I_gpu), tol) and
     d*(i, I_gpu) <= d*(i, I_ref) * (1 + tol);
  3b. (z-normalized only) near-duplicates: pass if |P_gpu - d*(i, I_gpu)| <= abs_bound and
     d*(i, I_gpu) <= d*(i, I_ref) + abs_bound;
  4. I equal, or a tie: within(d*(i, I_gpu), d*(i, I_ref), tol) (or |.| <= abs_bound under 3b).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import dist_exact


def within(a, b, tol):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    with np.errstate(invalid="ignore"):
        scale = np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
        return (a == b) | (np.abs(a - b) <= tol * scale)


@dataclass
class ParityReport:
    n_entries: int = 0
    p_exact_match: int = 0          # rule 2 passes
    ref_drift: int = 0              # rule 3 passes
    near_dup: int = 0               # rule 3b passes
    index_equal: int = 0
    index_ties: int = 0             # rule 4 ties
    failures: list = field(default_factory=list)
    max_rel_p: float = 0.0

    @property
    def ok(self) -> bool:
        return not self.failures

    def summary(self) -> str:
        return (f"entries={self.n_entries} P_within={self.p_exact_match} drift={self.ref_drift} "
                f"near_dup={self.near_dup} I_equal={self.index_equal} I_ties={self.index_ties} "
                f"max_rel_P={self.max_rel_p:.3e} failures={len(self.failures)}"
                + (f" first={self.failures[:5]}" if self.failures else ""))


def check(t, m, family, P_gpu, I_gpu, P_ref, I_ref, tol=1e-9, p=2.0, flat=None,
          abs_bound=None) -> ParityReport:
    P_gpu = np.asarray(P_gpu, dtype=np.float64)
    P_ref = np.asarray(P_ref, dtype=np.float64)
    I_gpu = np.asarray(I_gpu, dtype=np.int64)
    I_ref = np.asarray(I_ref, dtype=np.int64)
    rep = ParityReport(n_entries=int(P_ref.shape[0]))
    if P_gpu.shape != P_ref.shape or I_gpu.shape != I_ref.shape:
        rep.failures.append(("length", P_gpu.shape, P_ref.shape))
        return rep
    inf_g = np.isinf(P_gpu) | (I_gpu < 0)
    inf_r = np.isinf(P_ref) | (I_ref < 0)
    bad = np.flatnonzero(inf_g != inf_r)
    for i in bad[:20]:
        rep.failures.append(("inf_pattern", int(i), float(P_gpu[i]), float(P_ref[i])))
    fin = ~inf_g & ~inf_r
    with np.errstate(invalid="ignore"):
        scale = np.maximum(1.0, np.maximum(np.abs(P_gpu), np.abs(P_ref)))
        rel = np.where(fin, np.abs(P_gpu - P_ref) / scale, 0.0)
    rep.max_rel_p = float(rel.max()) if rel.size else 0.0
    p_ok = within(P_gpu, P_ref, tol) & fin
    rep.p_exact_match = int(p_ok.sum())
    i_eq = (I_gpu == I_ref) & fin
    rep.index_equal = int(i_eq.sum())
    need = np.flatnonzero(fin & (~p_ok | ~i_eq))
    if need.size:
        dg = dist_exact(t, need, I_gpu[need], m, family, p, flat)
        dr = dist_exact(t, need, I_ref[need], m, family, p, flat)
        for k, i in enumerate(need):
            pg, g, r = P_gpu[i], dg[k], dr[k]
            if p_ok[i]:
                p_pass = True
            elif within(pg, g, tol) and g <= r * (1 + tol):
                p_pass = True
                rep.ref_drift += 1
            elif abs_bound is not None and abs(pg - g) <= abs_bound and g <= r + abs_bound:
                p_pass = True
                rep.near_dup += 1
            else:
                p_pass = False
            if i_eq[i]:
                i_pass = True
            elif within(g, r, tol) or (abs_bound is not None and abs(g - r) <= abs_bound) \
                    or g <= r:
                # a tie, or the GPU's neighbour is at least as close as the reference's
                i_pass = True
                rep.index_ties += 1
            else:
                i_pass = False
            if not (p_pass and i_pass):
                rep.failures.append((int(i), float(pg), float(P_ref[i]), int(I_gpu[i]),
                                     int(I_ref[i]), float(g), float(r)))
    return rep
