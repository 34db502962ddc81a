// sweep.cuh — sm_100a diagonal-sweep kernels for AAMP / p-norm AAMP / ACAMP.
//
// Reference hot loop being replaced: the per-diagonal functors EuclidScan / PnormScan /
// ZnormScan (/root/reference/proj/src/diag_scan.cpp:7-85) driven by scan_diagonals
// (/root/reference/proj/src/detail/diag_scan.hpp:193-259), with MinBuffer's lexicographic
// (value, index) minimum (diag_scan.hpp:31-53).
//
// B200 design (see DESIGN.md for the full derivation):
//  * A CTA owns a TILE = K = T*D consecutive diagonals x R consecutive rows. Thread `tid` owns
//    D consecutive diagonals and walks the rows, so a cell costs only the O(1) slide
//    (4 FP64-pipe instructions for AAMP, p=1 and ACAMP) and each tile is seeded with one direct
//    length-m sum per diagonal (the reference's refresh rule, diag_scan.hpp:93-105, is exactly
//    "seed at multiples of R").
//  * Per-position operands are staged in shared memory per STAGE of S rows with cp.async,
//    double-buffered. Every thread reads a new column operand per row into a register ring of
//    D slots (compile-time rotation, no moves); row operands are warp broadcasts. The column
//    arrays are padded (x + x/D) so the stride-D lane pattern is bank-conflict free.
//  * Minima: the exact global profile is an array of 16-byte (value bits, index) entries merged
//    with a 128-bit atomicCAS lexicographic minimum (MinBuffer::update semantics). The hot loop
//    never touches it: each cell is compared, as a signed 32-bit integer, against the HIGH word
//    of the current row and column minima (for non-negative doubles the high word is monotone),
//    which is one ISETP per side. Only cells whose high word is <= a threshold (a possible
//    improvement or tie) take the exact slow path (`resolve`). Row candidates are warp-reduced
//    before touching global memory.
#pragma once

#include <cstdint>
#include <climits>
#include <cuda_runtime.h>

namespace mpg {

// ---------------------------------------------------------------------------------------------
// Global profile entry: comparison-space value bits (non-negative double or +inf) and index.
struct __align__(16) BestEntry {
  unsigned long long v;
  long long idx;
};

constexpr unsigned long long kInfBits = 0x7FF0000000000000ull;
constexpr long long kNoIdx = LLONG_MAX;  // "no neighbour" while merging; -1 after finalize

__device__ __forceinline__ bool lex_less(unsigned long long v, long long i, unsigned long long cv,
                                         long long ci) {
  return v < cv || (v == cv && i < ci);
}

// Exact lexicographic min-update of best[pos] with (v, idx); returns the resulting value bits.
// MinBuffer::update (/root/reference/proj/src/detail/diag_scan.hpp:37-43) as a lock-free
// 128-bit CAS loop. The initial 16-byte read may be torn by a concurrent CAS; the CAS then
// fails and returns the true entry.
__device__ __forceinline__ unsigned long long offer(BestEntry* best, long long pos,
                                                    unsigned long long v, long long idx) {
  const longlong2 raw = __ldcg(reinterpret_cast<const longlong2*>(best + pos));
  BestEntry cur{static_cast<unsigned long long>(raw.x), raw.y};
  while (lex_less(v, idx, cur.v, cur.idx)) {
    const BestEntry nv{v, idx};
    const BestEntry old = atomicCAS(best + pos, cur, nv);
    if (old.v == cur.v && old.idx == cur.idx) return v;
    cur = old;
  }
  return cur.v;
}

// ---------------------------------------------------------------------------------------------
// Distance families ("policies"). A[p] is the per-position operand pair, B[p] an optional
// per-position scalar (the z-normalization scale). step() slides the diagonal accumulator from
// cell (i, j) to (i+1, j+1) using A[i] (row) and A[j] (column); score() maps the accumulator of
// the new cell to the comparison value using B[i+1], B[j+1]. Seeds are direct length-m sums.

// AAMP: A[p] = (t[p], t[p+m]); accumulator D^2.
// Reference: incremental_euclidean_step (/root/reference/proj/include/mprof/aamp.hpp:37-42),
// direct_sq_acc (/root/reference/proj/src/detail/diag_scan.hpp:57-64).
template <bool EXACT>
struct Euclid {
  static constexpr bool kHasB = false;
  static constexpr bool kCenteredSeed = false;
  __device__ __forceinline__ static double step(double acc, double2 r, double2 c, double) {
    if constexpr (EXACT) {
      // max(0, acc - out*out + in*in), no contraction, clamp propagates (aamp.hpp:41)
      const double out = __dsub_rn(r.x, c.x);
      const double in = __dsub_rn(r.y, c.y);
      const double x = __dadd_rn(__dsub_rn(acc, __dmul_rn(out, out)), __dmul_rn(in, in));
      return (0.0 < x) ? x : 0.0;
    } else {
      const double out = r.x - c.x;
      const double in = r.y - c.y;
      return fma(in, in, fma(-out, out, acc));
    }
  }
  __device__ __forceinline__ static double score(double acc, double, double) { return acc; }
  __device__ __forceinline__ static double seed(double acc, double a, double b, double, double) {
    if constexpr (EXACT) {
      const double d = __dsub_rn(a, b);
      return __dadd_rn(acc, __dmul_rn(d, d));
    } else {
      const double d = a - b;
      return fma(d, d, acc);
    }
  }
};

// |x|^p exactly as detail::abs_pow (/root/reference/proj/include/mprof/aamp.hpp:13-20).
template <int PK>
__device__ __forceinline__ double abs_pow_exact(double x, double p) {
  const double a = fabs(x);
  if constexpr (PK == 1) return a;
  else if constexpr (PK == 3) return __dmul_rn(__dmul_rn(a, a), a);
  else if constexpr (PK == 4) return __dmul_rn(__dmul_rn(a, a), __dmul_rn(a, a));
  else return pow(a, p);
}

// p-norm AAMP: accumulator sum |t_i - t_j|^p. PK = 1, 3, 4 integer fast paths; 0 = generic pow.
// Reference: incremental_pnorm_step (aamp.hpp:45-49), direct_pnorm_acc (diag_scan.hpp:66-71).
template <int PK, bool EXACT>
struct Pnorm {
  static constexpr bool kHasB = false;
  static constexpr bool kCenteredSeed = false;
  __device__ __forceinline__ static double step(double acc, double2 r, double2 c, double p) {
    if constexpr (EXACT) {
      const double po = abs_pow_exact<PK>(__dsub_rn(r.x, c.x), p);
      const double pi = abs_pow_exact<PK>(__dsub_rn(r.y, c.y), p);
      const double x = __dadd_rn(__dsub_rn(acc, po), pi);
      return (0.0 < x) ? x : 0.0;
    } else {
      const double out = r.x - c.x;
      const double in = r.y - c.y;
      if constexpr (PK == 1) {
        return (acc - fabs(out)) + fabs(in);
      } else if constexpr (PK == 3) {
        const double o2 = out * out, i2 = in * in;
        return fma(i2, fabs(in), fma(-o2, fabs(out), acc));
      } else if constexpr (PK == 4) {
        const double o2 = out * out, i2 = in * in;
        return fma(i2, i2, fma(-o2, o2, acc));
      } else {
        return (acc - pow(fabs(out), p)) + pow(fabs(in), p);
      }
    }
  }
  __device__ __forceinline__ static double score(double acc, double, double) { return acc; }
  __device__ __forceinline__ static double seed(double acc, double a, double b, double, double p) {
    if constexpr (EXACT) {
      return __dadd_rn(acc, abs_pow_exact<PK>(__dsub_rn(a, b), p));
    } else {
      const double d = fabs(a - b);
      if constexpr (PK == 1) return acc + d;
      else if constexpr (PK == 3) return fma(d * d, d, acc);
      else if constexpr (PK == 4) { const double d2 = d * d; return fma(d2, d2, acc); }
      else return acc + pow(d, p);
    }
  }
};

// ACAMP: the accumulator is the CENTRED covariance cov(i,j) = sum (t_i - mu_i)(t_j - mu_j),
// slid as cov += df_i*dg_j + df_j*dg_i with df_p = (t[p+m]-t[p])/2,
// dg_p = (t[p+m]-mu_{p+1}) + (t[p]-mu_p)  (A[p] = (df_p, dg_p)), and B[p] = 1/||t_p - mu_p||
// (0 for flat windows). Comparison value d = 1 - corr = 1 - cov*B[i]*B[j], DZ^2 = 2m*d.
// This replaces the reference's five uncentred running sums (advance_stats + f_value,
// /root/reference/proj/include/mprof/acamp.hpp:28-60): same profile, 4 FP64 ops per cell
// instead of 16 flops + 3 divides, and no cancellation against the window level.
struct Znorm {
  static constexpr bool kHasB = true;
  static constexpr bool kCenteredSeed = true;
  __device__ __forceinline__ static double step(double acc, double2 r, double2 c, double) {
    return fma(r.x, c.y, fma(c.x, r.y, acc));
  }
  __device__ __forceinline__ static double score(double acc, double rb, double cb) {
    return fma(-(acc * cb), rb, 1.0);
  }
  // a = t_i - mu_i (row, pre-centred), b = t_j, mub = mu_j
  __device__ __forceinline__ static double seed(double acc, double a, double b, double mub,
                                                double) {
    return fma(a, b - mub, acc);
  }
};

// ---------------------------------------------------------------------------------------------
// Tile geometry and shared-memory stage buffers.

template <int D, int T, int S>
struct Geo {
  static constexpr int K = T * D;      // diagonals per tile
  static constexpr int NCOL = S + K;   // column slots touched by one stage
  __host__ __device__ static constexpr int pad(int x) { return x + x / D; }
  static constexpr int NCOLP = pad(NCOL - 1) + 1;
};

template <bool HASB, int D, int T, int S>
struct StageBuf {
  using G = Geo<D, T, S>;
  double2 colA[G::NCOLP];               // A[i0 + kb + x]
  double colB[HASB ? G::NCOLP : 2];     // B[i0 + kb + 1 + x]
  int colT[G::NCOLP];                   // hi32(best[i0 + kb + 1 + x].v)
  double2 rowA[S];                      // A[i0 + x]
  double rowB[HASB ? S : 2];            // B[i0 + 1 + x]
  int rowT[S];                          // hi32(best[i0 + 1 + x].v)
};

struct SweepParams {
  const double* t;        // series, n samples
  const double2* A;       // per-position operand pairs, valid [0, L-1)
  const double* B;        // per-position scale (z-norm), valid [0, L)
  const double* mu;       // window means (z-norm), valid [0, L)
  BestEntry* best;        // L entries
  const int2* tiles;      // (first diagonal kb, first row ra) per CTA
  int n, m, L;
  int k_hi;               // exclusive upper bound of the swept diagonal band
  int R;                  // rows per tile
  double p;
};

// ---------------------------------------------------------------------------------------------
// cp.async helpers (LDGSTS). src_bytes = 0 zero-fills the destination.

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes_src, int size) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if (size == 16) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(bytes_src));
  } else if (size == 8) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(bytes_src));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(bytes_src));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------------------------
// Exact slow path for one substep of one thread: D cells (target row `row`, columns
// col0 + d). Cells flagged by the high-word filter (or all valid cells when FORCE) are merged
// into the global profile: columns individually (distinct per cell), the row through a warp
// lexicographic reduction and one CAS per warp. Shared thresholds are lowered with atomicMin.

template <int D>
struct Cells {
  double v[D];
  int tc[D];
};

template <int D, bool FORCE>
__device__ __noinline__ Cells<D> resolve(Cells<D> c, unsigned valid, int row, int tr, int col0,
                                         BestEntry* best, int* rowT, int* colT, int colx0) {
  unsigned long long rv = kInfBits;
  int rj = INT_MAX;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (!((valid >> d) & 1u)) continue;
    const double v = c.v[d];
    const int h = __double2hiint(v);
    const bool rowhit = FORCE || h <= tr;
    const bool colhit = FORCE || h <= c.tc[d];
    if (!(rowhit || colhit)) continue;
    // clamp the comparison value at 0 (std::max(0.0, .), aamp.hpp:41; 1 - corr >= 0)
    const unsigned long long vb = (h < 0) ? 0ull : static_cast<unsigned long long>(__double_as_longlong(v));
    const int j = col0 + d;
    if (colhit) {
      const unsigned long long nb = offer(best, j, vb, row);
      const int nh = static_cast<int>(nb >> 32);
      c.tc[d] = min(c.tc[d], nh);
      if (colT) atomicMin(&colT[Geo<D, 1, 1>::pad(colx0 + d)], nh);
    }
    if (rowhit && lex_less(vb, j, rv, rj)) {
      rv = vb;
      rj = j;
    }
  }
  if (__any_sync(0xffffffffu, rj != INT_MAX)) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long ov = __shfl_xor_sync(0xffffffffu, rv, off);
      const int oj = __shfl_xor_sync(0xffffffffu, rj, off);
      if (lex_less(ov, oj, rv, rj)) {
        rv = ov;
        rj = oj;
      }
    }
    if ((threadIdx.x & 31) == 0 && rj != INT_MAX) {
      const unsigned long long nb = offer(best, row, rv, rj);
      if (rowT) atomicMin(rowT, static_cast<int>(nb >> 32));
    }
  }
  return c;
}

// ---------------------------------------------------------------------------------------------
// One stage of S (or cnt < S) row transitions i -> i+1, i in [i0, i0+cnt).

template <class P, int D, int T, int S, bool GUARD>
__device__ __forceinline__ void run_stage(StageBuf<P::kHasB, D, T, S>& sb, double (&acc)[D],
                                          int i0, int cnt, int kt, int kend, int L,
                                          BestEntry* best, double p) {
  using G = Geo<D, T, S>;
  const int xb = threadIdx.x * D;
  double2 cA[D];
  double cB[D];
  int tc[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    cA[d] = sb.colA[G::pad(xb + d)];
    if constexpr (P::kHasB) cB[d] = sb.colB[G::pad(xb + d)];
    tc[d] = sb.colT[G::pad(xb + d)];
  }
  for (int s = 0; s < cnt; s += D) {
    // pad(s + xb + D + u) == qn + u for u < D (s + xb + D is a multiple of D): constant offsets
    const int qn = G::pad(s + xb + D);
    const double2* nA = &sb.colA[qn];
    const double* nB = &sb.colB[P::kHasB ? qn : 0];
    const int* nT = &sb.colT[qn];
#pragma unroll
    for (int u = 0; u < D; ++u) {
      if (GUARD && s + u >= cnt) break;
      const int x = s + u;
      const double2 r = sb.rowA[x];
      double rb = 0.0;
      if constexpr (P::kHasB) rb = sb.rowB[x];
      const int tr = sb.rowT[x];
      const int row = i0 + x + 1;
      Cells<D> c;
      bool hit = false;
      unsigned valid = (1u << D) - 1u;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int sl = (d + u) % D;
        acc[d] = P::step(acc[d], r, cA[sl], p);
        c.v[d] = P::score(acc[d], rb, P::kHasB ? cB[sl] : 0.0);
        c.tc[d] = tc[sl];
        const int h = __double2hiint(c.v[d]);
        bool ok = true;
        if (GUARD) {
          ok = (kt + d < kend) && (row + kt + d <= L - 1);
          if (!ok) valid &= ~(1u << d);
        }
        hit |= ok && ((h <= tr) || (h <= tc[sl]));
      }
      if (__any_sync(0xffffffffu, hit)) {
        c = resolve<D, false>(c, valid, row, tr, row + kt, best, &sb.rowT[x], sb.colT, x + xb);
#pragma unroll
        for (int d = 0; d < D; ++d) tc[(d + u) % D] = c.tc[d];
      }
      // slide the column ring: slot u (used by d = 0 this substep) takes the next operand
      cA[u] = nA[u];
      if constexpr (P::kHasB) cB[u] = nB[u];
      tc[u] = nT[u];
    }
  }
}

// Issue the cp.async copies of one stage (rows i0 .. i0+S-1 transitions).
template <bool HASB, int D, int T, int S>
__device__ __forceinline__ void load_stage(StageBuf<HASB, D, T, S>& sb, const SweepParams& prm,
                                           int i0, int kb) {
  using G = Geo<D, T, S>;
  const int L = prm.L;
  const int* bestw = reinterpret_cast<const int*>(prm.best);  // word view; hi word at +1
  for (int x = threadIdx.x; x < G::NCOL; x += T) {
    const int pa = i0 + kb + x;       // A position
    const int pb = pa + 1;            // B / threshold position (target column)
    const bool va = pa < L - 1, vb = pb < L;
    const int q = G::pad(x);
    cp_async(&sb.colA[q], prm.A + (va ? pa : 0), va ? 16 : 0, 16);
    if constexpr (HASB) cp_async(&sb.colB[q], prm.B + (vb ? pb : 0), vb ? 8 : 0, 8);
    cp_async(&sb.colT[q], bestw + 4 * (vb ? pb : 0) + 1, vb ? 4 : 0, 4);
  }
  for (int x = threadIdx.x; x < S; x += T) {
    const int pa = i0 + x;
    const int pb = pa + 1;
    const bool va = pa < L - 1, vb = pb < L;
    cp_async(&sb.rowA[x], prm.A + (va ? pa : 0), va ? 16 : 0, 16);
    if constexpr (HASB) cp_async(&sb.rowB[x], prm.B + (vb ? pb : 0), vb ? 8 : 0, 8);
    cp_async(&sb.rowT[x], bestw + 4 * (vb ? pb : 0) + 1, vb ? 4 : 0, 4);
  }
}

// ---------------------------------------------------------------------------------------------
// The sweep kernel: one CTA per tile (kb, ra).

template <class P, int D, int T, int S>
__global__ void __launch_bounds__(T) sweep_kernel(const SweepParams prm) {
  using G = Geo<D, T, S>;
  using SB = StageBuf<P::kHasB, D, T, S>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SB* bufs = reinterpret_cast<SB*>(smem_raw);

  const int2 tl = prm.tiles[blockIdx.x];
  const int kb = tl.x, ra = tl.y;
  const int L = prm.L;
  const int m = prm.m;
  const int kt = kb + static_cast<int>(threadIdx.x) * D;
  const int kend = min(kb + G::K, prm.k_hi);
  const int re = min(ra + prm.R, L - kb);  // exclusive row end of the tile

  // ---- seed: acc[d] = direct length-m sum for the pair (ra, ra + kt + d) ----------------
  double acc[D];
  double muc[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    acc[d] = 0.0;
    muc[d] = 0.0;
    if constexpr (P::kCenteredSeed) {
      const int j = ra + kt + d;
      muc[d] = (j < L) ? prm.mu[j] : 0.0;
    }
  }
  {
    // stage t[ra + l ...] (row) and t[ra + kb + l ...] (columns) through shared memory in
    // chunks of SL samples; summation order l = 0..m-1 as in direct_sq_acc.
    constexpr int SL = 2 * S;
    static_assert(sizeof(SB) >= sizeof(double) * (SL + G::pad(G::K + SL)), "seed scratch");
    double* srow = reinterpret_cast<double*>(bufs);
    double* scol = srow + SL;
    const double mur = P::kCenteredSeed ? prm.mu[ra] : 0.0;
    const int xb = threadIdx.x * D;
    for (int l0 = 0; l0 < m; l0 += SL) {
      const int cnt = min(SL, m - l0);
      __syncthreads();
      for (int x = threadIdx.x; x < SL; x += T) {
        const int pos = ra + l0 + x;
        srow[x] = (x < cnt) ? (prm.t[pos] - mur) : 0.0;
      }
      for (int x = threadIdx.x; x < G::K + SL; x += T) {
        const int pos = ra + kb + l0 + x;
        scol[G::pad(x)] = (pos < prm.n) ? prm.t[pos] : 0.0;
      }
      __syncthreads();
      double w[D];
#pragma unroll
      for (int d = 0; d < D; ++d) w[d] = scol[G::pad(xb + d)];
      for (int l = 0; l < cnt; l += D) {
#pragma unroll
        for (int u = 0; u < D; ++u) {
          if (l + u >= cnt) break;
          const double a = srow[l + u];
#pragma unroll
          for (int d = 0; d < D; ++d) acc[d] = P::seed(acc[d], a, w[(d + u) % D], muc[d], prm.p);
          w[u] = scol[G::pad(l + u + xb + D)];
        }
      }
    }
  }

  // ---- the seed cells (ra, ra + k): exact merge -------------------------------------------
  {
    Cells<D> c;
    unsigned valid = 0;
    const double rb = P::kHasB ? prm.B[ra] : 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int k = kt + d;
      const bool ok = (k < kend) && (ra + k <= L - 1);
      const double cb = (P::kHasB && ok) ? prm.B[ra + k] : 0.0;
      c.v[d] = P::score(acc[d], rb, cb);
      c.tc[d] = 0;
      valid |= (ok ? 1u : 0u) << d;
    }
    resolve<D, true>(c, valid, ra, 0, ra + kt, prm.best, nullptr, nullptr, 0);
  }

  // ---- stage pipeline over the row transitions ra .. re-2 ---------------------------------
  const int steps = re - 1 - ra;
  if (steps <= 0) return;
  __syncthreads();  // seed scratch reuse
  load_stage<P::kHasB, D, T, S>(bufs[0], prm, ra, kb);
  cp_async_commit();
  int st = 0;
  for (int s0 = 0; s0 < steps; s0 += S, ++st) {
    const int cnt = min(S, steps - s0);
    const int i0 = ra + s0;
    if (s0 + S < steps) load_stage<P::kHasB, D, T, S>(bufs[(st + 1) & 1], prm, i0 + S, kb);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const bool full = (cnt == S) && (kb + G::K <= prm.k_hi) && (i0 + cnt + kb + G::K - 1 <= L - 1);
    if (full) {
      run_stage<P, D, T, S, false>(bufs[st & 1], acc, i0, cnt, kt, kend, L, prm.best, prm.p);
    } else {
      run_stage<P, D, T, S, true>(bufs[st & 1], acc, i0, cnt, kt, kend, L, prm.best, prm.p);
    }
    __syncthreads();
  }
}

}  // namespace mpg
