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
// Operand layouts of A[p] (built by the host, see k_build_pairs / k_znorm_pairs):
enum PairKind { kPairsRaw = 0, kPairsDeltaSum = 1, kPairsZnorm = 2 };

// Fast-filter key of a cell: for distance-like accumulators the high word of the value (smaller
// = better, monotone for non-negative doubles); see Znorm for the covariance key.
__device__ __forceinline__ int hi_key(double v) { return __double2hiint(v); }

template <bool EXACT>
struct Euclid {
  static constexpr bool kHasB = false;
  static constexpr bool kCenteredSeed = false;
  static constexpr bool kCovFilter = false;
  static constexpr bool kColScale = false;
  // fast mode: A[p] = (delta_p, sigma_p) = (t[p+m] - t[p], t[p+m] + t[p]) and
  //   in^2 - out^2 = (a' - b')^2 - (a - b)^2 = (delta_i - delta_j)(sigma_i - sigma_j),
  // one DFMA + two DADD per cell instead of two DFMA + two DADD.
  // exact mode: A[p] = (t[p], t[p+m]) and the reference's evaluation order.
  static constexpr int kPairs = EXACT ? kPairsRaw : kPairsDeltaSum;
  __device__ __forceinline__ static double step(double acc, double2 r, double2 c, double) {
    if constexpr (EXACT) {
      // max(0, acc - out*out + in*in), no contraction, clamp propagates (aamp.hpp:41)
      const double out = __dsub_rn(r.x, c.x);
      const double in = __dsub_rn(r.y, c.y);
      const double x = __dadd_rn(__dsub_rn(acc, __dmul_rn(out, out)), __dmul_rn(in, in));
      return (0.0 < x) ? x : 0.0;
    } else {
      return fma(r.x - c.x, r.y - c.y, acc);
    }
  }
  __device__ __forceinline__ static int key(double acc) { return hi_key(acc); }
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
  static constexpr bool kCovFilter = false;
  static constexpr bool kColScale = false;
  static constexpr int kPairs = kPairsRaw;
  __device__ __forceinline__ static int key(double acc) { return hi_key(acc); }
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
//
// Fast filter on the covariance alone (no per-cell normalisation): for a cell that can reach a
// threshold tau (d <= tau < 1), cov >= (1 - tau) / (B_i B_j) >= (1 - tau_max) / (max B_r max B_c)
// over the rows / columns of the thread's block, so the hot loop keeps only max(cov) — the key
// ~hi(cov) is decreasing in cov — and the exact score is evaluated in the replay only:
// 2 DFMA per cell.
// COLSCALE selects the filter form (see run_stage): 0 = covariance only, 1 = cov * B_j.
template <bool COLSCALE>
struct Znorm {
  static constexpr bool kHasB = true;
  static constexpr bool kCenteredSeed = true;
  static constexpr bool kCovFilter = true;
  static constexpr bool kColScale = COLSCALE;
  static constexpr int kPairs = kPairsZnorm;
  __device__ __forceinline__ static int key(double acc) { return ~__double2hiint(acc); }
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
  static constexpr int K = T * D;        // diagonals per tile
  static constexpr int NCOL = S + K;     // column operands live during one stage
  static constexpr int RING = K + 2 * S; // ring slots: live stage + the prefetched next stage
  __host__ __device__ static constexpr int pad(int x) { return x + x / D; }
  static constexpr int NCOLP = pad(NCOL - 1) + 1;
  static constexpr int RINGP = pad(RING - 1) + 1;
};

// Shared memory of one CTA. Column operands live in a RING indexed by X = (column position -
// tile column base): stage st uses X in [st*S, st*S + S + K) and prefetches only its S new
// operands for stage st+1, so one copy of the K-wide window is resident (not two). Thresholds
// (4 B per column) are re-read for the whole live window every stage (fresh minima from other
// CTAs) and double-buffered with the row operands.
template <bool HASB, int D, int T, int S>
struct SweepSmem {
  using G = Geo<D, T, S>;
  static_assert(G::RING % D == 0 && S % D == 0, "stage and ring must be multiples of D");
  static constexpr int NCB = G::NCOL / D + 1;  // column blocks of D
  double2 colA[G::RINGP];                      // ring: A[cbase + X] at pad(X mod RING)
  double colB[HASB ? G::RINGP : 2];            // ring: B[cbase + 1 + X]
  int colT[2][G::NCOLP];                       // hi32(best[i0 + kb + 1 + x].v), exact
  int colBM[2][NCB];                           // max of colT over aligned blocks of D
  double2 rowA[2][S];                          // A[i0 + x]
  double rowB[2][HASB ? S : 2];                // B[i0 + 1 + x]
  int rowT[2][S];                              // hi32(best[i0 + 1 + x].v), exact
  int rowBM[2][S / D];                         // max of rowT over aligned blocks of D
  // z-norm filter scales, rounded DOWN (a smaller scale only loosens the filter): per aligned
  // block of D columns in a ring of RING/D blocks (filled once, when the block arrives) and per
  // block of D rows of the stage.
  float colIB[HASB ? G::RING / D : 1];         // <= 1 / max colB of the block
  float rowIB[2][HASB ? S / D : 1];            // <= 1 / max rowB of the block
  float rowIBx[2][HASB ? S : 1];               // <= 1 / rowB of each row
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
  unsigned long long* stats;  // optional diagnostics (MPROF_STATS): [0] replays [1] offers
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
};

// Exact slow path for one BLOCK of D sub-steps of ONE lane, called divergently when the block's
// minimum high word passed the block threshold. The block is REPLAYED from the accumulators saved
// at its start with the identical arithmetic (bit-identical cell values), and every cell whose
// high word is <= the current exact column (row) threshold in shared memory (colT / rowT) is
// merged into the global column (row) minimum; thresholds are lowered with shared atomicMin.
template <class P, int D>
struct Acc {
  double a[D];
};

// Exact merge of one flagged cell (rarely reached): column entry first, then the row candidate.
__device__ __noinline__ void merge_cell(double v, int h, bool rowhit, bool colhit, int row, int j,
                                        int* ct, BestEntry* best, unsigned long long* rv, int* rj,
                                        unsigned long long* stats) {
  // clamp the comparison value at 0 (std::max(0.0, .), aamp.hpp:41; 1 - corr >= 0)
  const unsigned long long vb = (h < 0) ? 0ull : static_cast<unsigned long long>(__double_as_longlong(v));
  if (colhit) {
    atomicMin(ct, static_cast<int>(offer(best, j, vb, row) >> 32));
    if (stats) atomicAdd(&stats[1], 1ull);
  }
  if (rowhit && lex_less(vb, j, *rv, *rj)) {
    *rv = vb;
    *rj = j;
  }
}

// The replay of one block (D sub-steps x D diagonals of one lane), fully unrolled. The 2D-1
// column operands of the block are two aligned runs of D in the ring (c1 = X0+s+xb, c2 = +D) and
// the thresholds two aligned runs in the stage buffer; cell (u, d) uses run entry u + d.
template <class P, int D, bool GUARD>
__device__ __noinline__ void replay_block(Acc<P, D> acc, int s, int cnt, int i0, int kt, int kend,
                                          int L, double p, const double2* cA1, const double2* cA2,
                                          const double* cB1, const double* cB2, int* cT1,
                                          int* cT2, const double2* rowA, const double* rowB,
                                          int* rowT, BestEntry* best, unsigned long long* stats) {
  if (stats) atomicAdd(&stats[0], 1ull);
#pragma unroll
  for (int u = 0; u < D; ++u) {
    if (GUARD && s + u >= cnt) break;
    const int x = s + u;
    const double2 r = rowA[x];
    const double rb = P::kHasB ? rowB[x] : 0.0;
    const int row = i0 + x + 1;
    const int tr = *reinterpret_cast<volatile int*>(&rowT[x]);
    unsigned long long rv = kInfBits;
    int rj = INT_MAX;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int e = u + d;  // entry of the block's column run
      const double2 c = e < D ? cA1[e] : cA2[e - D];
      acc.a[d] = P::step(acc.a[d], r, c, p);
      const double v = P::score(acc.a[d], rb, P::kHasB ? (e < D ? cB1[e] : cB2[e - D]) : 0.0);
      if (GUARD && !((kt + d < kend) && (row + kt + d <= L - 1))) continue;
      const int h = __double2hiint(v);
      int* ct = e < D ? &cT1[e] : &cT2[e - D];
      const bool rowhit = h <= tr;
      const bool colhit = h <= *reinterpret_cast<volatile int*>(ct);
      if (rowhit || colhit) merge_cell(v, h, rowhit, colhit, row, row + kt + d, ct, best, &rv, &rj, stats);
    }
    if (rj != INT_MAX) {
      atomicMin(&rowT[x], static_cast<int>(offer(best, row, rv, rj) >> 32));
      if (stats) atomicAdd(&stats[1], 1ull);
    }
  }
}

// Merge of the seed cells (every valid cell, all lanes on the same row): columns per cell, the
// row through a warp lexicographic reduction and one CAS per warp. Called convergently.
template <int D>
__device__ __noinline__ void resolve_seed(Cells<D> c, unsigned valid, int row, int col0,
                                          BestEntry* best) {
  unsigned long long rv = kInfBits;
  int rj = INT_MAX;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (!((valid >> d) & 1u)) continue;
    const double v = c.v[d];
    const unsigned long long vb = (__double2hiint(v) < 0) ? 0ull : static_cast<unsigned long long>(__double_as_longlong(v));
    const int j = col0 + d;
    offer(best, j, vb, row);
    if (lex_less(vb, j, rv, rj)) {
      rv = vb;
      rj = j;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long ov = __shfl_xor_sync(0xffffffffu, rv, off);
    const int oj = __shfl_xor_sync(0xffffffffu, rj, off);
    if (lex_less(ov, oj, rv, rj)) {
      rv = ov;
      rj = oj;
    }
  }
  if ((threadIdx.x & 31) == 0 && rj != INT_MAX) offer(best, row, rv, rj);
}

// ---------------------------------------------------------------------------------------------
// One stage of S (or cnt < S) row transitions i -> i+1, i in [i0, i0+cnt).
// Filter: per block of D sub-steps a thread touches D rows and 2D-1 columns; theta = max of
// their thresholds (three shared loads per block, precomputed block maxima). A cell can only
// improve (or tie) its row or column minimum if its high word is <= theta. The hot loop only
// keeps the running minimum high word of the block (a VIMNMX3 tree, no branch); a block that
// passes is replayed exactly by `replay_block`.

template <class P, int D, int T, int S, bool GUARD>
__device__ __forceinline__ void run_stage(SweepSmem<P::kHasB, D, T, S>& sm, int b, int X0,
                                          double (&acc)[D], int i0, int cnt, int kt, int kend,
                                          int L, BestEntry* best, double p,
                                          unsigned long long* stats) {
  using G = Geo<D, T, S>;
  // z-norm filter form: 0 = covariance only vs a block bound (2 DFMA per cell; loose when the
  // window scales B vary inside a block, e.g. short windows); 1 = cov * B_j per cell vs a per-row
  // bound (2 DFMA + 1 DMUL per cell; tight up to the block's max threshold).
  constexpr bool kColScale = P::kColScale;
  const int xb = threadIdx.x * D;
  double2 cA[D];
  double cB[D];
  {
    const int q0 = G::pad((X0 + xb) % G::RING);  // X0 + xb is a multiple of D: no wrap inside
#pragma unroll
    for (int d = 0; d < D; ++d) {
      cA[d] = sm.colA[q0 + d];
      if constexpr (kColScale) cB[d] = sm.colB[q0 + d];
    }
  }
  const double2* rowA = sm.rowA[b];
  for (int s = 0; s < cnt; s += D) {
    // the D operands entering during this block are contiguous in the ring: constant offsets
    const int qn = G::pad((X0 + s + xb + D) % G::RING);
    const double2* nA = &sm.colA[qn];
    const double* nB = &sm.colB[P::kHasB ? qn : 0];
    const int cb = s / D + threadIdx.x;
    const int tmax = max(sm.rowBM[b][s / D], max(sm.colBM[b][cb], sm.colBM[b][cb + 1]));
    int theta = tmax;
    double num = 0.0;  // kColScale: 1 - tau_max (with margin), 0 = every cell may qualify
    if constexpr (P::kCovFilter) {
      if (tmax >= 0x3FF00000) {
        theta = INT_MAX;  // some threshold >= 1: any cell may qualify
      } else {
        num = (1.0 - __hiloint2double(tmax, -1)) * (1.0 - 0x1p-40);  // margin for roundings
        if constexpr (!kColScale) {
          const int cq = (X0 / D + cb) % (G::RING / D);
          const float ic = fminf(sm.colIB[cq], sm.colIB[cq + 1 == G::RING / D ? 0 : cq + 1]);
          const double th = num * static_cast<double>(sm.rowIB[b][s / D]) * static_cast<double>(ic);
          theta = ~__double2hiint(th);
        }
      }
    }
    Acc<P, D> acc0;
#pragma unroll
    for (int d = 0; d < D; ++d) acc0.a[d] = acc[d];
    int hmin = INT_MAX;
    bool hit = false;
#pragma unroll
    for (int u = 0; u < D; ++u) {
      if (GUARD && s + u >= cnt) break;
      const int x = s + u;
      const double2 r = rowA[x];
      const int row = i0 + x + 1;
      int hu = INT_MAX;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int sl = (d + u) % D;
        acc[d] = P::step(acc[d], r, cA[sl], p);
        int h;
        if constexpr (kColScale) h = ~__double2hiint(acc[d] * cB[sl]);
        else h = P::key(acc[d]);
        if (GUARD && !((kt + d < kend) && (row + kt + d <= L - 1))) h = INT_MAX;
        hu = min(hu, h);
      }
      if constexpr (kColScale) {
        // row bound for this sub-step: cov * B_j >= (1 - tau) / B_i
        const int tu = (num == 0.0) ? INT_MAX
                                    : ~__double2hiint(num * static_cast<double>(sm.rowIBx[b][x]));
        hit |= hu <= tu;
      } else {
        hmin = min(hmin, hu);
      }
      // slide the column ring: slot u (used by d = 0 this substep) takes the next operand
      cA[u] = nA[u];
      if constexpr (kColScale) cB[u] = nB[u];
    }
    if constexpr (!kColScale) hit = hmin <= theta;
    if (hit) {
      const int q1 = G::pad((X0 + s + xb) % G::RING);
      const int q2 = G::pad((X0 + s + xb + D) % G::RING);
      int* colT = sm.colT[b];
      replay_block<P, D, GUARD>(acc0, s, cnt, i0, kt, kend, L, p, &sm.colA[q1], &sm.colA[q2],
                                &sm.colB[P::kHasB ? q1 : 0], &sm.colB[P::kHasB ? q2 : 0],
                                &colT[G::pad(s + xb)], &colT[G::pad(s + xb + D)], rowA,
                                sm.rowB[b], sm.rowT[b], best, stats);
    }
  }
}

// Block maxima of the freshly loaded thresholds (after the stage's cp.async completed).
template <bool HASB, int D, int T, int S>
__device__ __forceinline__ void stage_block_max(SweepSmem<HASB, D, T, S>& sm, int b, int X0) {
  using G = Geo<D, T, S>;
  using SM = SweepSmem<HASB, D, T, S>;
  for (int blk = threadIdx.x; blk < SM::NCB; blk += T) {
    int mx = INT_MIN;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int x = blk * D + d;
      if (x < G::NCOL) mx = max(mx, sm.colT[b][G::pad(x)]);
    }
    sm.colBM[b][blk] = mx;
  }
  for (int blk = threadIdx.x; blk < S / D; blk += T) {
    int mx = INT_MIN;
#pragma unroll
    for (int d = 0; d < D; ++d) mx = max(mx, sm.rowT[b][blk * D + d]);
    sm.rowBM[b][blk] = mx;
  }
  if constexpr (HASB) {
    // B >= 0: the maximum high word bounds max B from above (low word all ones); its float,
    // rounded up, and the reciprocal rounded down give a lower bound of 1 / max B.
    auto inv_bound = [](int hmax) -> float {
      return __frcp_rd(__double2float_ru(__hiloint2double(hmax, -1)));
    };
    const int first = (X0 == 0) ? 0 : (X0 + G::K) / D;  // column blocks that arrived for this stage
    const int last = (X0 + G::NCOL) / D;
    for (int bx = first + static_cast<int>(threadIdx.x); bx < last; bx += T) {
      const int q = G::pad((bx * D) % G::RING);
      const int* w = reinterpret_cast<const int*>(&sm.colB[q]);
      int hmax = 0;
#pragma unroll
      for (int d = 0; d < D; ++d) hmax = max(hmax, w[2 * d + 1]);
      sm.colIB[bx % (G::RING / D)] = inv_bound(hmax);
    }
    for (int x = threadIdx.x; x < S; x += T)
      sm.rowIBx[b][x] = inv_bound(reinterpret_cast<const int*>(&sm.rowB[b][x])[1]);
    for (int blk = threadIdx.x; blk < S / D; blk += T) {
      const int* w = reinterpret_cast<const int*>(&sm.rowB[b][blk * D]);
      int hmax = 0;
#pragma unroll
      for (int d = 0; d < D; ++d) hmax = max(hmax, w[2 * d + 1]);
      sm.rowIB[b][blk] = inv_bound(hmax);
    }
  }
}

// Issue the cp.async copies of stage st (row transitions i0 .. i0+S-1, i0 = ra + st*S):
// its row operands and thresholds, the thresholds of its whole live column window, and the
// column operands that enter the ring with it (all NCOL for stage 0, S afterwards).
template <bool HASB, int D, int T, int S>
__device__ __forceinline__ void load_stage(SweepSmem<HASB, D, T, S>& sm, const SweepParams& prm,
                                           int st, int ra, int kb) {
  using G = Geo<D, T, S>;
  const int L = prm.L;
  const int b = st & 1;
  const int i0 = ra + st * S;
  const int* bestw = reinterpret_cast<const int*>(prm.best);  // word view; hi word at +1
  for (int x = threadIdx.x; x < G::NCOL; x += T) {
    const int pb = i0 + kb + 1 + x;
    const bool vb = pb < L;
    cp_async(&sm.colT[b][G::pad(x)], bestw + 4 * (vb ? pb : 0) + 1, vb ? 4 : 0, 4);
  }
  const int Xlo = st == 0 ? 0 : st * S + G::K;
  const int Xhi = st * S + G::NCOL;
  for (int X = Xlo + threadIdx.x; X < Xhi; X += T) {
    const int pa = ra + kb + X;
    const bool va = pa < L - 1, vb = pa + 1 < L;
    const int q = G::pad(X % G::RING);
    cp_async(&sm.colA[q], prm.A + (va ? pa : 0), va ? 16 : 0, 16);
    if constexpr (HASB) cp_async(&sm.colB[q], prm.B + (vb ? pa + 1 : 0), vb ? 8 : 0, 8);
  }
  for (int x = threadIdx.x; x < S; x += T) {
    const int pa = i0 + x;
    const int pb = pa + 1;
    const bool va = pa < L - 1, vb = pb < L;
    cp_async(&sm.rowA[b][x], prm.A + (va ? pa : 0), va ? 16 : 0, 16);
    if constexpr (HASB) cp_async(&sm.rowB[b][x], prm.B + (vb ? pb : 0), vb ? 8 : 0, 8);
    cp_async(&sm.rowT[b][x], bestw + 4 * (vb ? pb : 0) + 1, vb ? 4 : 0, 4);
  }
}

// ---------------------------------------------------------------------------------------------
// The sweep kernel: one CTA per tile (kb, ra).

template <class P, int D, int T, int S, int MINB>
__global__ void __launch_bounds__(T, MINB) sweep_kernel(const SweepParams prm) {
  using G = Geo<D, T, S>;
  using SM = SweepSmem<P::kHasB, D, T, S>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);

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
    static_assert(sizeof(SM) >= sizeof(double) * (SL + G::pad(G::K + SL)), "seed scratch");
    double* srow = reinterpret_cast<double*>(smem_raw);
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
      valid |= (ok ? 1u : 0u) << d;
    }
    resolve_seed<D>(c, valid, ra, ra + kt, prm.best);
  }

  // ---- stage pipeline over the row transitions ra .. re-2 ---------------------------------
  const int steps = re - 1 - ra;
  if (steps <= 0) return;
  __syncthreads();  // seed scratch reuse
  load_stage<P::kHasB, D, T, S>(sm, prm, 0, ra, kb);
  cp_async_commit();
  for (int st = 0, s0 = 0; s0 < steps; s0 += S, ++st) {
    const int cnt = min(S, steps - s0);
    const int i0 = ra + s0;
    if (s0 + S < steps) load_stage<P::kHasB, D, T, S>(sm, prm, st + 1, ra, kb);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    stage_block_max<P::kHasB, D, T, S>(sm, st & 1, s0);
    __syncthreads();
    const bool full = (cnt == S) && (kb + G::K <= prm.k_hi) && (i0 + cnt + kb + G::K - 1 <= L - 1);
    if (full) {
      run_stage<P, D, T, S, false>(sm, st & 1, s0, acc, i0, cnt, kt, kend, L, prm.best, prm.p, prm.stats);
    } else {
      run_stage<P, D, T, S, true>(sm, st & 1, s0, acc, i0, cnt, kt, kend, L, prm.best, prm.p, prm.stats);
    }
    __syncthreads();  // stage st's buffers (rows, thresholds, ring slots) are free for st+2
  }
}

}  // namespace mpg
