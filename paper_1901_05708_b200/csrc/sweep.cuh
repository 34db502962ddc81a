// sweep.cuh — sm_100a diagonal-sweep kernels for AAMP / p-norm AAMP / ACAMP.
//
// Reference hot loop being replaced: the per-diagonal functors EuclidScan / PnormScan /
// ZnormScan (/root/reference/proj/src/diag_scan.cpp:7-85) driven by scan_diagonals
// (/root/reference/proj/src/detail/diag_scan.hpp:193-259), with MinBuffer's lexicographic
// (value, index) minimum (diag_scan.hpp:31-53).
//
// B200 design (DESIGN.md §3 has the derivation and the measurements):
//  * A CTA owns a TILE = K = T*D consecutive diagonals x R consecutive rows. Thread `tid` owns
//    D consecutive diagonals and walks the rows; each tile is seeded with one direct length-m
//    sum per diagonal (the reference's refresh rule, diag_scan.hpp:93-105, is exactly "seed at
//    multiples of R"), then every cell costs the O(1) slide: 3 FP64-pipe instructions for AAMP
//    ((delta, sigma) form), 2 or 3 for ACAMP (centred covariance, covariance filter).
//  * Column operands stream through a shared-memory RING (cp.async), one new operand per thread
//    per row into a register ring of D slots with compile-time rotation; row operands are warp
//    broadcasts; padding x -> x + x/D keeps the stride-D lane pattern bank-conflict free.
//  * Minima: the exact global profile is an array of 16-byte (value bits, index) entries merged
//    with a 128-bit atomicCAS lexicographic minimum (MinBuffer::update semantics). The hot loop
//    never touches it: per block of D sub-steps it keeps the minimum 32-bit key of its cells
//    and compares it once with the block's maximum threshold; a passing block is replayed
//    bit-identically through the exact slow path.
//  * FP32 mode: the same machinery with float accumulators/operands (policies *F32); values are
//    promoted exactly to double for the merge, and finalize recomputes the reported distance of
//    the chosen pair in FP64.
#pragma once

#include <cstdint>
#include <climits>
#include <type_traits>
#include <cuda_runtime.h>

namespace mpg {

// Device-side bounds checks (MPROF_CHECKS=1 builds only; compute-sanitizer is not available on
// this pool): every shared-memory ring / table index and every profile position a kernel touches
// is checked and a violation traps (the launch fails with an illegal-instruction error).
#ifndef MPROF_CHECKS
#define MPROF_CHECKS 0
#endif
constexpr int kStageRowsMax = 512;  // largest rows-per-stage of any policy (checks only)
#if MPROF_CHECKS
#define MPG_CHECK(cond) \
  do {                  \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define MPG_CHECK(cond) \
  do {                  \
  } while (0)
#endif

// Rows of a replayed block unrolled per iteration (replay_block; 1 = rolled, 8 = fully unrolled;
// 0 = by policy: unrolled for the covariance-only filters, whose replays the form probe keeps rare,
// rolled otherwise -- see replay_block).
#ifndef MPROF_REPLAY_UNROLL
#define MPROF_REPLAY_UNROLL 0
#endif

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
// 128-bit CAS loop. The initial 16-byte read is not guaranteed single-copy atomic as a whole
// (each aligned 8-byte word is): it may pair a value with the index of an older or newer entry.
// Entries only decrease, so a read value word above v, or below it, decides the offer on its own
// (below: no improvement; above: the CAS decides); only an exact value tie depends on the index,
// and a torn read there (the new value with the old, smaller index) could drop a valid offer, so
// a tie verdict of "no improvement" is confirmed by an atomic snapshot (a CAS that writes back
// what it compares with).
__device__ __forceinline__ unsigned long long offer(BestEntry* best, long long pos,
                                                    unsigned long long v, long long idx) {
  MPG_CHECK(pos >= 0 && idx >= -1);
  const longlong2 raw = __ldcg(reinterpret_cast<const longlong2*>(best + pos));
  BestEntry cur{static_cast<unsigned long long>(raw.x), raw.y};
  bool atomic_read = false;  // cur was returned by a CAS (an atomic read of the entry)
  for (;;) {
    if (lex_less(v, idx, cur.v, cur.idx)) {
      const BestEntry old = atomicCAS(best + pos, cur, BestEntry{v, idx});
      if (old.v == cur.v && old.idx == cur.idx) return v;
      cur = old;
    } else {
      if (atomic_read || cur.v != v) return cur.v;
      const BestEntry snap = atomicCAS(best + pos, cur, cur);
      if (snap.v == cur.v && snap.idx == cur.idx) return cur.v;
      cur = snap;
    }
    atomic_read = true;
  }
}

// ---------------------------------------------------------------------------------------------
// Distance families ("policies"). A[p] is the per-position operand pair, B[p] an optional
// per-position scalar (the z-normalization scale). step() slides the diagonal accumulator from
// cell (i, j) to (i+1, j+1) using A[i] (row) and A[j] (column); score() maps the accumulator of
// the new cell to the comparison value using B[i+1], B[j+1]; key() is the 32-bit fast-filter
// key (smaller = better). Seeds are direct length-m sums, always in FP64.

// Operand layouts of A[p] (built by the host, see k_build_pairs / k_znorm_pairs):
enum PairKind { kPairsRaw = 0, kPairsDeltaSum = 1, kPairsZnorm = 2 };

// Threshold words are high words of FP64 comparison values. FP64 keys compare with them
// directly; FP32 keys are float bits, so a threshold is converted to the float bound rounded UP
// (a looser filter is always safe: the replay decides exactly).
struct KeyF64 {
  __device__ __forceinline__ static int key(double v) { return __double2hiint(v); }
  __device__ __forceinline__ static int tau(int hi) { return hi; }
  // covariance-filter key and bound (larger covariance = better): ~hi is decreasing
  __device__ __forceinline__ static int cov_key(double c) { return ~__double2hiint(c); }
  __device__ __forceinline__ static int cov_bound(double th) { return ~__double2hiint(th); }
  // covariance-only form in raw (order-preserving) words: hit <=> max raw(cov) >= raw bound
  __device__ __forceinline__ static int cov_raw(double c) { return __double2hiint(c); }
  __device__ __forceinline__ static int cov_bound_raw_f(float th) {  // th > 0, exact in double
    return __double2hiint(static_cast<double>(th));
  }
};
struct KeyF32 {
  __device__ __forceinline__ static int key(float v) { return __float_as_int(v); }
  __device__ __forceinline__ static int tau(int hi) {
    if (hi >= 0x47EFFFFF) return INT_MAX;  // at or beyond FLT_MAX (incl. +inf): pass everything
    return __float_as_int(__double2float_ru(__hiloint2double(hi, -1)));
  }
  __device__ __forceinline__ static int cov_key(float c) { return ~__float_as_int(c); }
  __device__ __forceinline__ static int cov_bound(double th) {
    return ~__float_as_int(__double2float_rd(th));
  }
  __device__ __forceinline__ static int cov_raw(float c) { return __float_as_int(c); }
  __device__ __forceinline__ static int cov_bound_raw_f(float th) { return __float_as_int(th); }
};

// AAMP. Reference: incremental_euclidean_step (/root/reference/proj/include/mprof/aamp.hpp:37-42),
// direct_sq_acc (/root/reference/proj/src/detail/diag_scan.hpp:57-64).
// fast mode: A[p] = (delta_p, sigma_p) = (t[p+m] - t[p], t[p+m] + t[p]) and
//   in^2 - out^2 = (a' - b')^2 - (a - b)^2 = (delta_i - delta_j)(sigma_i - sigma_j),
// one DFMA + two DADD per cell instead of two DFMA + two DADD.
// exact mode: A[p] = (t[p], t[p+m]) and the reference's evaluation order.
template <bool EXACT>
struct Euclid : KeyF64 {
  using Base = Euclid;  // FP64 policy used by the first-diagonal pre-pass
  using V = double;
  using V2 = double2;
  using VB = double;
  #ifndef MPROF_STAGE_WIDE
#define MPROF_STAGE_WIDE 256
#endif
  // 256-row stages: C4 -1.2 % (AAMP keeps 4 CTAs/SM). Tried for the covariance-only z-norm
  // kernel too: C4 -1.2 % but C5 +2 % (its larger shared memory drops it to 3 CTAs/SM).
  static constexpr int kStageRows = EXACT ? 128 : MPROF_STAGE_WIDE;
  static constexpr bool kHasB = false;
  static constexpr bool kCenteredSeed = false;
  static constexpr bool kCovFilter = false;
  static constexpr bool kColScale = false;
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
  else return pow(a, p);  // generic and half-integer p: std::pow, as the reference
}

// sqrt(a), a >= 0, for the half-integer p-norm path. MPROF_HALF_SQRT = 2 (default): the MUFU
// double rsqrt seed (rsqrt.approx.f64) + two Newton steps in FP64, worst relative error 3.9e-16
// over 1e-130..1e130 for normal inputs (tools/sqrt_check; C3 p = 2.5: 71 ms); 3: one Newton step
// (1.2e-12, 54 ms);
// 1: a * rsqrt(a) (CUDA's double rsqrt, 123 ms); 0: IEEE sqrt (135 ms).
#ifndef MPROF_HALF_SQRT
#define MPROF_HALF_SQRT 2
#endif
__device__ __forceinline__ double sqrt_fast(double a) {
  if constexpr (MPROF_HALF_SQRT == 1) {
    return a > 0.0 ? a * rsqrt(a) : 0.0;
  } else if constexpr (MPROF_HALF_SQRT == 2 || MPROF_HALF_SQRT == 3) {
    // MUFU.RSQ64H seed (PTX rsqrt.approx.f64, full double range) + Newton steps in FP64
    // a must be normal (the seed flushes denormals to 0): pow_fast clamps its argument
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    const double h = 0.5 * a;
    y = y * fma(-h * y, y, 1.5);
    if constexpr (MPROF_HALF_SQRT == 2) y = y * fma(-h * y, y, 1.5);
    return a * y;
  } else {
    return sqrt(a);
  }
}

// a^p (a >= 0) in the fast mode. PK = 1, 3, 4: exact products; PK = -k: the half-integer
// p = k / 2 (k odd) as a^((k-1)/2) sqrt(a) (~10 FP64-pipe instructions instead of pow's ~100;
// C3 p = 2.5: 746 -> 135 ms); PK = 0, any other p: pow (exp2(p log2 a) with CUDA's double
// exp2 / log2 measured slower: C3 p = 2.7 746 -> 1286 ms).
template <int PK>
__device__ __forceinline__ double pow_fast(double a, double p) {
  if constexpr (PK == 1) return a;
  else if constexpr (PK == 3) return a * a * a;
  else if constexpr (PK == 4) { const double a2 = a * a; return a2 * a2; }
  else if constexpr (PK < 0) {
    constexpr int h = (-PK - 1) / 2;  // integer part of p, >= 1 (p >= 1)
    static_assert(h >= 1, "half-integer p >= 1.5");
    // sqrt of max(a, DBL_MIN) (integer ops on the high word): for a < DBL_MIN the product
    // a^h sqrt(.) underflows to 0 either way, so the clamp changes no result and keeps the hot
    // path branch-free (a branch to an IEEE fallback measured 103 ms instead of 71 on C3 p = 2.5)
    const int hi = __double2hiint(a);
    const bool tiny = hi < 0x00100000;
    const double an = __hiloint2double(tiny ? 0x00100000 : hi, tiny ? 0 : __double2loint(a));
    const double r = sqrt_fast(an);
    if constexpr (h == 1) return a * r;
    else if constexpr (h == 2) return (a * a) * r;
    else return (a * a) * (a * r);
  } else {
    return pow(a, p);
  }
}

// p-norm AAMP: accumulator sum |t_i - t_j|^p. PK = 1, 3, 4 integer fast paths, PK = -3, -5, -7 the
// half-integers p = 1.5, 2.5, 3.5 (fast mode; the exact mode evaluates them with pow like the
// reference), 0 = generic p. Reference: incremental_pnorm_step (aamp.hpp:45-49), direct_pnorm_acc
// (diag_scan.hpp:66-71).
template <int PK, bool EXACT>
struct Pnorm : KeyF64 {
  using Base = Pnorm;
  using V = double;
  using V2 = double2;
  using VB = double;
  static constexpr bool kHasB = false;
  static constexpr bool kCenteredSeed = false;
  static constexpr bool kCovFilter = false;
  static constexpr bool kColScale = false;
  static constexpr int kPairs = kPairsRaw;
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
        return (acc - pow_fast<PK>(fabs(out), p)) + pow_fast<PK>(fabs(in), p);
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
      else return acc + pow_fast<PK>(d, p);
    }
  }
};

// ACAMP: the accumulator is the CENTRED covariance cov(i,j) = sum (t_i - mu_i)(t_j - mu_j),
// slid as cov += df_i*dg_j + df_j*dg_i with df_p = (t[p+m]-t[p])/2,
// dg_p = (t[p+m]-mu_{p+1}) + (t[p]-mu_p)  (A[p] = (df_p, dg_p)), and B[p] = 1/||t_p - mu_p||
// (0 for flat windows). Comparison value d = 1 - corr = 1 - cov*B[i]*B[j], DZ^2 = 2m*d.
// This replaces the reference's five uncentred running sums (advance_stats + f_value,
// /root/reference/proj/include/mprof/acamp.hpp:28-60): same profile, no divide, and no
// cancellation against the window level.
// Fast filter (run_stage): for a cell that can reach a threshold tau < 1,
// cov * B_i * B_j >= 1 - tau, so the hot loop tests cov alone against a block bound
// (COLSCALE = 0: 2 DFMA per cell) or cov * B_j against a per-row bound (COLSCALE = 1:
// + 1 DMUL per cell, tight when the window scales vary, e.g. short windows).
template <bool COLSCALE>
// Stage rows of the covariance-only kernels (measured, sweep ms, 128 -> 256 rows): EuclidCov C4
// 118.4 -> 115.7, random walk n = 2^18, m = 256 8.10 -> 8.06; Znorm C4 116.6 -> 116.2 but C5
// 2055 -> 2130 and a random walk n = 2^20, m = 512 129.1 -> 133.4, so only EuclidCov uses 256.
#ifndef MPROF_STAGE_COV
#define MPROF_STAGE_COV 128
#endif
#ifndef MPROF_STAGE_ECOV
#define MPROF_STAGE_ECOV 256
#endif
struct Znorm : KeyF64 {
  using Base = Znorm;
  using V = double;
  using V2 = double2;
  using VB = double;
  static constexpr int kStageRows = COLSCALE ? 128 : MPROF_STAGE_COV;
  static constexpr bool kHasB = true;
  static constexpr bool kCenteredSeed = true;
  static constexpr bool kCovFilter = true;
  static constexpr bool kColScale = COLSCALE;
#ifndef MPROF_ZN_COV_WARPS
#define MPROF_ZN_COV_WARPS 16
#endif
  // per SM; measured: the +cB ring wants registers
  static constexpr int kMinWarps = COLSCALE ? 12 : MPROF_ZN_COV_WARPS;
  static constexpr int kPairs = kPairsZnorm;
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

// AAMP in covariance form (fast FP64 mode, long windows): the accumulator is the CENTRED
// covariance slid exactly as Znorm does (A2[p] = (df_p, dg_p), 2 DFMA per cell), and
//   D^2(i, j) = S_i + S_j + m (mu_i - mu_j)^2 - 2 cov(i, j),   S_p = ||t_p - mu_p||^2
// (the well-conditioned split of ||x - y||^2 into centred parts and means). The hot loop keeps
// only cov: a cell can reach a threshold tau only if 2 cov >= S_i + S_j + m (mu_i - mu_j)^2 - tau,
// bounded per block from per-stage tables of min S, the mean range and max tau of its rows and
// column pair (SB[p] = {S_p rounded down, mu_p - t[0] rounded down} as float2 in the rings).
// Exact comparison values (replays, seed cells) use the FP64 S and mu from global memory. The
// diagonal block next to the exclusion zone runs the (delta, sigma) kernel (Base) instead: there
// the neighbours are within the block bound's slack. Replaces EuclidScan's slide
// (/root/reference/proj/src/diag_scan.cpp:7-24, incremental_euclidean_step aamp.hpp:37-42).
struct EuclidCov : KeyF64 {
  static constexpr int kStageRows = MPROF_STAGE_ECOV;
  using Base = Euclid<false>;
  using V = double;
  using V2 = double2;
  using VB = float2;
  static constexpr bool kHasB = true;
  static constexpr bool kCenteredSeed = true;
  static constexpr bool kCovFilter = true;
  static constexpr bool kColScale = false;
  static constexpr bool kEuclidCov = true;
  static constexpr bool kPairsAlt = true;  // operands in SweepParams::A2
  static constexpr int kMinWarps = 16;
  static constexpr int kPairs = kPairsZnorm;
  __device__ __forceinline__ static double step(double acc, double2 r, double2 c, double) {
    return fma(r.x, c.y, fma(c.x, r.y, acc));
  }
  // a = t_i - mu_i (row, pre-centred), b = t_j, mub = mu_j
  __device__ __forceinline__ static double seed(double acc, double a, double b, double mub,
                                                double) {
    return fma(a, b - mub, acc);
  }
  __device__ __forceinline__ static double value(double cov, double si, double sj, double mi,
                                                 double mj, double md) {
    const double dm = mi - mj;
    return fma(md * dm, dm, si + sj) - 2.0 * cov;
  }
};

// A covariance-only policy with longer hit groups, selected per series by the form probe when
// its sample saw (almost) no replays: a group of HG_WIDE blocks per data-dependent branch (the
// replay of a passing group costs more, so replay-heavy series keep the policy's own HG).
// (measured with the probe gating, sweep ms HG 4 -> 8 -> 16: C4 AAMP 112.9 -> 109.9 -> 140.5,
// C4 ACAMP 114.5 -> 112.3 -> 129.0; 16 spills)
#ifndef MPROF_HIT_GROUP_WIDE
#define MPROF_HIT_GROUP_WIDE 8
#endif
template <class P>
struct Wide : P {
  static constexpr int kHitGroup = MPROF_HIT_GROUP_WIDE;
};

// Dense<P>: the same slide without the block filter -- every cell is compared exactly with its
// row and column thresholds as it is computed, and candidates are reduced per CTA in shared
// memory (exact 128-bit lexicographic minima) and offered to the global profile once per stage.
// Chosen per series for noise-like data, where the filter passes (and replays) nearly every block
// (plan_series' noise test).
template <class P>
struct Dense : P {
  static constexpr bool kDense = true;
  static constexpr int kHitGroup = 1;
};

template <class P>
constexpr bool is_dense() {
  if constexpr (requires { P::kDense; }) return P::kDense;
  else return false;
}

template <class P>
constexpr int hit_group_of() {
  if constexpr (requires { P::kHitGroup; }) return P::kHitGroup;
  else return 0;
}

template <class P>
constexpr bool is_euclid_cov() {
  if constexpr (requires { P::kEuclidCov; }) return P::kEuclidCov;
  else return false;
}

// Exact per-cell inputs of comparison values that are not kept in the rings (EuclidCov): in
// static shared memory, written once per CTA, so the hot loop keeps no registers for them.
struct CellCtx {
  const double* S;
  const double* mu;
  double md;
};
__shared__ CellCtx g_cell_ctx;

// Comparison value of cell (i, j) from its accumulator.
template <class P>
__device__ __forceinline__ double cell_value(typename P::V acc, typename P::VB rb,
                                             typename P::VB cb, int i, int j) {
  if constexpr (is_euclid_cov<P>()) {
    const CellCtx& cc = g_cell_ctx;
    return P::value(acc, __ldg(cc.S + i), __ldg(cc.S + j), __ldg(cc.mu + i), __ldg(cc.mu + j),
                    cc.md);
  } else {
    return static_cast<double>(P::score(acc, rb, cb));
  }
}

// ---- FP32 mode policies ------------------------------------------------------------------------
// Same slides in float; seeds in FP64 (rounded once to float). Operands are built relative to a
// global offset c (the series mean) so that float keeps the digits that matter: AAMP
// A = (delta, sigma - 2c), p-norm A = (t - c, t[p+m] - c); ACAMP's (df, dg) and B are
// offset-free. Comparison values are promoted exactly to double for the merge.

struct EuclidF32 : KeyF32 {
  using Base = Euclid<false>;
  using V = float;
  using V2 = float2;
  using VB = float;
  static constexpr bool kHasB = false;
  static constexpr bool kCenteredSeed = false;
  static constexpr bool kCovFilter = false;
  static constexpr bool kColScale = false;
  static constexpr int kPairs = kPairsDeltaSum;
  __device__ __forceinline__ static float step(float acc, float2 r, float2 c, double) {
    return fmaf(r.x - c.x, r.y - c.y, acc);
  }
  __device__ __forceinline__ static float score(float acc, float, float) { return acc; }
  __device__ __forceinline__ static double seed(double acc, double a, double b, double, double) {
    const double d = a - b;
    return fma(d, d, acc);
  }
};

template <int PK>
struct PnormF32 : KeyF32 {
  using Base = Pnorm<PK, false>;
  using V = float;
  using V2 = float2;
  using VB = float;
  static constexpr bool kHasB = false;
  static constexpr bool kCenteredSeed = false;
  static constexpr bool kCovFilter = false;
  static constexpr bool kColScale = false;
  static constexpr int kPairs = kPairsRaw;
  __device__ __forceinline__ static float step(float acc, float2 r, float2 c, double p) {
    const float out = fabsf(r.x - c.x);
    const float in = fabsf(r.y - c.y);
    if constexpr (PK == 1) return (acc - out) + in;
    else if constexpr (PK == 3) return fmaf(in * in, in, fmaf(-out * out, out, acc));
    else if constexpr (PK == 4) { const float o2 = out * out, i2 = in * in; return fmaf(i2, i2, fmaf(-o2, o2, acc)); }
    else return (acc - powf(out, static_cast<float>(p))) + powf(in, static_cast<float>(p));
  }
  __device__ __forceinline__ static float score(float acc, float, float) { return acc; }
  __device__ __forceinline__ static double seed(double acc, double a, double b, double, double p) {
    return Pnorm<PK, false>::seed(acc, a, b, 0.0, p);
  }
};

template <bool COLSCALE>
struct ZnormF32 : KeyF32 {
  using Base = Znorm<COLSCALE>;
  using V = float;
  using V2 = float2;
  using VB = float;
  static constexpr bool kHasB = true;
  static constexpr bool kCenteredSeed = true;
  static constexpr bool kCovFilter = true;
  static constexpr bool kColScale = COLSCALE;
  static constexpr int kPairs = kPairsZnorm;
  __device__ __forceinline__ static float step(float acc, float2 r, float2 c, double) {
    return fmaf(r.x, c.y, fmaf(c.x, r.y, acc));
  }
  __device__ __forceinline__ static float score(float acc, float rb, float cb) {
    return fmaf(-(acc * cb), rb, 1.0f);
  }
  __device__ __forceinline__ static double seed(double acc, double a, double b, double mub, double) {
    return fma(a, b - mub, acc);
  }
};

// Name of a sweep policy as reported in mprof_run_info::policy.
template <class P>
constexpr const char* policy_name() {
  if constexpr (std::is_same_v<P, Euclid<false>>) return "Euclid";
  else if constexpr (std::is_same_v<P, Euclid<true>>) return "Euclid<exact>";
  else if constexpr (std::is_same_v<P, EuclidCov>) return "EuclidCov";
  else if constexpr (std::is_same_v<P, Wide<EuclidCov>>) return "Wide<EuclidCov>";
  else if constexpr (std::is_same_v<P, Znorm<false>>) return "Znorm<0>";
  else if constexpr (std::is_same_v<P, Znorm<true>>) return "Znorm<1>";
  else if constexpr (std::is_same_v<P, Wide<Znorm<false>>>) return "Wide<Znorm<0>>";
  else if constexpr (std::is_same_v<P, Pnorm<1, false>>) return "Pnorm<1>";
  else if constexpr (std::is_same_v<P, Pnorm<3, false>>) return "Pnorm<3>";
  else if constexpr (std::is_same_v<P, Pnorm<4, false>>) return "Pnorm<4>";
  else if constexpr (std::is_same_v<P, Pnorm<0, false>>) return "Pnorm<p>";
  else if constexpr (std::is_same_v<P, Pnorm<-3, false>>) return "Pnorm<1.5>";
  else if constexpr (std::is_same_v<P, Pnorm<-5, false>>) return "Pnorm<2.5>";
  else if constexpr (std::is_same_v<P, Pnorm<-7, false>>) return "Pnorm<3.5>";
  else if constexpr (std::is_same_v<P, Pnorm<1, true>>) return "Pnorm<1,exact>";
  else if constexpr (std::is_same_v<P, Pnorm<3, true>>) return "Pnorm<3,exact>";
  else if constexpr (std::is_same_v<P, Pnorm<4, true>>) return "Pnorm<4,exact>";
  else if constexpr (std::is_same_v<P, Pnorm<0, true>>) return "Pnorm<p,exact>";
  else if constexpr (std::is_same_v<P, EuclidF32>) return "EuclidF32";
  else if constexpr (std::is_same_v<P, PnormF32<1>>) return "PnormF32<1>";
  else if constexpr (std::is_same_v<P, PnormF32<3>>) return "PnormF32<3>";
  else if constexpr (std::is_same_v<P, PnormF32<4>>) return "PnormF32<4>";
  else if constexpr (std::is_same_v<P, PnormF32<0>>) return "PnormF32<p>";
  else if constexpr (std::is_same_v<P, ZnormF32<false>>) return "ZnormF32<0>";
  else if constexpr (std::is_same_v<P, ZnormF32<true>>) return "ZnormF32<1>";
  else if constexpr (std::is_same_v<P, Dense<Euclid<false>>>) return "Dense<Euclid>";
  else if constexpr (std::is_same_v<P, Dense<Znorm<true>>>) return "Dense<Znorm<1>>";
  else if constexpr (std::is_same_v<P, Dense<Pnorm<1, false>>>) return "Dense<Pnorm<1>>";
  else if constexpr (std::is_same_v<P, Dense<Pnorm<3, false>>>) return "Dense<Pnorm<3>>";
  else return "?";
}

// ---------------------------------------------------------------------------------------------
// Tile geometry and shared memory.

template <int D, int T, int S>
struct Geo {
  static constexpr int K = T * D;        // diagonals per tile
  static constexpr int NCOL = S + K;     // column operands live during one stage
  static constexpr int RING = K + 2 * S; // ring slots: live stage + the prefetched next stage
  __host__ __device__ static constexpr int pad(int x) { return x + x / D; }
  static constexpr int NCOLP = pad(NCOL - 1) + 1;
  static constexpr int RINGP = pad(RING - 1) + 1;
};

// Sampled keys (experiment switch, off): measured with HG = 2, sweep ms 1 B200, off -> on: C4
// AAMP 118.4 -> 116.3, C4 ACAMP 116.4 -> 113.3, but C5 ACAMP 2056 -> 2175 and a random walk
// n = 2^20, m = 512 ACAMP 129.0 -> 136.8: the one-step margin (m-lag differences x window
// deviations, ~1 % of the covariance scale) is comparable to the 1 - correlation slack of the
// nearest neighbours, so many more blocks pass and replay.
#ifndef MPROF_SAMPLED_KEYS
#define MPROF_SAMPLED_KEYS 0
#endif

// Shared memory of one CTA. Column operands live in a RING indexed by X = (column position -
// tile column base): stage st uses X in [st*S, st*S + S + K) and prefetches only its S new
// operands for stage st+1, so one copy of the K-wide window is resident (not two). Thresholds
// (4 B per column) are re-read for the whole live window every stage (fresh minima from other
// CTAs) and double-buffered with the row operands.
// ROWA = false (the constant-row kernel, whose row operands are kernel parameters) drops the row
// operand buffers.
template <class P, int D, int T, int S, bool ROWA = true>
struct SweepSmem {
  using G = Geo<D, T, S>;
  using V2 = typename P::V2;
  using VB = typename P::VB;
  static constexpr bool HASB = P::kHasB;
  static_assert(G::RING % D == 0 && S % D == 0, "stage and ring must be multiples of D");
  static constexpr int NCB = G::NCOL / D + 1;  // column blocks of D
  V2 colA[G::RINGP];                           // ring: A[cbase + X] at pad(X mod RING)
  VB colB[HASB ? G::RINGP : 2];                // ring: B[cbase + 1 + X]
  int colT[2][G::NCOLP];                       // hi32(best[i0 + kb + 1 + x].v), exact
  // Block tables are single-buffered: they are rebuilt between the two barriers of each stage,
  // when no warp reads them. The covariance forms keep their own tables instead of the max
  // threshold words.
  static constexpr bool EQ = is_euclid_cov<P>();
  static constexpr bool ZQ = P::kCovFilter && !P::kColScale && !EQ;
  static constexpr bool TW = !(ZQ || EQ);     // filters on threshold words (colBM2 / rowBM)
  int colBM2[TW ? NCB : 1];                    // max of colT over columns [cD, cD + 2D)
  V2 rowA[ROWA ? 2 : 1][ROWA ? S : 1];         // A[i0 + x]
  VB rowB[2][HASB ? S : 2];                    // B[i0 + 1 + x]
  int rowT[2][S];                              // hi32(best[i0 + 1 + x].v), exact
  int rowBM[TW ? S / D : 1];                   // max of rowT over aligned blocks of D
  // z-norm filter scales, rounded DOWN (a smaller scale only loosens the filter).
  float rowIBx[P::kColScale ? S : 1];          // <= 1 / rowB of each row (column-scaled form)
  // Covariance-only z-norm filter, per stage: for row block r, {lower bound of (1 - tau_r) *
  // IB_r, IB_r}; for column block c (covering stage columns [cD, cD + 2D)), {lower bound of
  // (1 - tau_c) * IB_c, IB_c}, tau = max threshold, IB <= 1 / max B of the block; -inf = "some
  // threshold >= 1, every cell may pass". A block's covariance bound is then
  // min(RQ_r * IB_c, CQ_c * IB_r) (= (1 - max(tau_r, tau_c)) * IB_r * IB_c).
  float2 zrow[ZQ ? S / D : 1];
  float2 zcol[ZQ ? NCB : 1];
  // Covariance-form AAMP filter, per stage: {min S (down), min mu (down), max mu (up),
  // max tau (up)} of each row block and column block pair.
  float4 erow[EQ ? S / D : 1];
  float4 ecol[EQ ? NCB : 1];
  // Sampled keys (FP64 covariance forms): the hot loop takes the keys of sub-steps 1, 3, 5, 7
  // only. Every other cell of the block is one slide step before a sampled cell, and one step
  // changes a covariance by at most RX*CY + CX*RY, the per-block upper bounds {max |A.x|,
  // max |A.y|} of the row block (drow) and the column block pair (dcol), float rounded up; the
  // block bound is lowered by that amount.
  static constexpr bool SK = (ZQ || EQ) && sizeof(typename P::V) == 8 && MPROF_SAMPLED_KEYS;
  float2 drow[SK ? S / D : 1];
  float2 dcol[SK ? NCB : 1];
  // Dense<P>: the stage's exact candidates of its rows and of its live column window
  static constexpr bool DN = is_dense<P>();
  BestEntry crow[DN ? S : 1];
  BestEntry ccol[DN ? G::NCOL : 1];
};

struct SweepParams {
  const double* t;        // series, n samples
  const double2* A;       // FP64 per-position operand pairs, valid [0, L-1)
  const double* B;        // FP64 per-position scale (z-norm), valid [0, L)
  const float2* A32;      // FP32 mode operand pairs
  const float* B32;       // FP32 mode scales
  const double* mu;       // window means (z-norm, covariance-form AAMP), valid [0, L)
  const double2* A2;      // covariance-form AAMP operand pairs (df, dg), valid [0, L-1)
  const float2* SB;       // covariance-form AAMP ring scalars {S rd, mu - t[0] rd}, valid [0, L)
  const double* S;        // covariance-form AAMP centred sums of squares, valid [0, L)
  BestEntry* best;        // L entries
  const int4* tiles;      // (first diagonal kb, first row ra, row end re, -) per CTA
  int n, m, L;
  int k_hi;               // exclusive upper bound of the swept diagonal band
  int R;                  // rows per tile
  int row_hi;             // exclusive upper bound of the swept rows (L for a full sweep)
  double p;
  unsigned long long* stats;  // optional diagnostics (MPROF_STATS): [0] replays [1] offers
  double* scratch;            // L doubles of scratch (first-diagonal pass)
};


template <class P>
__device__ __forceinline__ const typename P::V2* pairs_of(const SweepParams& prm) {
  if constexpr (is_euclid_cov<P>()) return prm.A2;
  else if constexpr (sizeof(typename P::V) == 8) return prm.A;
  else return prm.A32;
}
template <class P>
__device__ __forceinline__ const typename P::VB* scales_of(const SweepParams& prm) {
  if constexpr (is_euclid_cov<P>()) return prm.SB;
  else if constexpr (sizeof(typename P::V) == 8) return prm.B;
  else return prm.B32;
}

// ---------------------------------------------------------------------------------------------
// cp.async helpers (LDGSTS). An invalid source zero-fills the destination.

template <int SIZE>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src = valid ? SIZE : 0;
  if constexpr (SIZE == 16) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  } else if constexpr (SIZE == 8) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------------------------
// Exact slow path.

template <int D>
struct Cells {
  double v[D];
};

template <class P, int D>
struct Acc {
  typename P::V a[D];
};

// Exact merge of one flagged cell (rarely reached): column entry first, then the row candidate.
// Positions (row, j) index the profile being swept; the stored neighbour indices are mapped by
// out_index (identity except for reflected sweeps) so ties compare in original coordinates.
static __device__ __noinline__ void merge_cell(double v, int h, bool rowhit, bool colhit, int row, int j,
                                        int* ct, BestEntry* best, unsigned long long* rv,
                                        int* rj, unsigned long long* stats) {
  MPG_CHECK(row >= 0 && j > row);
  // clamp the comparison value at 0 (std::max(0.0, .), aamp.hpp:41; 1 - corr >= 0)
  const unsigned long long vb = (h < 0) ? 0ull : static_cast<unsigned long long>(__double_as_longlong(v));
  if (colhit) {
    atomicMin(ct, static_cast<int>(offer(best, j, vb, row) >> 32));
    if (stats) atomicAdd(&stats[1], 1ull);
  }
  const int jo = j;
  if (rowhit && lex_less(vb, jo, *rv, *rj)) {
    *rv = vb;
    *rj = jo;
  }
}

// The replay of one block (D sub-steps x D diagonals of one lane), fully unrolled, from the
// accumulators saved at the block start: bit-identical recomputation of the fast path, then every
// cell whose (FP64-promoted) value has a high word <= the current exact column (row) threshold
// in shared memory is merged. The 2D-1 column operands of the block are two aligned runs of D in
// the ring (c1 = X0+s+xb, c2 = +D), the thresholds two aligned runs in the stage buffer; cell
// (u, d) uses run entry u + d.
template <class P, int D, bool GUARD>
__device__ __noinline__ Acc<P, D> replay_block(Acc<P, D> acc, int s, int cnt, int i0, int kt, int kend,
                                          int L, double p, const typename P::V2* cA1,
                                          const typename P::V2* cA2, const typename P::VB* cB1,
                                          const typename P::VB* cB2, int* cT1, int* cT2,
                                          const typename P::V2* rowA, const typename P::VB* rowB,
                                          int* rowT, BestEntry* best, unsigned long long* stats) {
  using V2 = typename P::V2;
  using VB = typename P::VB;
  if (stats) atomicAdd(&stats[0], 1ull);
  // Unrolling the row loop pays where replays are rare and clustered (the covariance-only
  // filters, confirmed by the form probe: C5 2101 vs 2317 ms, C4 ACAMP 118.8 vs 123.5 ms), but on
  // series where most blocks replay (noise-like data, loose thresholds everywhere) the unrolled
  // 64-cell body thrashes the instruction cache (ncu: 61 % of stall samples "no instruction";
  // uniform noise n = 2^13, m = 256: 5.7 ms unrolled vs 2.15 ms rolled), so the other filters roll it.
  constexpr bool kCovOnly = P::kCovFilter && !P::kColScale;
  constexpr int kUnroll = MPROF_REPLAY_UNROLL ? MPROF_REPLAY_UNROLL : (kCovOnly ? D : 1);
#pragma unroll kUnroll
  for (int u = 0; u < D; ++u) {
    if (GUARD && s + u >= cnt) break;
    const int x = s + u;
    MPG_CHECK(x >= 0 && x < kStageRowsMax);
    const V2 r = rowA[x];
    const VB rb = P::kHasB ? rowB[x] : VB{};
    const int row = i0 + x + 1;
    const int tr = *reinterpret_cast<volatile int*>(&rowT[x]);
    unsigned long long rv = kInfBits;
    int rj = INT_MAX;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int e = u + d;  // entry of the block's column run
      const V2 c = e < D ? cA1[e] : cA2[e - D];
      acc.a[d] = P::step(acc.a[d], r, c, p);
      if (GUARD && !((kt + d < kend) && (row + kt + d <= L - 1))) continue;
      const double v = cell_value<P>(acc.a[d], rb, P::kHasB ? (e < D ? cB1[e] : cB2[e - D]) : VB{},
                                     row, row + kt + d);
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
  return acc;  // the block's end accumulators (start of the next block of a replayed group)
}

// Warp-cooperative replay of lane `src`'s hit group: lane q < D takes diagonal q of src's
// blocks (accumulator `a` = src's acc0.a[q]), so a group replays in D sub-steps per block instead
// of D*D cells on one lane while the other 31 lanes wait. Per sub-step every active lane
// evaluates its cell exactly as replay_block does (same slide, same value, same clamp), offers
// its column, and the row candidates of the D lanes are reduced lexicographically (warp
// shuffles) into one row offer. Offers are exact lexicographic minima, so the order in which the
// cells of a sub-step are merged does not change the result. Called convergently by the warp.
template <class P, int D, int HG, bool GUARD>
__device__ __noinline__ void coop_replay(typename P::V a, int src, int s0, int cnt, int i0, int kts,
                                         int kend, int L, double p,
                                         const typename P::V2* colA, const typename P::VB* colB,
                                         int* colT, int X0, int xbs, int ring,
                                         const typename P::V2* rowA, const typename P::VB* rowB,
                                         int* rowT, BestEntry* best, unsigned long long* stats) {
  using V2 = typename P::V2;
  using VB = typename P::VB;
  const int q = threadIdx.x & 31;
  const bool act = q < D;
  if (stats && q == 0) atomicAdd(&stats[0], 1ull);
#pragma unroll 1
  for (int g = 0; g < HG; ++g) {
    const int s = s0 + g * D;
    if (GUARD && s >= cnt) break;
    const int q1 = (X0 + s + xbs) % ring;  // the block's two aligned runs of D ring entries
    const int q2 = (X0 + s + xbs + D) % ring;
#pragma unroll 1
    for (int u = 0; u < D; ++u) {
      if (GUARD && s + u >= cnt) break;
      const int x = s + u;
      const V2 r = rowA[x];
      const VB rb = P::kHasB ? rowB[x] : VB{};
      const int row = i0 + x + 1;
      const int e = u + q;  // entry of the block's column run (lanes q < D)
      const int ce = act ? (e < D ? q1 + e : q2 + e - D) : q1;
      const V2 c = colA[ce + ce / D];
      if (act) a = P::step(a, r, c, p);
      const int k = kts + q;
      const bool valid = act && (!GUARD || ((k < kend) && (row + k <= L - 1)));
      unsigned long long rv = kInfBits;
      int rj = INT_MAX;
      if (valid) {
        const int j = row + k;
        const VB cb = P::kHasB ? colB[ce + ce / D] : VB{};
        const double v = cell_value<P>(a, rb, cb, row, j);
        const int h = __double2hiint(v);
        const int xc = s + xbs + e;  // column offset within the stage window
        int* ct = &colT[xc + xc / D];
        const int tr = *reinterpret_cast<volatile int*>(&rowT[x]);
        const unsigned long long vb = (h < 0) ? 0ull : static_cast<unsigned long long>(__double_as_longlong(v));
        if (h <= *reinterpret_cast<volatile int*>(ct)) {
          atomicMin(ct, static_cast<int>(offer(best, j, vb, row) >> 32));
          if (stats) atomicAdd(&stats[1], 1ull);
        }
        if (h <= tr) {
          rv = vb;
          rj = j;
        }
      }
#pragma unroll
      for (int off = D / 2; off > 0; off >>= 1) {
        const unsigned long long ov = __shfl_xor_sync(0xffffffffu, rv, off);
        const int oj = __shfl_xor_sync(0xffffffffu, rj, off);
        if (lex_less(ov, oj, rv, rj)) {
          rv = ov;
          rj = oj;
        }
      }
      if (q == 0 && rj != INT_MAX) {
        atomicMin(&rowT[x], static_cast<int>(offer(best, row, rv, rj) >> 32));
        if (stats) atomicAdd(&stats[1], 1ull);
      }
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
    const int jo = j;
    if (lex_less(vb, jo, rv, rj)) {
      rv = vb;
      rj = jo;
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
// their thresholds (block maxima precomputed per stage). A cell can only improve (or tie) its
// row or column minimum if its key is <= theta. The hot loop keeps the running minimum key of
// the block (a VIMNMX3 tree, no branch); a block that passes is replayed by `replay_block`.

// Blocks per hit test (one data-dependent branch and one saved accumulator set per group of HG
// blocks instead of per block; a passing group is replayed whole). Measured (sweep ms, 1 B200):
//   covariance-only filters, HG 1 -> 2 -> 4: C4 AAMP 122.7 -> 118.4 -> 115.7, C4 ACAMP 121.7 ->
//   116.6 -> 115.2, C5 ACAMP 2088 -> 2054 -> 2365 (C5 replays ~1e8 blocks: larger groups replay
//   more); column-scaled z-norm (C2) 2.93 -> 2.84; (delta, sigma) AAMP (random walk n = 2^18,
//   m = 128) 8.96 -> 8.83, FP32 C4 AAMP 96.5 -> 92.3; p-norm (C3) p = 1 11.7 -> 12.7, p = 3
//   16.5 -> 17.3, p = 2.5 746 -> 776 (slow-settling thresholds, many replays), so p-norm keeps
//   HG = 1. A per-block hit mask with a
//   merge-free advance over the blocks that did not pass measured slower (C4 AAMP 117.8 at HG 4).
#ifndef MPROF_HIT_GROUP_COV
#define MPROF_HIT_GROUP_COV 2   // covariance-only filters (EuclidCov, Znorm)
#endif
// covariance-form AAMP (EuclidCov), HG 2 -> 4: C4 115.7 -> 113.2, C5-shaped AAMP 1856 -> 1812, but
// random walk m = 256 8.11 -> 8.27, C2-shaped AAMP 6.09 -> 6.48 and a sinusoid (C3 series,
// m = 1024) 53.6 -> 74.2 (replay-heavy), so 2.
#ifndef MPROF_HIT_GROUP_ECOV
#define MPROF_HIT_GROUP_ECOV 2
#endif
#ifndef MPROF_HIT_GROUP_CS
#define MPROF_HIT_GROUP_CS 2    // column-scaled z-norm
#endif
// Warp-cooperative replay (coop_replay; experiment switch, off): parity-green, but C5 ACAMP
// 2052 -> 2262 ms and a random walk n = 2^20, m = 512 ACAMP 129.0 -> 142.5 ms: the replays
// cluster (several lanes of a warp pass together), and serialising them lane by lane through
// the warp costs more than the lanes' concurrent per-lane replays.
#ifndef MPROF_COOP_REPLAY
#define MPROF_COOP_REPLAY 0
#endif
// Warp-uniform hit branch (experiment switch, off): C4 ACAMP 116.7 -> 119.7 ms, C5 2054 -> 2104.
#ifndef MPROF_HIT_VOTE
#define MPROF_HIT_VOTE 0
#endif
#ifndef MPROF_SPLIT_DFMA
#define MPROF_SPLIT_DFMA 0
#endif
#ifndef MPROF_HIT_GROUP_DS
#define MPROF_HIT_GROUP_DS 2    // (delta, sigma) AAMP, FP64 and FP32
#endif
#ifndef MPROF_HIT_GROUP
#define MPROF_HIT_GROUP 1       // other value-key filters (p-norm, exact mode)
#endif

// Exact lexicographic min-update of a shared-memory entry (Dense<P>'s per-stage candidates).
__device__ __forceinline__ void offer_shared(BestEntry* e, unsigned long long v, long long idx) {
  BestEntry cur = *e;
  while (lex_less(v, idx, cur.v, cur.idx)) {
    const BestEntry old = atomicCAS(e, cur, BestEntry{v, idx});
    if (old.v == cur.v && old.idx == cur.idx) return;
    cur = old;
  }
}

// One stage of a Dense<P> sweep: the slide of the hot loop (register ring of column operands,
// row operand broadcast), and for EVERY cell an exact comparison with the row threshold and the
// column threshold in shared memory; a cell that can improve or tie goes into the CTA's
// shared-memory candidates (ccol per live column, crow per row of the stage; flushed to the
// global profile at the stage end by dense_flush) and tightens the shared threshold word.
template <class P, int D, int T, int S, bool GUARD>
__device__ __forceinline__ void dense_stage(SweepSmem<P, D, T, S>& sm, int b, int X0,
                                            typename P::V (&acc)[D], int i0, int cnt, int kt,
                                            int kend, int L, double p) {
  using G = Geo<D, T, S>;
  using V2 = typename P::V2;
  using VB = typename P::VB;
  const int xb = threadIdx.x * D;
  V2 cA[D];
  VB cB[D];
  {
    const int q0 = G::pad((X0 + xb) % G::RING);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      cA[d] = sm.colA[q0 + d];
      if constexpr (P::kHasB) cB[d] = sm.colB[q0 + d];
    }
  }
  const V2* rowA = sm.rowA[b];
  int* colT = sm.colT[b];
  for (int s = 0; s < cnt; s += D) {
    const int qn = G::pad((X0 + s + xb + D) % G::RING);
    MPG_CHECK(qn + D <= G::RINGP);
    const V2* nA = &sm.colA[qn];
    const VB* nB = &sm.colB[P::kHasB ? qn : 0];
#pragma unroll
    for (int u = 0; u < D; ++u) {
      if (GUARD && s + u >= cnt) break;
      const int x = s + u;
      MPG_CHECK(x < S);
      const V2 r = rowA[x];
      const VB rb = P::kHasB ? sm.rowB[b][x] : VB{};
      const int row = i0 + x + 1;
      const int tr = *reinterpret_cast<volatile int*>(&sm.rowT[b][x]);
      unsigned long long rv = kInfBits;
      int rj = INT_MAX;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int sl = (d + u) % D;
        acc[d] = P::step(acc[d], r, cA[sl], p);
        if (GUARD && !((kt + d < kend) && (row + kt + d <= L - 1))) continue;
        const int j = row + kt + d;
        const double v = cell_value<P>(acc[d], rb, P::kHasB ? cB[sl] : VB{}, row, j);
        const int h = __double2hiint(v);
        const unsigned long long vb = (h < 0) ? 0ull : static_cast<unsigned long long>(__double_as_longlong(v));
        const int xc = x + xb + d;  // column offset in the stage window
        MPG_CHECK(xc < G::NCOL && j < L);
        int* ct = &colT[G::pad(xc)];
        if (h <= *reinterpret_cast<volatile int*>(ct)) {
          offer_shared(&sm.ccol[xc], vb, row);
          atomicMin(ct, h < 0 ? 0 : h);
        }
        if (h <= tr && lex_less(vb, j, rv, rj)) {
          rv = vb;
          rj = j;
        }
      }
      // the row is shared by the whole CTA: reduce the warp's candidates first (lexicographic,
      // shuffles), one shared-memory offer per warp instead of one per thread
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
          offer_shared(&sm.crow[x], rv, rj);
          atomicMin(&sm.rowT[b][x], static_cast<int>(rv >> 32));
        }
      }
      cA[u] = nA[u];
      if constexpr (P::kHasB) cB[u] = nB[u];
    }
  }
}

// Dense<P>: offer the stage's shared candidates to the global profile and reset them (between
// the stage's CTA barriers: no warp touches them). Rows i0 + 1 + x; columns at stage offset x are
// position i0 + kb + 1 + x (load_stage's colT positions).
template <class P, int D, int T, int S>
__device__ __forceinline__ void dense_flush(SweepSmem<P, D, T, S>& sm, BestEntry* best, int i0,
                                            int kb, int L) {
  using G = Geo<D, T, S>;
  for (int x = threadIdx.x; x < S; x += T) {
    const BestEntry e = sm.crow[x];
    if (e.idx != kNoIdx && i0 + 1 + x < L) offer(best, i0 + 1 + x, e.v, e.idx);
    sm.crow[x] = BestEntry{kInfBits, kNoIdx};
  }
  for (int x = threadIdx.x; x < G::NCOL; x += T) {
    const BestEntry e = sm.ccol[x];
    if (e.idx != kNoIdx && i0 + kb + 1 + x < L) offer(best, i0 + kb + 1 + x, e.v, e.idx);
    sm.ccol[x] = BestEntry{kInfBits, kNoIdx};
  }
}

// Blocks per hit test of policy P's kernel (the policy's own choice, else per filter kind).
template <class P>
__host__ __device__ constexpr int hit_group_for() {
  constexpr bool EQ = is_euclid_cov<P>();
  constexpr bool ZQ = P::kCovFilter && !P::kColScale && !EQ;
  if constexpr (hit_group_of<P>() != 0) return hit_group_of<P>();
  else if constexpr (EQ) return MPROF_HIT_GROUP_ECOV;
  else if constexpr (ZQ) return MPROF_HIT_GROUP_COV;
  else if constexpr (P::kColScale) return MPROF_HIT_GROUP_CS;
  else return P::kPairs == kPairsDeltaSum ? MPROF_HIT_GROUP_DS : MPROF_HIT_GROUP;
}

template <class P, int D, int T, int S, bool GUARD>
__device__ __forceinline__ void run_stage(SweepSmem<P, D, T, S>& sm, int b, int X0,
                                          typename P::V (&acc)[D], int i0, int cnt, int kt,
                                          int kend, int L, BestEntry* best, double p,
                                          unsigned long long* stats) {
  if constexpr (is_dense<P>()) {
    dense_stage<P, D, T, S, GUARD>(sm, b, X0, acc, i0, cnt, kt, kend, L, p);
    return;
  }
  using G = Geo<D, T, S>;
  using V2 = typename P::V2;
  using VB = typename P::VB;
  constexpr bool kColScale = P::kColScale;
  const int xb = threadIdx.x * D;
  V2 cA[D];
  VB cB[D];
  {
    const int q0 = G::pad((X0 + xb) % G::RING);  // X0 + xb is a multiple of D: no wrap inside
#pragma unroll
    for (int d = 0; d < D; ++d) {
      cA[d] = sm.colA[q0 + d];
      if constexpr (kColScale) cB[d] = sm.colB[q0 + d];
    }
  }
  const V2* rowA = sm.rowA[b];
  // Block threshold (software-pipelined: block s+D's is computed during block s, unconditionally
  // with a clamped index, so its shared-load -> convert -> multiply chain overlaps the block's
  // FP64 work instead of sitting between the block's hit test and the next block).
  // theta: key bound of the block; num: covariance filters' 1 - tau_max (0 = every cell may pass)
  auto block_theta = [&](int s, int& theta, double& num) {
    const int cb = s / D + threadIdx.x;
    const int tmax = max(sm.rowBM[s / D], sm.colBM2[cb]);
    theta = P::tau(tmax);
    num = 0.0;
    if constexpr (P::kCovFilter && kColScale) {
      if (tmax >= 0x3FF00000) theta = INT_MAX;  // some threshold >= 1: any cell may qualify
      else num = (1.0 - __hiloint2double(tmax, -1)) * (1.0 - 0x1p-40);  // margin for roundings
    }
  };
  // Covariance-only form: the stage tables make it two broadcast/strided loads and float math;
  // the bound is kept as a raw word (hit <=> max raw(cov) >= bound), INT_MIN = every cell may
  // pass. Computed unconditionally (index clamped) so it schedules into the block's FP64 work.
  constexpr bool ZQ = SweepSmem<P, D, T, S>::ZQ || SweepSmem<P, D, T, S>::EQ;  // raw cov keys
  constexpr bool SKON = SweepSmem<P, D, T, S>::SK && !GUARD;  // sampled keys (interior stages)
  constexpr int HG = hit_group_for<P>();
  static_assert(S % (HG * D) == 0, "a full stage is whole hit groups");
  const float md_f = static_cast<float>(is_euclid_cov<P>() ? g_cell_ctx.md : 0.0);
  auto block_theta_cov = [&](int s) {
    float th;
    if constexpr (SweepSmem<P, D, T, S>::EQ) {
      // 2 cov >= S_i + S_j + m (mu_i - mu_j)^2 - tau over the block's rows and columns
      const float4 rq = sm.erow[s / D];
      const float4 cq = sm.ecol[s / D + threadIdx.x];
      const float gap = fmaxf(0.f, fmaxf(__fsub_rd(cq.y, rq.z), __fsub_rd(rq.y, cq.z)));
      const float ss = __fmaf_rd(__fmul_rd(md_f, gap), gap, __fadd_rd(rq.x, cq.x));
      // margin for the FP64 roundings of the replay's value (relative to its terms)
      th = 0.5f * __fsub_rd(__fmul_rd(ss, 1.f - 0x1p-20f), fmaxf(rq.w, cq.w));
    } else {
      const float2 rq = sm.zrow[s / D];
      const float2 cq = sm.zcol[s / D + threadIdx.x];
      th = fminf(__fmul_rd(rq.x, cq.y), __fmul_rd(cq.x, rq.y));
    }
    if constexpr (SKON) {
      const float2 dr = sm.drow[s / D];
      const float2 dc = sm.dcol[s / D + threadIdx.x];
      th = __fsub_rd(th, __fmaf_ru(dr.x, dc.y, __fmul_ru(dc.x, dr.y)));
    }
    return th > 0.f ? P::cov_bound_raw_f(th) : INT_MIN;
  };
  int theta_nx;
  double num_nx = 0.0;
  if constexpr (ZQ) theta_nx = block_theta_cov(0);
  else block_theta(0, theta_nx, num_nx);
  for (int s0 = 0; s0 < cnt; s0 += HG * D) {
    // HG blocks share one hit test (one data-dependent branch) and one saved accumulator set; a
    // group that passes is replayed block by block from the group start.
    Acc<P, D> acc0;
#pragma unroll
    for (int d = 0; d < D; ++d) acc0.a[d] = acc[d];
    bool hit = false;
#pragma unroll
    for (int g = 0; g < HG; ++g) {
      const int s = s0 + g * D;
      if (HG > 1 && GUARD && s >= cnt) break;
      // the D operands entering during this block are contiguous in the ring: constant offsets
      const int qn = G::pad((X0 + s + xb + D) % G::RING);
      const V2* nA = &sm.colA[qn];
      const VB* nB = &sm.colB[P::kHasB ? qn : 0];
      const int theta = theta_nx;
      const double num = num_nx;
      if constexpr (ZQ) theta_nx = block_theta_cov(min(s + D, S - D));
      else block_theta(min(s + D, S - D), theta_nx, num_nx);
      int hmin = ZQ ? INT_MIN : INT_MAX;  // ZQ: running MAX of raw covariance words
#pragma unroll
      for (int u = 0; u < D; ++u) {
        if (GUARD && s + u >= cnt) break;
        const int x = s + u;
        const V2 r = rowA[x];
        const int row = i0 + x + 1;
        int hu = ZQ ? INT_MIN : INT_MAX;
#if MPROF_SPLIT_DFMA
        if constexpr (P::kCovFilter && sizeof(typename P::V) == 8) {
          // the two DFMAs of the slide as two passes over the D diagonals: each pass reads the
          // same row operand in the same slot (register reuse cache), same arithmetic as step()
          typename P::V tmp[D];
#pragma unroll
          for (int d = 0; d < D; ++d) tmp[d] = fma(cA[(d + u) % D].x, r.y, acc[d]);
#pragma unroll
          for (int d = 0; d < D; ++d) acc[d] = fma(cA[(d + u) % D].y, r.x, tmp[d]);
        }
#endif
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int sl = (d + u) % D;
#if MPROF_SPLIT_DFMA
          if constexpr (!(P::kCovFilter && sizeof(typename P::V) == 8))
#endif
          acc[d] = P::step(acc[d], r, cA[sl], p);
          if constexpr (ZQ) {
            if (!SKON || (u & 1)) {
              int h = P::cov_raw(acc[d]);
              if (GUARD && !((kt + d < kend) && (row + kt + d <= L - 1))) h = INT_MIN;
              hu = max(hu, h);
            }
          } else {
            int h;
            if constexpr (kColScale) h = P::cov_key(acc[d] * cB[sl]);
            else h = P::key(acc[d]);
            if (GUARD && !((kt + d < kend) && (row + kt + d <= L - 1))) h = INT_MAX;
            hu = min(hu, h);
          }
        }
        if constexpr (kColScale) {
          // row bound for this sub-step: cov * B_j >= (1 - tau) / B_i
          const int tu = (num == 0.0) ? INT_MAX
                                      : P::cov_bound(num * static_cast<double>(sm.rowIBx[x]));
          hit |= hu <= tu;
        } else if constexpr (ZQ) {
          hmin = max(hmin, hu);
        } else {
          hmin = min(hmin, hu);
        }
        // slide the column ring: slot u (used by d = 0 this substep) takes the next operand
        cA[u] = nA[u];
        if constexpr (kColScale) cB[u] = nB[u];
      }
      if constexpr (ZQ) hit |= hmin >= theta;
      else if constexpr (!kColScale) hit |= hmin <= theta;
    }
#if MPROF_COOP_REPLAY
    if constexpr (HG > 1) {
      unsigned pend = __ballot_sync(0xffffffffu, hit);
      while (pend) {
        const int src = __ffs(pend) - 1;
        pend &= pend - 1;
        const int lane = threadIdx.x & 31;
        typename P::V a{};
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const typename P::V v = __shfl_sync(0xffffffffu, acc0.a[d], src);
          if (lane == d) a = v;
        }
        coop_replay<P, D, HG, GUARD>(a, src, s0, cnt, i0, kt + (src - lane) * D, kend, L, p,
                                     sm.colA, sm.colB, sm.colT[b], X0, (threadIdx.x - lane + src) * D,
                                     G::RING, rowA, sm.rowB[b], sm.rowT[b], best, stats);
      }
      continue;
    }
#endif
#if MPROF_HIT_VOTE
    // warp-uniform branch: the whole warp replays the group when any lane passes (a lane whose
    // group did not pass finds no cell in the replay, the filter being conservative)
    if (__any_sync(0xffffffffu, hit)) {
#else
    if (hit) {
#endif
      int* colT = sm.colT[b];
#pragma unroll 1
      for (int g = 0; g < HG; ++g) {
        const int s = s0 + g * D;
        if (HG > 1 && GUARD && s >= cnt) break;
        const int q1 = G::pad((X0 + s + xb) % G::RING);
        const int q2 = G::pad((X0 + s + xb + D) % G::RING);
        acc0 = replay_block<P, D, GUARD>(acc0, s, cnt, i0, kt, kend, L, p, &sm.colA[q1],
                                         &sm.colA[q2], &sm.colB[P::kHasB ? q1 : 0],
                                         &sm.colB[P::kHasB ? q2 : 0], &colT[G::pad(s + xb)],
                                         &colT[G::pad(s + xb + D)], rowA, sm.rowB[b], sm.rowT[b],
                                         best, stats);
      }
    }
  }
}

// Upper bound of B from its storage word: FP64 high word (low word all ones), FP32 bits.
template <class VB>
__device__ __forceinline__ int scale_word(const VB* p) {
  if constexpr (sizeof(VB) == 8) return reinterpret_cast<const int*>(p)[1];
  else return __float_as_int(*p);
}
// B >= 0: a lower bound of 1 / max B from the largest word of a block.
template <class VB>
__device__ __forceinline__ float inv_bound(int w) {
  if constexpr (sizeof(VB) == 8) return __frcp_rd(__double2float_ru(__hiloint2double(w, -1)));
  else return __frcp_rd(__int_as_float(w));
}

// Lower bound of (1 - tau) * ib, tau <= the largest value with high word tmax; -inf when tau may
// reach 1 (every cell may qualify) or the bound underflows.
__device__ __forceinline__ float one_minus_tau_ib(int tmax, float ib) {
  if (tmax >= 0x3FF00000) return -INFINITY;
  const float u = __double2float_rd((1.0 - __hiloint2double(tmax, -1)) * (1.0 - 0x1p-40));
  return u > 0.f ? __fmul_rd(u, ib) : -INFINITY;
}

// Covariance-form AAMP tables: an upper bound (float) of the comparison values with high word
// <= w (+inf for the unset threshold), and of a mean stored rounded down.
__device__ __forceinline__ float tau_up(int w) {
  if (w >= 0x7FF00000) return INFINITY;
  return w < 0 ? 0.f : __double2float_ru(__hiloint2double(w, -1));
}
__device__ __forceinline__ float mu_up(float v) {
  return v == -INFINITY ? v : __fadd_ru(v, fmaxf(fabsf(v) * 0x1p-22f, 0x1p-126f));
}

// Block maxima of the freshly loaded thresholds (after the stage's cp.async completed).
template <class P, int D, int T, int S, bool ROWA = true>
__device__ __forceinline__ void stage_block_max(SweepSmem<P, D, T, S, ROWA>& sm, int b, int X0) {
  using G = Geo<D, T, S>;
  using SM = SweepSmem<P, D, T, S>;
  using VB = typename P::VB;
  static_assert(SM::NCB <= 2 * T && S / D <= T - 32, "block-table work split");
  // This section runs between the stage's two CTA barriers, so its critical path (the busiest
  // thread) is what the CTA waits for. Column pair c = blocks c and c+1 (the columns
  // [cD, cD + 2D - 1) one thread's block touches): each thread reduces ONE aligned block of D
  // words and takes its neighbour's from the next lane (lane 31 reduces the neighbour itself);
  // a second round covers blocks T .. NCB-1. Row blocks go to warp 1, which has no second round.
  const int t = threadIdx.x, lane = t & 31;
  if constexpr (SM::SK) {
    using V2 = typename P::V2;
    // |value| upper-bound words: high word without the sign (low word taken as all ones)
    auto absw = [](double v) { return __double2hiint(v) & 0x7FFFFFFF; };
    auto absb = [](int w) { return __double2float_ru(__hiloint2double(w, -1)); };
    auto dblock = [&](int blk) {
      int2 w = make_int2(0, 0);
      if (blk < SM::NCB) {
        const int q = G::pad((X0 + blk * D) % G::RING);
#pragma unroll
        for (int d = 0; d < D; ++d) {
          if (blk * D + d < G::NCOL) {
            const V2 a = sm.colA[q + d];
            w.x = max(w.x, absw(a.x));
            w.y = max(w.y, absw(a.y));
          }
        }
      }
      return w;
    };
#pragma unroll
    for (int base = 0; base < 2 * T; base += T) {
      if (base >= SM::NCB - 1) break;
      const int c = base + t;
      const int2 v = dblock(c);
      int2 o;
      o.x = __shfl_down_sync(0xffffffffu, v.x, 1);
      o.y = __shfl_down_sync(0xffffffffu, v.y, 1);
      if (lane == 31) o = dblock(c + 1);
      if (c < SM::NCB - 1) sm.dcol[c] = make_float2(absb(max(v.x, o.x)), absb(max(v.y, o.y)));
    }
    static_assert(S / D <= T - 64, "row blocks of the step bound on warp 2");
    if (t >= 64 && t < 64 + S / D) {
      const int r = t - 64;
      int2 w = make_int2(0, 0);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const V2 a = sm.rowA[b][r * D + d];
        w.x = max(w.x, absw(a.x));
        w.y = max(w.y, absw(a.y));
      }
      sm.drow[r] = make_float2(absb(w.x), absb(w.y));
    }
  }
  if constexpr (SM::EQ) {
    // {min S, min mu, max mu, max tau} per aligned block of D columns; pair c = blocks c, c+1
    auto block = [&](int blk) {
      float4 v = make_float4(INFINITY, INFINITY, -INFINITY, 0.f);
      int tm = INT_MIN;
      if (blk < SM::NCB) {
        const int q = G::pad((X0 + blk * D) % G::RING);
#pragma unroll
        for (int d = 0; d < D; ++d) {
          if (blk * D + d < G::NCOL) {
            tm = max(tm, sm.colT[b][G::pad(blk * D + d)]);
            const float2 sb = sm.colB[q + d];
            v.x = fminf(v.x, sb.x);
            v.y = fminf(v.y, sb.y);
            v.z = fmaxf(v.z, sb.y);
          }
        }
      }
      v.w = tau_up(tm);
      return v;
    };
#pragma unroll
    for (int base = 0; base < 2 * T; base += T) {
      if (base >= SM::NCB - 1) break;
      const int c = base + t;
      const float4 v = block(c);
      float4 o;
      o.x = __shfl_down_sync(0xffffffffu, v.x, 1);
      o.y = __shfl_down_sync(0xffffffffu, v.y, 1);
      o.z = __shfl_down_sync(0xffffffffu, v.z, 1);
      o.w = __shfl_down_sync(0xffffffffu, v.w, 1);
      if (lane == 31) o = block(c + 1);
      if (c < SM::NCB - 1)
        sm.ecol[c] = make_float4(fminf(v.x, o.x), fminf(v.y, o.y), mu_up(fmaxf(v.z, o.z)),
                                 fmaxf(v.w, o.w));
    }
    if (t >= 32 && t < 32 + S / D) {
      const int r = t - 32;
      float4 v = make_float4(INFINITY, INFINITY, -INFINITY, 0.f);
      int tm = INT_MIN;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        tm = max(tm, sm.rowT[b][r * D + d]);
        const float2 sb = sm.rowB[b][r * D + d];
        v.x = fminf(v.x, sb.x);
        v.y = fminf(v.y, sb.y);
        v.z = fmaxf(v.z, sb.y);
      }
      sm.erow[r] = make_float4(v.x, v.y, mu_up(v.z), tau_up(tm));
    }
    return;
  }
  auto block = [&](int blk, int& tm, int& hm) {
    tm = INT_MIN;
    hm = 0;
    if (blk >= SM::NCB) return;
    const int q = G::pad((X0 + blk * D) % G::RING);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (blk * D + d < G::NCOL) {
        tm = max(tm, sm.colT[b][G::pad(blk * D + d)]);
        if constexpr (SM::ZQ) hm = max(hm, scale_word<VB>(&sm.colB[q + d]));
      }
    }
  };
#pragma unroll
  for (int base = 0; base < 2 * T; base += T) {
    if (base >= SM::NCB - 1) break;
    const int c = base + t;
    int tm, hm;
    block(c, tm, hm);
    int tn = __shfl_down_sync(0xffffffffu, tm, 1);
    int hn = __shfl_down_sync(0xffffffffu, hm, 1);
    if (lane == 31) block(c + 1, tn, hn);
    if (c < SM::NCB - 1) {
      const int tmax = max(tm, tn);
      if constexpr (SM::TW) sm.colBM2[c] = tmax;
      if constexpr (SM::ZQ) {
        const float ib = inv_bound<VB>(max(hm, hn));
        sm.zcol[c] = make_float2(one_minus_tau_ib(tmax, ib), ib);
      }
    }
  }
  if (t >= 32 && t < 32 + S / D) {
    const int r = t - 32;
    int mx = INT_MIN, hmax = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      mx = max(mx, sm.rowT[b][r * D + d]);
      if constexpr (SM::ZQ) hmax = max(hmax, scale_word<VB>(&sm.rowB[b][r * D + d]));
    }
    if constexpr (SM::TW) sm.rowBM[r] = mx;
    if constexpr (SM::ZQ) {
      const float ib = inv_bound<VB>(hmax);
      sm.zrow[r] = make_float2(one_minus_tau_ib(mx, ib), ib);
    }
  }
  if constexpr (P::kColScale) {
    for (int x = t; x < S; x += T) sm.rowIBx[x] = inv_bound<VB>(scale_word<VB>(&sm.rowB[b][x]));
  }
}

// Issue the cp.async copies of stage st (row transitions i0 .. i0+S-1, i0 = ra + st*S):
// its row operands and thresholds, the thresholds of its whole live column window, and the
// column operands that enter the ring with it (all NCOL for stage 0, S afterwards).
template <class P, int D, int T, int S, bool ROWA = true>
__device__ __forceinline__ void load_stage(SweepSmem<P, D, T, S, ROWA>& sm, const SweepParams& prm,
                                           int st, int ra, int kb) {
  using G = Geo<D, T, S>;
  using V2 = typename P::V2;
  using VB = typename P::VB;
  const V2* A = pairs_of<P>(prm);
  const VB* Bs = scales_of<P>(prm);
  const int L = prm.L;
  const int b = st & 1;
  const int i0 = ra + st * S;
  const int* bestw = reinterpret_cast<const int*>(prm.best);  // word view; hi word at +1
  MPG_CHECK(i0 >= 0 && kb >= 0 && i0 + kb < L);
  for (int x = threadIdx.x; x < G::NCOL; x += T) {
    const int pb = i0 + kb + 1 + x;
    const bool vb = pb < L;
    cp_async<4>(&sm.colT[b][G::pad(x)], bestw + 4 * (vb ? pb : 0) + 1, vb);
  }
  const int Xlo = st == 0 ? 0 : st * S + G::K;
  const int Xhi = st * S + G::NCOL;
  for (int X = Xlo + threadIdx.x; X < Xhi; X += T) {
    const int pa = ra + kb + X;
    const bool va = pa < L - 1, vb = pa + 1 < L;
    const int q = G::pad(X % G::RING);
    cp_async<sizeof(V2)>(&sm.colA[q], A + (va ? pa : 0), va);
    if constexpr (P::kHasB) cp_async<sizeof(VB)>(&sm.colB[q], Bs + (vb ? pa + 1 : 0), vb);
  }
  for (int x = threadIdx.x; x < S; x += T) {
    const int pa = i0 + x;
    const int pb = pa + 1;
    const bool va = pa < L - 1, vb = pb < L;
    if constexpr (ROWA) cp_async<sizeof(V2)>(&sm.rowA[b][x], A + (va ? pa : 0), va);
    if constexpr (P::kHasB) cp_async<sizeof(VB)>(&sm.rowB[b][x], Bs + (vb ? pb : 0), vb);
    cp_async<4>(&sm.rowT[b][x], bestw + 4 * (vb ? pb : 0) + 1, vb);
  }
}

// ---------------------------------------------------------------------------------------------
// The sweep kernel: one CTA per tile (kb, ra).

template <class P, int D, int T, int S, int MINB>
__global__ void __launch_bounds__(T, MINB) sweep_kernel(const SweepParams prm) {
  using G = Geo<D, T, S>;
  using SM = SweepSmem<P, D, T, S>;
  using V = typename P::V;
  using VB = typename P::VB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);

  const int4 tl = prm.tiles[blockIdx.x];
  const int kb = tl.x, ra = tl.y;
  const int re = tl.z;  // exclusive row end of the tile (<= L - kb, <= row_hi)
  MPG_CHECK(kb >= 1 && ra >= 0 && ra < re && re <= prm.L - kb && re <= prm.row_hi && tl.w > kb &&
            tl.w <= prm.L);
  const int L = prm.L;
  const int m = prm.m;
  const int kt = kb + static_cast<int>(threadIdx.x) * D;
  const int kend = min(min(tl.w, kb + G::K), prm.k_hi);  // the tile's diagonals: [kb, kend)
  if constexpr (is_euclid_cov<P>()) {
    if (threadIdx.x == 0) g_cell_ctx = CellCtx{prm.S, prm.mu, static_cast<double>(m)};
    __syncthreads();
  }

  // ---- seed (FP64): direct length-m sum for the pair (ra, ra + kt + d) --------------------
  double sacc[D];
  double muc[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    sacc[d] = 0.0;
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
          for (int d = 0; d < D; ++d) sacc[d] = P::seed(sacc[d], a, w[(d + u) % D], muc[d], prm.p);
          w[u] = scol[G::pad(l + u + xb + D)];
        }
      }
    }
  }
  V acc[D];
#pragma unroll
  for (int d = 0; d < D; ++d) acc[d] = static_cast<V>(sacc[d]);

  // ---- the seed cells (ra, ra + k): exact merge -------------------------------------------
  {
    const VB* Bs = scales_of<P>(prm);
    Cells<D> c;
    unsigned valid = 0;
    const VB rb = P::kHasB ? Bs[ra] : VB{};
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int k = kt + d;
      const bool ok = (k < kend) && (ra + k <= L - 1);
      const VB cb = (P::kHasB && ok) ? Bs[ra + k] : VB{};
      c.v[d] = ok ? cell_value<P>(acc[d], rb, cb, ra, ra + k) : 0.0;
      valid |= (ok ? 1u : 0u) << d;
    }
    resolve_seed<D>(c, valid, ra, ra + kt, prm.best);
  }

  // ---- stage pipeline over the row transitions ra .. re-2 ---------------------------------
  // Two CTA barriers per stage: (1) stage st+1's copies landed and every warp finished stage st
  // (its row/threshold buffers and the ring slots of offsets [st*S, st*S + S) are free), then
  // the block maxima of st+1 are computed and the copies of st+2 are issued into the freed
  // buffers, a whole stage ahead of use; (2) the block maxima are visible.
  const int steps = re - 1 - ra;
  if (steps <= 0) return;
  const int nst = (steps + S - 1) / S;
  __syncthreads();  // seed scratch reuse
  if constexpr (SM::DN) {
    for (int x = threadIdx.x; x < S; x += T) sm.crow[x] = BestEntry{kInfBits, kNoIdx};
    for (int x = threadIdx.x; x < G::NCOL; x += T) sm.ccol[x] = BestEntry{kInfBits, kNoIdx};
  }
  load_stage<P, D, T, S>(sm, prm, 0, ra, kb);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  stage_block_max<P, D, T, S>(sm, 0, 0);
  if (nst > 1) load_stage<P, D, T, S>(sm, prm, 1, ra, kb);
  cp_async_commit();
  __syncthreads();
  for (int st = 0; st < nst; ++st) {
    const int s0 = st * S;
    const int cnt = min(S, steps - s0);
    const int i0 = ra + s0;
    const bool full = (cnt == S) && (kb + G::K <= kend) && (i0 + cnt + kb + G::K - 1 <= L - 1);
    if (full) {
      run_stage<P, D, T, S, false>(sm, st & 1, s0, acc, i0, cnt, kt, kend, L, prm.best, prm.p, prm.stats);
    } else {
      run_stage<P, D, T, S, true>(sm, st & 1, s0, acc, i0, cnt, kt, kend, L, prm.best, prm.p, prm.stats);
    }
    if (st + 1 == nst) {
      if constexpr (SM::DN) {
        __syncthreads();
        dense_flush<P, D, T, S>(sm, prm.best, i0, kb, L);
      }
      break;
    }
    cp_async_wait<0>();
    __syncthreads();
    if constexpr (SM::DN) dense_flush<P, D, T, S>(sm, prm.best, i0, kb, L);
    stage_block_max<P, D, T, S>(sm, (st + 1) & 1, s0 + S);
    if (st + 2 < nst) load_stage<P, D, T, S>(sm, prm, st + 2, ra, kb);
    cp_async_commit();
    __syncthreads();
  }
}

}  // namespace mpg
