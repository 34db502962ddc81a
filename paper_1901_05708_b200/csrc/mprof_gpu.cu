// mprof_gpu.cu — host orchestration, auxiliary kernels and the C ABI (include/mprof_gpu.h).
//
// Pipeline of one sweep (replaces mprof::detail::run_engine,
// /root/reference/proj/src/diag_scan.cpp:89-140):
//   init_best -> operand prep (pairs / z-norm statistics) -> first-diagonal thresholds
//   -> sweep_kernel (all tiles) -> [z-norm flat-pair rule] -> split to (cmp, idx)
//   -> finalize (comparison value -> distance).
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/mprof_gpu.h"
#include "sweep.cuh"
#include "sweep_rc.h"

using namespace mpg;

namespace {

// ---- tile configuration (one instantiation for every family) -------------------------------
#ifndef MPROF_TILE_D
#define MPROF_TILE_D 8
#endif
#ifndef MPROF_TILE_T
#define MPROF_TILE_T 128
#endif
#ifndef MPROF_TILE_S
#define MPROF_TILE_S 128
#endif
#ifndef MPROF_MIN_BLOCKS
#define MPROF_MIN_BLOCKS 4
#endif
constexpr int kD = MPROF_TILE_D;  // diagonals per thread
constexpr int kT = MPROF_TILE_T;  // threads per CTA
constexpr int kS = MPROF_TILE_S;  // rows per shared-memory stage
constexpr int kK = kD * kT;
// covariance-only z-norm filter when the mean min/max window-scale ratio over 2*kD windows is at
// least this (calibrated on the BASELINE workloads: m=1024 0.983, m=512 0.967 -> cov-only is
// faster; m=256 0.93 -> column-scaled is 1.8x faster)
constexpr double kZnCovFilterMinSpread = 0.955;
// the same test for the covariance-form AAMP kernel (EuclidCov): measured on random walks,
// m=1024 (spread 0.983) -10.7 %, m=256 (0.93) -7 %, m=128 +6.5 %, m=100 (C1) 3.9x slower
constexpr double kAampCovMinSpread = 0.92;
// Form probe (probe_form): kProbeTiles short tiles of kProbeRows rows swept with the
// covariance-form kernel before the main launch; above kProbeMaxReplays replayed blocks per cell
// the (delta, sigma) kernel sweeps the band instead.
constexpr int kProbeTiles = 148, kProbeRows = 256;
constexpr double kProbeMaxReplays = 5e-6, kProbeMinCells = 4e9;
// z-norm: the covariance-only filter against the column-scaled one (+1 DMUL per cell): measured
// replayed blocks per cell of the covariance-only form where it still wins: C5 1.6e-5, random
// walk m = 512 1.6e-5; where the column-scaled form wins: C3 sinusoids m = 1024 4.7e-5, m = 256
// 7.1e-4.
constexpr double kProbeMaxReplaysZ = 3e-5;
// Longer hit groups (Wide<P>) when the probe saw at most 1e-5 replayed blocks per cell: measured
// HG 2 -> 4, C4 AAMP 115.7 -> 113.2 ms, C4 ACAMP 116.6 -> 115.2 ms (0 probe replays), while a
// random walk m = 256 AAMP (10 probe replays) went 8.11 -> 8.27 and C5 (834) 2054 -> 2365. The
// bound was 5e-8 (~2 replays) in round 1; the round-2 probe sample sees 204 replays on C4 ACAMP
// (5.3e-6 per cell), where HG 8 still measured 118.7 -> 115.9 ms; C5 (2e-5) keeps HG 2.
#ifndef MPROF_WIDE_MAX_REPLAYS
#define MPROF_WIDE_MAX_REPLAYS 1e-5
#endif
constexpr double kProbeWideMaxReplays = MPROF_WIDE_MAX_REPLAYS;
// Noise test (k_noise_test): random admissible pairs evaluated directly; above this fraction
// passing the first-diagonal thresholds the series would sweep with Dense<P> (no block filter).
// Off by default (> 1): measured on uniform noise, m = 256, Dense<P> wins only at the smallest
// sizes (AAMP n = 2^13 1.75 vs 2.15 ms, ACAMP 0.83 vs 1.6 ms) and loses from n = 2^14 on (n = 2^16:
// AAMP 12.0 vs 4.9 ms, ACAMP 8.0 vs 3.9 ms) -- DESIGN.md §3.5. Dense<P> stays available through
// mprof_ctx_set_form(DENSE).
constexpr int kNoiseSamples = 2048;
#ifndef MPROF_NOISE_DENSE_FRAC
#define MPROF_NOISE_DENSE_FRAC 2.0
#endif
constexpr double kNoiseDenseFrac = MPROF_NOISE_DENSE_FRAC;

// Experiment / diagnostic switches, read once per process from the environment. The defaults are
// the product configuration; tests and bench never set them (tools/ and DESIGN.md experiments do).
struct Knobs {
  long long rows_per_tile = 0;  // MPROF_ROWS_PER_TILE: fixed rows per tile (0 = choose_R)
  bool tile_debug = false;      // MPROF_TILE_DEBUG: print the schedule model's candidates
  bool tile_order_lpt = false;  // MPROF_TILE_ORDER_LPT: longest-first tile order
  int zn_filter = 0;            // MPROF_ZN_FILTER=cov|col: force the z-norm filter form
  bool zn_no_near = false;      // MPROF_ZN_NO_NEAR: no column-scaled near-diagonal block
  bool stats = false;           // MPROF_STATS: count replays / offers (stderr)
  int aamp_cov = -1;            // MPROF_AAMP_COV=0|1: force the AAMP form (-1: by window spread)
  bool no_graph = false;        // MPROF_NO_GRAPH: planned sweeps launch their window chain directly
};
const Knobs& knobs() {
  static const Knobs k = [] {
    Knobs r;
    if (const char* e = getenv("MPROF_ROWS_PER_TILE")) r.rows_per_tile = std::max(1LL, atoll(e));
    r.tile_debug = getenv("MPROF_TILE_DEBUG") != nullptr;
    r.tile_order_lpt = getenv("MPROF_TILE_ORDER_LPT") != nullptr;
    if (const char* e = getenv("MPROF_ZN_FILTER")) r.zn_filter = !strcmp(e, "cov") ? 1 : !strcmp(e, "col") ? 2 : 0;
    r.zn_no_near = getenv("MPROF_ZN_NO_NEAR") != nullptr;
    r.stats = getenv("MPROF_STATS") != nullptr;
    if (const char* e = getenv("MPROF_AAMP_COV")) r.aamp_cov = atoi(e) ? 1 : 0;
    r.no_graph = getenv("MPROF_NO_GRAPH") != nullptr;
    return r;
  }();
  return k;
}

thread_local std::string g_last_error;

int32_t fail(int32_t code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int32_t cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky non-fatal state
  return fail(e == cudaErrorMemoryAllocation ? MPROF_E_OOM : MPROF_E_CUDA, "%s: %s", what,
              cudaGetErrorString(e));
}

#define CK(expr)                                       \
  do {                                                 \
    cudaError_t e__ = (expr);                          \
    if (e__ != cudaSuccess) return cuda_fail(e__, #expr); \
  } while (0)

// ---------------------------------------------------------------------------------------------
// auxiliary kernels

// Initial profile. With B (z-norm) flat windows are PINNED to (0, -1), an entry nothing can
// beat and whose threshold word (0) no cell passes: every pair with a flat side scores exactly
// d = 1 (or the flat-flat minimum), so flat rows/columns would otherwise tie on every cell of the
// sweep. k_flat_fix assigns their final entries directly.
__global__ void k_init_best(BestEntry* best, const double* __restrict__ B, int L) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x)
    best[i] = (B && B[i] == 0.0) ? BestEntry{0ull, -1} : BestEntry{kInfBits, kNoIdx};
}

// A[p] for p in [0, L-1): kPairsRaw (t[p], t[p+m]); kPairsDeltaSum (t[p+m]-t[p], t[p+m]+t[p])
__global__ void k_build_pairs(const double* __restrict__ t, double2* __restrict__ A, int L, int m,
                              int kind) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L - 1; p += gridDim.x * blockDim.x) {
    const double a = t[p], b = t[p + m];
    A[p] = kind == kPairsDeltaSum ? make_double2(b - a, b + a) : make_double2(a, b);
  }
}

// Window statistics, register-blocked: a CTA of kWsT threads owns kWsSpan = kWsT * kWsW
// consecutive windows, thread tid the kWsW windows P0 + tid * kWsW + [0, kWsW). The samples are
// staged through shared memory in chunks of kWsC window offsets (each sample read from global
// once per CTA and chunk instead of once per window) and every thread keeps a register ring of
// kWsW samples, so a window offset l costs ONE shared load per thread for kWsW windows. Every
// window's sums keep the one-window loop's order l = 0..m-1, so the results are bit-identical to
// summing each window on its own.
#ifndef MPROF_WS_T
#define MPROF_WS_T 128
#endif
constexpr int kWsW = 8, kWsT = MPROF_WS_T, kWsC = 256, kWsSpan = kWsT * kWsW;
constexpr int kWsSmem = (kWsSpan + kWsC) + (kWsSpan + kWsC) / kWsW;  // padded: q -> q + q / kWsW
__device__ __forceinline__ int ws_pad(int q) { return q + q / kWsW; }

// One pass over the window offsets l = 0..m-1 of the CTA's windows: op(w, x) with x = sample
// P0 + tid * kWsW + w + l (minus `shift`), in increasing l for every w.
template <class Op>
__device__ __forceinline__ void ws_pass(const double* __restrict__ t, int n, int P0, int m,
                                        double shift, double* sh, Op op) {
  const int tb = threadIdx.x * kWsW;
  for (int l0 = 0; l0 < m; l0 += kWsC) {
    const int cl = min(kWsC, m - l0);
    __syncthreads();  // previous chunk / pass consumed
    for (int q = threadIdx.x; q < kWsSpan + cl; q += kWsT) {
      const int g = P0 + l0 + q;
      sh[ws_pad(q)] = g < n ? t[g] - shift : 0.0;
    }
    __syncthreads();
    double x[kWsW];  // slot (w + l) % kWsW holds sample tb + w + l of the chunk
#pragma unroll
    for (int w = 0; w < kWsW; ++w) x[w] = sh[ws_pad(tb + w)];
    for (int lb = 0; lb < cl; lb += kWsW) {
#pragma unroll
      for (int u = 0; u < kWsW; ++u) {
        const int l = lb + u;
        if (l < cl) {
#pragma unroll
          for (int w = 0; w < kWsW; ++w) op(w, x[(w + u) % kWsW]);
        }
        const int q = tb + kWsW + l;
        x[u] = q < kWsSpan + cl ? sh[ws_pad(q)] : 0.0;
      }
    }
  }
}

// Per-window mean and inverse centred norm, two-pass (the well-conditioned form; the reference
// derives var from running sums, acamp.hpp:42-47). Flat windows (population variance <=
// flat_threshold, the reference's rule acamp.hpp:55-56 / oracle.cpp:81-84) get B = 0.
__global__ void __launch_bounds__(kWsT) k_znorm_stats(const double* __restrict__ t, int L, int m,
                                                      double flat_thr, double* __restrict__ mu,
                                                      double* __restrict__ B) {
  __shared__ double sh[kWsSmem];
  const int n = L + m - 1;
  for (int P0 = blockIdx.x * kWsSpan; P0 < L; P0 += gridDim.x * kWsSpan) {
    double s[kWsW], ss[kWsW], mean[kWsW];
#pragma unroll
    for (int w = 0; w < kWsW; ++w) s[w] = ss[w] = 0.0;
    ws_pass(t, n, P0, m, 0.0, sh, [&](int w, double x) { s[w] += x; });
#pragma unroll
    for (int w = 0; w < kWsW; ++w) mean[w] = s[w] / m;
    ws_pass(t, n, P0, m, 0.0, sh, [&](int w, double x) {
      const double d = x - mean[w];
      ss[w] = fma(d, d, ss[w]);
    });
#pragma unroll
    for (int w = 0; w < kWsW; ++w) {
      const int p = P0 + threadIdx.x * kWsW + w;
      if (p < L) {
        mu[p] = mean[w];
        const double var = ss[w] / m;
        B[p] = (var <= flat_thr) ? 0.0 : 1.0 / sqrt(ss[w]);
      }
    }
  }
}

// Covariance-form AAMP statistics (EuclidCov in sweep.cuh): two-pass window mean mu_p and
// centred sum of squares S_p (FP64, exact inputs of the comparison values), the float ring
// scalars SB[p] = {S_p rounded down, mu_p - t[0] rounded down} of the filter tables, and
// Bq[p] = 1/sqrt(S_p) (0 for a constant window) for the spread test (k_bspread). Same blocking
// as k_znorm_stats; the samples are staged as t - t[0].
__global__ void __launch_bounds__(kWsT) k_euclid_stats(const double* __restrict__ t, int L, int m,
                                                       double* __restrict__ mu,
                                                       double* __restrict__ S,
                                                       float2* __restrict__ SB,
                                                       double* __restrict__ Bq,
                                                       unsigned int* __restrict__ out_of_range) {
  __shared__ double sh[kWsSmem];
  const int n = L + m - 1;
  const double t0 = t[0];
  for (int P0 = blockIdx.x * kWsSpan; P0 < L; P0 += gridDim.x * kWsSpan) {
    double s[kWsW], ss[kWsW], mean0[kWsW];
#pragma unroll
    for (int w = 0; w < kWsW; ++w) s[w] = ss[w] = 0.0;
    ws_pass(t, n, P0, m, t0, sh, [&](int w, double x) { s[w] += x; });
#pragma unroll
    for (int w = 0; w < kWsW; ++w) mean0[w] = s[w] / m;  // mean of t - t[0]: keeps the digits of level-offset series
    ws_pass(t, n, P0, m, t0, sh, [&](int w, double x) {
      const double d = x - mean0[w];
      ss[w] = fma(d, d, ss[w]);
    });
#pragma unroll
    for (int w = 0; w < kWsW; ++w) {
      const int p = P0 + threadIdx.x * kWsW + w;
      if (p < L) {
        mu[p] = mean0[w] + t0;
        S[p] = ss[w];
        // the float filter tables need S and mu - t[0] well inside float range
        if (!(ss[w] < 1e30 && fabs(mean0[w]) < 1e30)) atomicOr(out_of_range, 1u);
        SB[p] = make_float2(__double2float_rd(ss[w]), __double2float_rd(mean0[w]));
        Bq[p] = ss[w] > 0.0 ? 1.0 / sqrt(ss[w]) : 0.0;
      }
    }
  }
}

int ws_grid(int L) { return std::max(1, std::min((L + kWsSpan - 1) / kWsSpan, 148 * 8)); }

// A[p] = (df_p, dg_p) for the centred-covariance slide (see Znorm in sweep.cuh).
__global__ void k_znorm_pairs(const double* __restrict__ t, const double* __restrict__ mu,
                              double2* __restrict__ A, int L, int m) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L - 1; p += gridDim.x * blockDim.x) {
    const double a = t[p], b = t[p + m];
    A[p] = make_double2(0.5 * (b - a), (b - mu[p + 1]) + (a - mu[p]));
  }
}

// FP32 mode operands (sweep.cuh, *F32 policies). c = series mean (device scalar) is the offset
// that keeps float's digits where the differences are: DeltaSum (delta, sigma - 2c), Raw
// (t - c, t[p+m] - c); z-norm (df, dg) and B are offset-free.
__global__ void k_mean(const double* __restrict__ t, int n, double* out) {
  double s = 0.0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) s += t[p];
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s / n);
}

__global__ void k_build_pairs32(const double* __restrict__ t, float2* __restrict__ A, int L, int m,
                                int kind, const double* __restrict__ mean) {
  const double c = *mean;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L - 1; p += gridDim.x * blockDim.x) {
    const double a = t[p], b = t[p + m];
    A[p] = kind == kPairsDeltaSum ? make_float2((float)(b - a), (float)((b - c) + (a - c)))
                                  : make_float2((float)(a - c), (float)(b - c));
  }
}

__global__ void k_znorm_pairs32(const double2* __restrict__ A, const double* __restrict__ B,
                                float2* __restrict__ A32, float* __restrict__ B32, int L) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L; p += gridDim.x * blockDim.x) {
    if (p < L - 1) A32[p] = make_float2((float)A[p].x, (float)A[p].y);
    B32[p] = (float)B[p];
  }
}

// Spread of the window scales B inside the sweep's filter blocks: mean over windows of
// 2*kD consecutive positions of min B / max B (flat windows skipped). Close to 1 (long windows)
// the covariance-only z-norm filter is tight; lower, the per-cell column-scaled form wins.
__global__ void k_bspread(const double* __restrict__ B, int L, double* out) {
  double sum = 0.0, cnt = 0.0;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; (b + 1) * 2 * kD <= L; b += gridDim.x * blockDim.x) {
    double mn = INFINITY, mx = 0.0;
    for (int d = 0; d < 2 * kD; ++d) {
      const double v = B[b * 2 * kD + d];
      if (v > 0.0) { mn = fmin(mn, v); mx = fmax(mx, v); }
    }
    if (mx > 0.0) { sum += mn / mx; cnt += 1.0; }
  }
  for (int off = 16; off > 0; off >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, off);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], sum);
    atomicAdd(&out[1], cnt);
  }
}

// Thresholds from diagonal k1 = exclusion: every cell (i, i+k1) evaluated directly and merged
// exactly. These are genuine cells, so the (merged) result is unchanged; they only give the
// high-word filter near-final thresholds before the tiles start.
template <class PP>
__global__ void k_first_diag(SweepParams prm, int k1) {
  using P = typename PP::Base;  // FP64 evaluation, also in FP32 mode
  // Runs of kRun consecutive cells (i, i + k1) per thread: a direct length-m seed at the run's
  // first cell, then the policy's O(1) slide (as the tiles do, over far shorter runs). No
  // atomics: this pass runs alone on the profile, the row entry i of cell i is written only by
  // its cell's thread (lexicographic min with what is there: +inf, a pinned flat window, or the
  // previous profile of an extension), and the column entries i + k1 are merged by
  // k_first_diag_cols from the cell values left in prm.scratch.
  constexpr int kRun = 16;
  const int L = prm.L;
  const int cells = min(L - k1, prm.row_hi);  // cells (i, i + k1), i < cells
  const int lane = threadIdx.x & 31;
  const int nruns = (cells + kRun - 1) / kRun;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  // a warp takes 32 runs: their seeds are computed cooperatively (lanes stride over l, coalesced
  // loads; the fast mode's seeds need not follow the reference's summation order), then every
  // lane slides its own run
  for (int base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < nruns; base += warps * 32) {
    double mine = 0.0;
    for (int r = 0; r < 32 && base + r < nruns; ++r) {
      const int i0 = (base + r) * kRun, j0 = i0 + k1;
      const double mui = P::kCenteredSeed ? prm.mu[i0] : 0.0;
      const double muj = P::kCenteredSeed ? prm.mu[j0] : 0.0;
      double part = 0.0;
      for (int l = lane; l < prm.m; l += 32) part = P::seed(part, prm.t[i0 + l] - mui, prm.t[j0 + l], muj, prm.p);
      for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
      if (lane == r) mine = part;
    }
    const int run = base + lane;
    if (run >= nruns) continue;
    const int i0 = run * kRun, j0 = i0 + k1;
    double acc = mine;
    const int end = min(kRun, cells - i0);
    for (int q = 0; q < end; ++q) {
      const int i = i0 + q, j = j0 + q;
      MPG_CHECK(i >= 0 && j < L);
      if (q > 0) acc = P::step(acc, prm.A[i - 1], prm.A[j - 1], prm.p);
      const double v = P::score(acc, P::kHasB ? prm.B[i] : 0.0, P::kHasB ? prm.B[j] : 0.0);
      const unsigned long long vb =
          (__double2hiint(v) < 0) ? 0ull : static_cast<unsigned long long>(__double_as_longlong(v));
      prm.scratch[i] = __longlong_as_double(static_cast<long long>(vb));
      const BestEntry cur = prm.best[i];
      const long long jo = j;
      if (lex_less(vb, jo, cur.v, cur.idx)) prm.best[i] = BestEntry{vb, jo};
    }
  }
}

// Column side of the first-diagonal pass: entry j takes cell (j - k1, j).
__global__ void k_first_diag_cols(SweepParams prm, int k1) {
  const int cells = min(prm.L - k1, prm.row_hi);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cells; i += gridDim.x * blockDim.x) {
    const int j = i + k1;
    const unsigned long long vb = static_cast<unsigned long long>(__double_as_longlong(prm.scratch[i]));
    const BestEntry cur = prm.best[j];
    const long long io = i;
    if (lex_less(vb, io, cur.v, cur.idx)) prm.best[j] = BestEntry{vb, io};
  }
}

// Noise test (plan_series): nsamp admissible pairs (i, i + k) drawn by a fixed hash, each evaluated
// directly (one warp, the policy's seed sum) in the comparison space, and counted when it would
// pass the thresholds the first-diagonal prepass left in best[] (value <= max of the row and
// column entries' values). On a random walk the prepass thresholds (nearest neighbours at k =
// exclusion) are far below a random pair; on noise-like data they are ordinary pair distances
// and about half the random pairs pass -- the block filter then passes almost every block.
template <class PP>
__global__ void k_noise_test(SweepParams prm, int k1, int nsamp, unsigned int* count) {
  using P = typename PP::Base;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const long long span = (long long)prm.L - k1;  // admissible diagonals [k1, L)
  for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nsamp; q += warps) {
    unsigned long long h = 0x9e3779b97f4a7c15ull * (unsigned long long)(q + 1);
    h ^= h >> 31;
    h *= 0xbf58476d1ce4e5b9ull;
    h ^= h >> 29;
    const int k = k1 + (int)(h % (unsigned long long)span);
    const int i = (int)((h >> 32) % (unsigned long long)(prm.L - k));
    const int j = i + k;
    const double mui = P::kCenteredSeed ? prm.mu[i] : 0.0;
    const double muj = P::kCenteredSeed ? prm.mu[j] : 0.0;
    double acc = 0.0;
    for (int l = lane; l < prm.m; l += 32) acc = P::seed(acc, prm.t[i + l] - mui, prm.t[j + l], muj, prm.p);
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) {
      const double v = P::score(acc, P::kHasB ? prm.B[i] : 0.0, P::kHasB ? prm.B[j] : 0.0);
      const unsigned long long vb = v < 0.0 ? 0ull : static_cast<unsigned long long>(__double_as_longlong(v));
      const unsigned long long th = max(prm.best[i].v, prm.best[j].v);
      if (vb <= th) atomicAdd(count, 1u);
    }
  }
}

// z-normalized flat-pair rule (f_value, /root/reference/proj/include/mprof/acamp.hpp:52-60):
// two flat windows score the minimum possible value (distance 0), so a flat window's nearest
// neighbour is the SMALLEST admissible flat window; the sweep scored every pair with a flat
// side as corr = 0 (d = 1, distance sqrt(2m)), which is already right for flat rows without a
// flat partner and for every non-flat row.
constexpr int kChunk = 1024;
__global__ void k_flat_chunk_min(const double* __restrict__ B, int L, int* __restrict__ cmin) {
  __shared__ int sm[32];
  const int c = blockIdx.x;
  int best = INT_MAX;
  for (int x = threadIdx.x; x < kChunk; x += blockDim.x) {
    const int p = c * kChunk + x;
    if (p < L && B[p] == 0.0) best = min(best, p);
  }
  for (int off = 16; off > 0; off >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, off));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = (threadIdx.x < (blockDim.x >> 5)) ? sm[threadIdx.x] : INT_MAX;
    for (int off = 16; off > 0; off >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, off));
    if (threadIdx.x == 0) cmin[c] = best;
  }
}

// Smallest flat position in [lo, hi] using per-chunk minima (cmin) to skip chunks.
__device__ int first_flat(const double* __restrict__ B, const int* __restrict__ cmin, int lo, int hi) {
  if (hi < lo) return INT_MAX;
  for (int c = lo / kChunk; c <= hi / kChunk; ++c) {
    const int cm = cmin[c];
    if (cm == INT_MAX) continue;
    if (cm >= lo) return cm <= hi ? cm : INT_MAX;
    const int x1 = min(hi, c * kChunk + kChunk - 1);  // first chunk only: scan from lo
    for (int x = lo; x <= x1; ++x)
      if (B[x] == 0.0) return x;
  }
  return INT_MAX;
}

// Final entries of the flat windows i (pinned during the sweep), for the band of diagonals
// [k_lo, k_hi) (k_lo >= exclusion): the smallest flat f with |i - f| in the band scores the
// minimum (distance 0); without one, every admissible partner scores d = 1 (distance sqrt(2m))
// and the smallest admissible index wins the tie; without any admissible partner: (+inf, -1).
__global__ void k_flat_fix(const double* __restrict__ B, int L, int k_lo, int k_hi,
                           const int* __restrict__ cmin, BestEntry* best) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    if (B[i] != 0.0) continue;
    int f = first_flat(B, cmin, max(0, i - k_hi + 1), i - k_lo);
    if (f == INT_MAX) f = first_flat(B, cmin, i + k_lo, min(L - 1, i + k_hi - 1));
    if (f != INT_MAX) {
      best[i] = BestEntry{0ull, static_cast<long long>(f)};
      continue;
    }
    int j = INT_MAX;
    if (i - k_lo >= 0 && max(0, i - k_hi + 1) <= i - k_lo) j = max(0, i - k_hi + 1);
    else if (i + k_lo <= L - 1) j = i + k_lo;
    const unsigned long long one = static_cast<unsigned long long>(__double_as_longlong(1.0));
    best[i] = (j == INT_MAX) ? BestEntry{kInfBits, kNoIdx} : BestEntry{one, static_cast<long long>(j)};
  }
}

// ---- brute-force profile (the reference's oracle, /root/reference/proj/src/oracle.cpp:51-132) --
// Direct distances with the reference's evaluation order (no contraction), the smallest j
// winning ties. O(L^2 m): a checker and the CLI's `--engine oracle`, not the hot path.
__global__ void k_moments(const double* __restrict__ t, int L, int m, double* __restrict__ mean,
                          double* __restrict__ var) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L; p += gridDim.x * blockDim.x) {
    double sum = 0.0, sumsq = 0.0;  // oracle.cpp:35-47
    for (int l = 0; l < m; ++l) {
      const double v = t[p + l];
      sum = __dadd_rn(sum, v);
      sumsq = __dadd_rn(sumsq, __dmul_rn(v, v));
    }
    const double mu = __ddiv_rn(sum, (double)m);
    double vv = __dsub_rn(__ddiv_rn(sumsq, (double)m), __dmul_rn(mu, mu));
    if (vv < 0.0) vv = 0.0;
    mean[p] = mu;
    var[p] = vv;
  }
}

__device__ __forceinline__ double bf_abs_pow(double x, double p) {  // oracle.cpp:17-24
  const double a = fabs(x);
  if (p == 1.0) return a;
  if (p == 2.0) return __dmul_rn(a, a);
  if (p == 3.0) return __dmul_rn(__dmul_rn(a, a), a);
  if (p == 4.0) return __dmul_rn(__dmul_rn(a, a), __dmul_rn(a, a));
  return pow(a, p);
}

__device__ double bf_dist(const double* __restrict__ t, int i, int j, int m, int family, double p,
                          double flat, const double* __restrict__ mean,
                          const double* __restrict__ var) {
  double sum = 0.0;
  if (family == MPROF_EUCLIDEAN) {
    for (int l = 0; l < m; ++l) {
      const double d = __dsub_rn(t[i + l], t[j + l]);
      sum = __dadd_rn(sum, __dmul_rn(d, d));
    }
    return sqrt(sum);
  }
  if (family == MPROF_PNORM) {
    for (int l = 0; l < m; ++l) sum = __dadd_rn(sum, bf_abs_pow(__dsub_rn(t[i + l], t[j + l]), p));
    return pow(sum, 1.0 / p);
  }
  const double va = var[i], vb = var[j];
  const bool fa = va <= flat, fb = vb <= flat;
  if (fa && fb) return 0.0;
  if (fa || fb) return sqrt(2.0 * (double)m);
  const double ma = mean[i], mb = mean[j];
  const double ia = __ddiv_rn(1.0, sqrt(va)), ib = __ddiv_rn(1.0, sqrt(vb));
  for (int l = 0; l < m; ++l) {
    const double d = __dsub_rn(__dmul_rn(__dsub_rn(t[i + l], ma), ia), __dmul_rn(__dsub_rn(t[j + l], mb), ib));
    sum = __dadd_rn(sum, __dmul_rn(d, d));
  }
  return sqrt(sum);
}

// one CTA per row i; lexicographic (distance, j) minimum over admissible j
// rows == nullptr: every row i < L into P[i], I[i]; else row rows[r] into P[r], I[r], r < nrows.
__global__ void k_brute(const double* __restrict__ t, int L, int m, int excl, int family, double p,
                        double flat, const double* __restrict__ mean,
                        const double* __restrict__ var, double* __restrict__ P,
                        int64_t* __restrict__ I, const int64_t* __restrict__ rows, int nrows) {
  __shared__ double sv[32];
  __shared__ int sj[32];
  const int nout = rows ? nrows : L;
  for (int r = blockIdx.x; r < nout; r += gridDim.x) {
    const int i = rows ? (int)rows[r] : r;
    double bv = INFINITY;
    int bj = INT_MAX;
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
      if (abs(i - j) < excl) continue;
      const double d = bf_dist(t, i, j, m, family, p, flat, mean, var);
      if (d < bv || (d == bv && j < bj)) { bv = d; bj = j; }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
      if (ov < bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
    }
    if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; sj[threadIdx.x >> 5] = bj; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (sv[w] < bv || (sv[w] == bv && sj[w] < bj)) { bv = sv[w]; bj = sj[w]; }
      P[r] = bj == INT_MAX ? INFINITY : bv;
      I[r] = bj == INT_MAX ? -1 : bj;
    }
    __syncthreads();
  }
}

// ---- streaming extension (build_engine_state / extend_profile) -----------------------------
// The stored profile of the first l_old windows seeds the extended sweep: entry i takes the
// lexicographic minimum with its stored (comparison value, neighbour); pinned flat windows (B = 0)
// keep their pin (k_flat_fix sets them at the end), untouched entries (-1) add nothing.
__global__ void k_seed_prev(BestEntry* __restrict__ best, const double* __restrict__ B,
                            const double* __restrict__ cmp_old, const int64_t* __restrict__ idx_old,
                            int l_old) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < l_old; i += gridDim.x * blockDim.x) {
    if ((B && B[i] == 0.0) || idx_old[i] < 0) continue;
    const BestEntry prev{static_cast<unsigned long long>(__double_as_longlong(cmp_old[i])), idx_old[i]};
    const BestEntry cur = best[i];
    if (lex_less(prev.v, prev.idx, cur.v, cur.idx)) best[i] = prev;
  }
}

// EngineState tail cursors: for completed diagonal k = excl + r, the window pair (pos, pos + k)
// at its last cell (pos = L - 1 - k, partner L - 1), evaluated directly by one warp:
// Euclidean / p-norm: the comparison-space accumulator (DiagonalCursor::acc, aamp.hpp:27-32);
// z-normalized: the five sums of DiagStats (acamp.hpp:12-20) into out[5r .. 5r+4].
__global__ void k_tail(const double* __restrict__ t, int L, int m, int excl, int count, int family,
                       double p, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < count; r += warps) {
    const int k = excl + r, i = L - 1 - k, j = L - 1;
    double a = 0.0, b = 0.0, aa = 0.0, bb = 0.0, ab = 0.0;
    for (int l = lane; l < m; l += 32) {
      const double x = t[i + l], y = t[j + l];
      if (family == MPROF_ZNORMALIZED) {
        a += x; b += y; aa = fma(x, x, aa); bb = fma(y, y, bb); ab = fma(x, y, ab);
      } else if (family == MPROF_EUCLIDEAN || p == 2.0) {
        a = fma(x - y, x - y, a);
      } else {
        const double d = fabs(x - y);
        a += p == 1.0 ? d : p == 3.0 ? d * d * d : p == 4.0 ? (d * d) * (d * d) : pow(d, p);
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, off);
      b += __shfl_xor_sync(0xffffffffu, b, off);
      aa += __shfl_xor_sync(0xffffffffu, aa, off);
      bb += __shfl_xor_sync(0xffffffffu, bb, off);
      ab += __shfl_xor_sync(0xffffffffu, ab, off);
    }
    if (lane == 0) {
      if (family == MPROF_ZNORMALIZED) {
        double* o = out + 5LL * r;
        o[0] = a; o[1] = b; o[2] = aa; o[3] = bb; o[4] = ab;
      } else {
        out[r] = a;
      }
    }
  }
}

// An empty partial profile (a band without diagonals): +inf / no neighbour.
__global__ void k_split_empty(double* __restrict__ cmp, int64_t* __restrict__ idx, int L) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    cmp[i] = INFINITY;
    idx[i] = -1;
  }
}

__global__ void k_split(const BestEntry* __restrict__ best, double* __restrict__ cmp,
                        int64_t* __restrict__ idx, int L) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    const BestEntry e = best[i];
    const bool none = e.v == kInfBits || e.idx == kNoIdx || e.idx < 0;
    cmp[i] = none ? __longlong_as_double(static_cast<long long>(kInfBits))
                  : __longlong_as_double(static_cast<long long>(e.v));
    idx[i] = none ? -1 : e.idx;
  }
}

// to_distance (/root/reference/proj/src/detail/diag_scan.hpp:153-167) and f_to_dz
// (/root/reference/proj/include/mprof/acamp.hpp:86-91) for the GPU comparison spaces.
// One warp per entry. In the default mode the distance of the chosen pair (i, idx[i]) is
// RECOMPUTED directly (O(m), two-pass z-normalization) instead of converting the running
// comparison value: the sweep decides the argmin, the reported value carries no sliding drift
// and near-duplicate z-normalized windows come out at ~1e-14 instead of sqrt(eps). Flat rules
// as f_value / dist_znorm (acamp.hpp:52-57, oracle.cpp:81-84). In the exact (parity) mode the
// reference's own conversion of the comparison value is applied.
// Warp-wide sum over l < m of |a[l] - b[l]|^PK (PK = 0: generic pow), every lane gets the sum.
template <int PK>
__device__ __forceinline__ double lane_lp_sum(const double* __restrict__ a, const double* __restrict__ b,
                                              int m, int lane, double p) {
  double s = 0.0;
#pragma unroll 4
  for (int l = lane; l < m; l += 32) {
    const double d = fabs(a[l] - b[l]);
    if constexpr (PK == 2) s = fma(d, d, s);
    else if constexpr (PK == 1) s += d;
    else if constexpr (PK == 3) s = fma(d * d, d, s);
    else if constexpr (PK == 4) { const double d2 = d * d; s = fma(d2, d2, s); }
    else s += pow(d, p);
  }
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

// Distance of entry i from its comparison value v and neighbour j, computed by one warp (every
// lane returns it).
__device__ __forceinline__ double finalize_entry(const double* __restrict__ t,
                                                 const double* __restrict__ mu,
                                                 const double* __restrict__ B, int i, double v,
                                                 long long j, int lane, int m, int family,
                                                 double p, int exact) {
    const double md = (double)m;
    double out;
    if (isinf(v) || j < 0) {
      out = v;
    } else if (exact) {
      if (family == MPROF_EUCLIDEAN) out = sqrt(v);
      else if (family == MPROF_PNORM) out = (p == 1.0) ? v : (p == 2.0) ? sqrt(v) : pow(v, 1.0 / p);
      else out = sqrt(fmax(0.0, fmin(2.0 * md * v, 4.0 * md)));
    } else if (family == MPROF_ZNORMALIZED) {
      const double bi = B[i], bj = B[j];
      if (bi == 0.0 || bj == 0.0) {
        out = (bi == 0.0 && bj == 0.0) ? 0.0 : sqrt(2.0 * md);
      } else {
        const double mi = mu[i], mj = mu[j];
        double s = 0.0;
#pragma unroll 4
        for (int l = lane; l < m; l += 32) {
          const double d = (t[i + l] - mi) * bi - (t[j + l] - mj) * bj;
          s = fma(d, d, s);
        }
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        out = sqrt(fmin(md * s, 4.0 * md));
      }
    } else {
      const bool l2 = family == MPROF_EUCLIDEAN || p == 2.0;
      const double s = l2         ? lane_lp_sum<2>(t + i, t + j, m, lane, p)
                       : p == 1.0 ? lane_lp_sum<1>(t + i, t + j, m, lane, p)
                       : p == 3.0 ? lane_lp_sum<3>(t + i, t + j, m, lane, p)
                       : p == 4.0 ? lane_lp_sum<4>(t + i, t + j, m, lane, p)
                                  : lane_lp_sum<0>(t + i, t + j, m, lane, p);
      out = l2 ? sqrt(s) : (p == 1.0) ? s : pow(s, 1.0 / p);
    }
    return out;
}

__global__ void k_finalize_range(const double* __restrict__ t, const double* __restrict__ cmp,
                                 const int64_t* __restrict__ idx, const double* __restrict__ mu,
                                 const double* __restrict__ B, double* __restrict__ P, int lo, int hi,
                                 int m, int family, double p, int exact) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < hi; i += warps) {
    const double out = finalize_entry(t, mu, B, i, cmp[i], idx[i], lane, m, family, p, exact);
    if (lane == 0) P[i] = out;
  }
}

// Fused multi-process merge + finalize + all-gather over peer memory (CUDA IPC / NVLink): one
// warp per entry i of [lo, hi); lane r < nin loads rank r's partial (cmp, idx)[i] (peer loads,
// in parallel), a warp shuffle takes the lexicographic (value, index) minimum (MinBuffer::absorb,
// /root/reference/proj/src/detail/diag_scan.hpp:45-52; the same rule as k_merge), the warp
// finalizes the entry, and lane r < nout stores (P, I)[i] into rank r's output buffers (peer
// stores). Replaces the two ncclMin all-reduces + the finalize + the all-gather.
struct PeerSet {
  const double* cmp[MPROF_MAX_PEERS];
  const int64_t* idx[MPROF_MAX_PEERS];
  double* P[MPROF_MAX_PEERS];
  int64_t* I[MPROF_MAX_PEERS];
  int nin, nout;
};

__global__ void k_merge_finalize_peers(const double* __restrict__ t, const PeerSet ps,
                                       const double* __restrict__ mu, const double* __restrict__ B,
                                       int lo, int hi, int m, int family, double p, int exact) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < hi; i += warps) {
    double v = __longlong_as_double(0x7FF0000000000000ll);  // +inf
    long long j = -1;
    if (lane < ps.nin) {
      v = ps.cmp[lane][i];
      j = ps.idx[lane][i];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, off);
      const long long oj = __shfl_xor_sync(0xffffffffu, j, off);
      // k_merge's rule, made symmetric so every lane ends with the same pair: smaller value,
      // then smaller index; an untouched entry (-1) loses to any index at an equal value
      const bool take = ov < v || (ov == v && (j < 0 || (oj >= 0 && oj < j)));
      if (take) {
        v = ov;
        j = oj;
      }
    }
    const double out = finalize_entry(t, mu, B, i, v, j, lane, m, family, p, exact);
    if (lane < ps.nout) {
      ps.P[lane][i] = out;
      ps.I[lane][i] = j;
    }
  }
}

__global__ void k_merge(double* __restrict__ cmp, int64_t* __restrict__ idx,
                        const double* __restrict__ ocmp, const int64_t* __restrict__ oidx, int L) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    const double a = cmp[i], b = ocmp[i];
    const int64_t ia = idx[i], ib = oidx[i];
    if (b < a || (b == a && ib < ia)) {
      cmp[i] = b;
      idx[i] = ib;
    }
  }
}

__global__ void k_dfma_peak(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999999, c = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains alive
}

int grid_for(long long work, int block = 256) {
  long long g = (work + block - 1) / block;
  return static_cast<int>(std::max(1LL, std::min(g, 148LL * 32)));
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// context

struct mprof_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool timing = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t side = nullptr;  // concurrent near-diagonal z-norm tiles
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int num_sms = 148;
  // grow-only device workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // host-API staging
  void* io = nullptr;
  size_t io_bytes = 0;
  // Tile table cache: a few tables (least recently used replaced), so callers alternating
  // between engines or series shapes on one context (AAMP then ACAMP of the same series, the
  // usual host-API pattern) neither rebuild and re-upload the table nor rerun the schedule model.
  struct TileSlot {
    // (first diagonal, first row, row end, diagonal end), arranged as [tiles of the global
    // block next to the exclusion zone | other legacy-kernel tiles | constant-row tiles by
    // (first row, first diagonal)]
    std::vector<int4> h;
    long long n_near = 0;             // side-kernel tiles (covariance forms)
    long long n_legacy = 0;           // tiles the legacy kernel sweeps, n_near included
    std::vector<mpg::RcBand> bands;   // row bands of the constant-row part (offsets into h)
    int4* d = nullptr;
    size_t cap = 0;
    long long key[10] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
    unsigned long long used = 0;
  };
  static constexpr int kTileSlots = 4;
  TileSlot tile_slot[kTileSlots];
  TileSlot* tiles = &tile_slot[0];  // the table of the current sweep
  unsigned long long tile_clock = 0;
  struct RChoice {  // rows-per-tile choice cache
    long long key[9];
    long long R;
  };
  std::vector<RChoice> R_cache;
  // constant-row sweep (sweep_rc.h): streams, events, accumulator carry; on by default
  mpg::RcRes rc;
  bool rowconst = true;
  // pinned host copy of the operand pairs the window launches pass as kernel parameters, valid
  // for operand generation rc_host_gen of device array rc_host_src (prepare_operands bumps op_gen)
  void* rc_host = nullptr;
  size_t rc_host_cap = 0;          // bytes
  const void* rc_host_src = nullptr;
  unsigned long long rc_host_gen = 0, op_gen = 1;
  // z-norm statistics currently held in the workspace (series pointer, n, m, threshold)
  const double* stats_t = nullptr;
  uint64_t stats_n = 0, stats_m = 0;
  double stats_thr = -1.0;
  bool zn_colscale = false;  // z-norm filter form chosen for the current sweep
  bool aamp_cov = false;     // AAMP form chosen for the current sweep (covariance vs delta-sigma)
  bool wide = false;         // covariance-only policy with longer hit groups (probe: no replays)
  bool dense = false;        // Dense<P>: no block filter (noise-like series, plan_series)
  unsigned int* noise_cnt = nullptr;  // noise test counter
  double* d_spread = nullptr;
  int4* probe_d = nullptr;                 // AAMP form probe: tile list and replay counter
  unsigned long long* probe_cnt = nullptr;
  mprof_progress_fn progress = nullptr;  // anytime observer (band granularity)
  void* progress_user = nullptr;
  int form = MPROF_FORM_AUTO;             // filter-form override (mprof_ctx_set_form)
  long long plan_R = 0;                   // rows per tile of the last planned series
  unsigned long long probe_replays = 0;   // last form probe: replayed blocks / sample cells
  double probe_cells = 0.0;
  double noise_frac = -1.0;               // last noise test: fraction of random pairs passing
};

// Device-resident EngineState: the series, the comparison-space profile and scratch.
struct mprof_state {
  mprof_ctx* ctx = nullptr;  // owned: the state's own stream and workspace (any thread may use it)
  mprof_config cfg;
  uint64_t n = 0;
  double* t = nullptr;       // series (device)
  size_t t_bytes = 0;
  double* cmp = nullptr;     // comparison values [L]
  size_t cmp_bytes = 0;
  int64_t* idx = nullptr;    // neighbours [L]
  size_t idx_bytes = 0;
  double* P = nullptr;       // finalized distances scratch [L]
  size_t P_bytes = 0;
  uint64_t done = 0;         // completed diagonals, ascending from cfg.exclusion (build may cancel)
  long long plan_R = 0;      // the profile's sweep plan: rows per tile and kernel forms
  int plan_flags = 0;
};

// A planned band sweep of one series (mprof_plan_create): the per-series decisions, the prepared
// operands and the band's tile table, so that mprof_plan_sweep only enqueues kernels.
struct mprof_plan {
  mprof_ctx* ctx = nullptr;  // borrowed: must outlive every mprof_plan_sweep (not the destroy)
  int device = 0;
  const double* t = nullptr;
  uint64_t n = 0;
  mprof_config cfg;
  long long k_lo = 0, k_hi = 0;  // admissible band
  void* ws = nullptr;            // owned workspace (operands, profile, scratch)
  int4* tiles = nullptr;         // owned tile table
  long long ntiles = 0, n_near = 0, n_legacy = 0, R = 0;
  std::vector<mpg::RcBand> bands;  // constant-row part of the tile table
  int rc_policy = -1;
  void* host_pairs = nullptr;      // owned pinned mirror of the operand pairs (constant-row sweep)
  mpg::RcGraph rc_graph;           // the captured window chain
  bool aamp_cov = false, zn_colscale = false, wide = false, dense = false;
  unsigned long long probe_replays = 0;
  double probe_cells = 0.0;
};

namespace {

int32_t ensure(void** p, size_t* have, size_t need) {
  if (*have >= need) return MPROF_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  CK(cudaMalloc(p, need));
  *have = need;
  return MPROF_OK;
}

// Default contexts (ctx == NULL): one per device and calling thread, destroyed when the thread
// exits, so a thread pool does not leak workspaces and no two threads share a workspace.
struct DefaultContexts {
  std::unordered_map<int, mprof_ctx*> by_device;
  ~DefaultContexts();
};
thread_local DefaultContexts g_default_ctx;

int32_t resolve_ctx(mprof_ctx* in, mprof_ctx** out) {
  if (in) {
    CK(cudaSetDevice(in->device));
    *out = in;
    return MPROF_OK;
  }
  int dev = 0;
  CK(cudaGetDevice(&dev));
  auto it = g_default_ctx.by_device.find(dev);
  if (it != g_default_ctx.by_device.end()) {
    *out = it->second;
    return MPROF_OK;
  }
  mprof_ctx* c = nullptr;
  const int32_t st = mprof_ctx_create(dev, &c);
  if (st != MPROF_OK) return st;
  g_default_ctx.by_device[dev] = c;
  *out = c;
  return MPROF_OK;
}

DefaultContexts::~DefaultContexts() {
  // The main thread's thread-locals are destroyed while the process exits, when the CUDA runtime
  // (or the embedding interpreter's) may already be tearing down: leave those to the driver.
  if (static_cast<long>(syscall(SYS_gettid)) == static_cast<long>(getpid())) {
    by_device.clear();
    return;
  }
  // mprof_ctx_destroy erases its entry: take the contexts out first
  std::vector<mprof_ctx*> cs;
  for (auto& kv : by_device) cs.push_back(kv.second);
  by_device.clear();
  for (mprof_ctx* c : cs) mprof_ctx_destroy(c);
}

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// A state's own context: same device and form override as the context it derives from.
int32_t state_ctx(const mprof_ctx* from, mprof_ctx** out) {
  const int32_t st = mprof_ctx_create(from->device, out);
  if (st != MPROF_OK) return st;
  (*out)->form = from->form;
  return MPROF_OK;
}

// Releases a context's transient device memory (states keep only series + profile between calls).
void trim_ctx(mprof_ctx* c) {
  cudaStreamSynchronize(c->stream);
  cudaFree(c->ws);
  cudaFree(c->io);
  for (auto& sl : c->tile_slot) {
    cudaFree(sl.d);
    sl.d = nullptr;
    sl.cap = 0;
    std::fill(sl.key, sl.key + 10, -1LL);
    std::vector<int4>().swap(sl.h);
  }
  mpg::rc_release(c->rc);
  if (c->rc_host) cudaFreeHost(c->rc_host);
  c->rc_host = nullptr;
  c->rc_host_cap = 0;
  c->rc_host_src = nullptr;
  c->ws = c->io = nullptr;
  c->ws_bytes = c->io_bytes = 0;
  c->stats_t = nullptr;
}

// Diagonals of a complete state: [exclusion, n - m] (engine_state.hpp:37-39).
uint64_t state_total(const mprof_state* S) { return S->n - S->cfg.m - S->cfg.exclusion + 1; }

struct Workspace {
  double2* A;
  double* B;
  double* mu;
  BestEntry* best;
  int* cmin;
  float2* A32;
  float* B32;
  double* scalars;  // [0] series mean (FP32 offset)
  double* cv;       // first-diagonal cell values (prepass scratch)
  // covariance-form AAMP (own arrays: the z-norm statistics above are cached per series)
  double2* A2;      // (df, dg) operand pairs
  double* emu;      // window means
  double* S;        // centred sums of squares
  float2* SB;       // ring scalars {S rd, mu - t[0] rd}
};

size_t workspace_bytes(int L) {
  const size_t nA = align_up(sizeof(double2) * (size_t)L);
  const size_t nB = align_up(sizeof(double) * (size_t)L);
  const size_t nBest = align_up(sizeof(BestEntry) * (size_t)L);
  const size_t nC = align_up(sizeof(int) * ((size_t)L / kChunk + 2));
  const size_t nA32 = align_up(sizeof(float2) * (size_t)L);
  const size_t nB32 = align_up(sizeof(float) * (size_t)L);
  const size_t nS = align_up(8 * sizeof(double));
  return nA + 3 * nB + nBest + nC + nA32 + nB32 + nS + nA + 2 * nB + nA32;
}

// The workspace arrays of a profile of length L laid out from `base` (workspace_bytes(L) bytes).
void carve_at(char* base, int L, Workspace* w) {
  const size_t nA = align_up(sizeof(double2) * (size_t)L);
  const size_t nB = align_up(sizeof(double) * (size_t)L);
  const size_t nBest = align_up(sizeof(BestEntry) * (size_t)L);
  const size_t nC = align_up(sizeof(int) * ((size_t)L / kChunk + 2));
  const size_t nA32 = align_up(sizeof(float2) * (size_t)L);
  const size_t nB32 = align_up(sizeof(float) * (size_t)L);
  const size_t nS = align_up(8 * sizeof(double));
  w->A = reinterpret_cast<double2*>(base);
  w->B = reinterpret_cast<double*>(base + nA);
  w->mu = reinterpret_cast<double*>(base + nA + nB);
  w->best = reinterpret_cast<BestEntry*>(base + nA + 2 * nB);
  w->cmin = reinterpret_cast<int*>(base + nA + 2 * nB + nBest);
  w->A32 = reinterpret_cast<float2*>(base + nA + 2 * nB + nBest + nC);
  w->B32 = reinterpret_cast<float*>(base + nA + 2 * nB + nBest + nC + nA32);
  w->scalars = reinterpret_cast<double*>(base + nA + 2 * nB + nBest + nC + nA32 + nB32);
  w->cv = reinterpret_cast<double*>(base + nA + 2 * nB + nBest + nC + nA32 + nB32 + nS);
  char* e = base + nA + 3 * nB + nBest + nC + nA32 + nB32 + nS;
  w->A2 = reinterpret_cast<double2*>(e);
  w->emu = reinterpret_cast<double*>(e + nA);
  w->S = reinterpret_cast<double*>(e + nA + nB);
  w->SB = reinterpret_cast<float2*>(e + nA + 2 * nB);
}

// The context's grow-only workspace, carved for a profile of length L.
int32_t carve(mprof_ctx* c, int L, Workspace* w) {
  const int32_t st = ensure(&c->ws, &c->ws_bytes, workspace_bytes(L));
  if (st != MPROF_OK) return st;
  carve_at(static_cast<char*>(c->ws), L, w);
  return MPROF_OK;
}

int32_t ensure_znorm_stats(mprof_ctx* c, const double* d_t, uint64_t n, const mprof_config* cfg,
                           const Workspace& w) {
  if (c->stats_t == d_t && c->stats_n == n && c->stats_m == cfg->m &&
      c->stats_thr == cfg->flat_threshold)
    return MPROF_OK;
  const int L = (int)(n - cfg->m + 1);
  k_znorm_stats<<<ws_grid(L), kWsT, 0, c->stream>>>(d_t, L, (int)cfg->m, cfg->flat_threshold, w.mu, w.B);
  CK(cudaGetLastError());
  c->stats_t = d_t;
  c->stats_n = n;
  c->stats_m = cfg->m;
  c->stats_thr = cfg->flat_threshold;
  return MPROF_OK;
}

// Profile length rounded up to 1/8 of its octave: the per-series plan (choose_R, probe_form) is
// taken on it, so it does not change when a series grows a little.
long long quantize_len(long long L) {
  if (L <= 64) return L;
  const int e = 63 - __builtin_clzll((unsigned long long)L);
  const long long q = 1LL << (e - 3);
  return (L + q - 1) / q * q;
}

// ---- tile geometry -----------------------------------------------------------------------------
// Diagonals are cut into GLOBAL blocks of kK: [g0 + q kK, g0 + (q + 1) kK) ∩ [g0, L), with g0 the
// first tile diagonal of a full sweep (exclusion + 1 in the fast mode, whose first-diagonal
// prepass evaluates diagonal `exclusion`; exclusion in the exact mode). A band or an anytime chunk
// sweeps the part of each global block it holds, and every diagonal k is seeded at the rows of one
// grid that depends on the series only (rows per tile R from choose_R, shortened only for the
// final narrow global block), so the arithmetic of every cell -- and therefore the profile, ties
// included -- does not depend on how the diagonals are split across GPUs or chunks
// (the reference: bit-identical for any thread count, tests/test_aamp.cpp:262-274).
struct Grid {
  long long L, g0, row_hi;  // profile length, grid origin, rows swept ([0, row_hi))
  bool exact;
  int m, S;                 // window, rows per shared-memory stage of the sweep policy
  long long block_lo(long long k) const { return g0 + (k - g0) / kK * kK; }
  long long block_hi(long long k) const { return std::min(L, block_lo(k) + kK); }
};

// Rows per tile of a global block w < kK diagonals wide (the final one): a narrow tile is
// latency-bound per row (a thin tile of R rows costs ~3/4 of a full one), so its rows shrink with
// its width. Exact mode keeps R: runs are seeded at multiples of refresh_interval.
long long block_R(long long R, long long w, bool exact, int S) {
  if (exact || w >= kK) return R;
  return std::min(R, std::max<long long>(2 * S, (R * w / kK + S - 1) / S * S));
}

// Calls f(kb, ke, Rb) for every tile column: the part [kb, ke) of a global block inside the band
// [k_lo, k_hi), with the block's rows per tile.
template <class F>
void for_columns(const Grid& g, long long k_lo, long long k_hi, long long R, F&& f) {
  for (long long kb = k_lo; kb < k_hi;) {
    const long long ke = std::min(k_hi, g.block_hi(kb));
    f(kb, ke, block_R(R, g.block_hi(kb) - g.block_lo(kb), g.exact, g.S));
    kb = ke;
  }
}

long long count_tiles(const Grid& g, long long k_lo, long long k_hi, long long R) {
  long long t = 0;
  for_columns(g, k_lo, k_hi, R, [&](long long kb, long long, long long Rb) {
    t += (std::min<long long>(g.L - kb, g.row_hi) + Rb - 1) / Rb;
  });
  return t;
}

// Cells of the tile (diagonals [k0, k1), rows [ra, min(ra + R, row_hi)); diagonal k ends at row
// L - k): sum over k of clamp(min(A, B - k), 0), A = rows cap, B = L - ra.
double tile_cells(long long L, long long k0, long long k1, long long row_hi, long long ra, long long R) {
  const long long A = std::min(R, row_hi - ra), B = L - ra;
  if (A <= 0 || k0 >= k1) return 0.0;
  const long long kf = std::clamp(B - A, k0, k1);  // k < kf: full A rows
  const long long ke = std::clamp(B, k0, k1);      // kf <= k < ke: B - k rows
  const double full = (double)(kf - k0) * (double)A;
  const double tri = (double)(ke - kf) * (double)B - 0.5 * (double)(ke - 1 + kf) * (double)(ke - kf);
  return full + tri;
}

// The tile table of band [k_lo, k_hi) in launch order, int4 {first diagonal, first row, row end,
// diagonal end}, with each tile's modelled cost (row-steps of a full-width tile: cells / K, with a
// per-row latency floor of a quarter row-step for narrow tiles, plus the FP64 seeds, m per
// diagonal ~ 1/3 row-step each in FP64-pipe terms, and pipeline fill), in diagonal order; the
// columns of the global block next to the exclusion zone come first (they may run on the
// near-diagonal side stream, dispatch_sweep). Longest-first ordering of the partial tiles was
// measured: +1 % on C4 AAMP, -11 % on C3 (MPROF_TILE_ORDER_LPT keeps it for experiments).
// l_old > 0 (an EngineState extension from profile length l_old): only the tiles that hold a cell
// (i, i + k) with i + k >= l_old, i.e. a new window (row end re, column end ke: re + ke - 2 >=
// l_old); they are the fresh sweep's own tiles, so every cell keeps its fresh-sweep arithmetic.
void tile_list(const Grid& g, long long k_lo, long long k_hi, long long R, std::vector<int4>& tiles,
               std::vector<double>* costs, long long l_old = 0) {
  tiles.clear();
  std::vector<double> cost;
  const double fixed = (double)g.m / 3.0 + 2.0 * g.S;
  size_t first_block = 0;
  for_columns(g, k_lo, k_hi, R, [&](long long kb, long long ke, long long Rb) {
    const long long rend = std::min<long long>(g.L - kb, g.row_hi);
    for (long long ra = 0; ra < rend; ra += Rb) {
      const long long re = std::min(ra + Rb, rend);
      if (l_old > 0 && re + ke - 2 < l_old) continue;
      tiles.push_back(make_int4((int)kb, (int)ra, (int)re, (int)ke));
      const double cells = tile_cells(g.L, kb, ke, g.row_hi, ra, Rb);
      cost.push_back(std::max(cells / kK, cells / (double)(ke - kb) * 0.25) + fixed);
    }
    if (kb == k_lo) first_block = tiles.size();
  });
  if (knobs().tile_order_lpt) {  // experiments: decreasing cost after the first block
    std::vector<size_t> ord(tiles.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
    std::stable_sort(ord.begin() + first_block, ord.end(),
                     [&](size_t x, size_t y) { return cost[x] > cost[y]; });
    std::vector<int4> sorted(tiles.size());
    std::vector<double> sorted_cost(tiles.size());
    for (size_t i = 0; i < ord.size(); ++i) {
      sorted[i] = tiles[ord[i]];
      sorted_cost[i] = cost[ord[i]];
    }
    tiles.swap(sorted);
    cost.swap(sorted_cost);
  }
  if (costs) costs->swap(cost);
}

// Makespan (in row-steps of a full-width tile) of the band's tile list in launch order on `slots`
// resident CTAs: the block scheduler hands the next tile to the first free slot (list scheduling).
double schedule_makespan(const Grid& g, long long k_lo, long long k_hi, long long R, int slots) {
  std::vector<int4> tiles;
  std::vector<double> cost;
  tile_list(g, k_lo, k_hi, R, tiles, &cost);
  std::vector<double> heap(slots, 0.0);  // min-heap of slot free times
  auto cmp = std::greater<double>();
  double makespan = 0.0;
  for (double c : cost) {
    std::pop_heap(heap.begin(), heap.end(), cmp);
    heap.back() += c;
    makespan = std::max(makespan, heap.back());
    std::push_heap(heap.begin(), heap.end(), cmp);
  }
  return makespan;
}

// Rows per tile of a series (one value for every band, chunk and GPU count: see Grid). Exact mode
// aligns runs to refresh_interval (the reference's refresh points, diag_scan.hpp:97-104) or runs
// whole diagonals. Fast mode: the longest runs amortise the seeds best (R_max = 32 m rows, seeds
// <= ~1.6 % of the FP64 work), but a grid of a few waves loses up to a whole wave to its tail.
// Grids that still hold >= 16 waves of resident CTAs when split into kPlanBands equal-area bands
// keep R_max; otherwise the candidates R_max / j (stage multiples) are list-scheduled on the
// kernel's real residency (slots = occupancy x SMs) both for the whole sweep on one GPU (M1) and
// for the slowest of kPlanBands bands (M8), and the candidate with the smallest M8 among those
// within 1 % of the best M1 wins (ties -> longer tiles). The model runs on the profile length
// rounded up to 1/8 of its octave, so a series that grows a little (an EngineState extension)
// keeps its R and is extended incrementally. Cached per context and shape.
constexpr int kPlanBands = 8;
long long choose_R(const mprof_config* cfg, const Grid& gx, int slots) {
  Grid g = gx;
  if (!cfg->exact && g.row_hi == g.L) g.L = g.row_hi = quantize_len(g.L);
  if (cfg->exact) {
    if (cfg->refresh_interval > 0) return (long long)cfg->refresh_interval;
    return g.L;  // the whole diagonal is one run, like the reference's refresh = 0
  }
  const int S = g.S;
  long long Rmax = std::max<long long>(32LL * (long long)cfg->m, 8LL * S);
  Rmax = (Rmax + S - 1) / S * S;
  if (cfg->refresh_interval > 0) Rmax = std::min<long long>(Rmax, (long long)cfg->refresh_interval);
  if (knobs().rows_per_tile) return knobs().rows_per_tile;  // experiments
  const long long k_lo = g.g0, k_hi = g.L;
  if (k_lo >= k_hi || Rmax <= 2 * S ||
      count_tiles(g, k_lo, k_hi, Rmax) >= 16LL * kPlanBands * slots)
    return Rmax;
  std::vector<uint64_t> cuts(kPlanBands + 1);
  const uint64_t n = (uint64_t)(g.L + g.m - 1);
  if (mprof_band_cuts(n, (uint64_t)g.m, (uint64_t)cfg->exclusion, kPlanBands, cuts.data()) != MPROF_OK)
    return Rmax;
  struct Cand { long long R; double m1, m8; };
  std::vector<Cand> cand;
  long long prev = 0;
  for (int j = 1; j <= 32; ++j) {
    const long long Rj = j == 1 ? Rmax : std::max<long long>(2 * S, (Rmax / j + S - 1) / S * S);
    if (prev && Rj >= prev) continue;
    prev = Rj;
    if (j > 1 && count_tiles(g, k_lo, k_hi, Rj) > 32LL * kPlanBands * slots) break;
    Cand c{Rj, schedule_makespan(g, k_lo, k_hi, Rj, slots), 0.0};
    for (int b = 0; b < kPlanBands; ++b) {
      const long long a = std::max<long long>((long long)cuts[b], k_lo), z = (long long)cuts[b + 1];
      if (a < z) c.m8 = std::max(c.m8, schedule_makespan(g, a, z, Rj, slots));
    }
    if (knobs().tile_debug)
      fprintf(stderr, "[mprof tiles] slots %d R %lld tiles %lld M1 %.0f M8 %.0f\n", slots, Rj,
              count_tiles(g, k_lo, k_hi, Rj), c.m1, c.m8);
    cand.push_back(c);
    if (Rj == 2 * S) break;
  }
  double best_m1 = cand[0].m1;
  for (const Cand& c : cand) best_m1 = std::min(best_m1, c.m1);
  long long R = Rmax;
  double best_m8 = INFINITY;
  for (const Cand& c : cand)  // descending R: a later candidate must be strictly better
    if (c.m1 <= best_m1 * 1.01 && c.m8 < best_m8 * (1.0 - 1e-3)) {
      best_m8 = c.m8;
      R = c.R;
    }
  return R;
}

// Arranges a tile list (tile_list order: ascending first diagonal, then first row) for the sweep:
// the tiles of the global block next to the exclusion zone first (n_near; the covariance forms
// sweep them with their side kernel), and, for a constant-row sweep (rc), the full-width global
// blocks' tiles last, sorted by (first row, first diagonal) and described as row bands: all tiles
// of a band start at the same row, their row ends do not increase with the diagonal, so the tiles
// that still have a row transition in window w are a prefix of count[w] tiles.
void arrange_tiles(const Grid& g, bool near_block, bool rc, std::vector<int4>& h, long long* n_near,
                   long long* n_legacy, std::vector<mpg::RcBand>* bands) {
  *n_near = 0;
  if (near_block)
    while (*n_near < (long long)h.size() && h[*n_near].x < g.g0 + kK) ++*n_near;
  *n_legacy = (long long)h.size();
  bands->clear();
  if (!rc) return;
  auto full_width = [&](const int4& t) { return g.block_hi(t.x) - g.block_lo(t.x) == kK; };
  auto mid = std::stable_partition(h.begin() + *n_near, h.end(),
                                   [&](const int4& t) { return !full_width(t); });
  *n_legacy = mid - h.begin();
  std::sort(mid, h.end(), [](const int4& a, const int4& b) {
    return a.y != b.y ? a.y < b.y : a.x < b.x;
  });
  for (size_t i = (size_t)*n_legacy; i < h.size();) {
    size_t j = i;
    while (j < h.size() && h[j].y == h[i].y) ++j;
    mpg::RcBand bd;
    bd.off = (int)i;
    bd.ra = h[i].y;
    bd.count.push_back((int)(j - i));  // window 0: every tile seeds (and merges its seed cells)
    for (int w = 1;; ++w) {
      const long long r0 = (long long)bd.ra + (long long)w * mpg::kRcW;
      size_t cnt = 0;
      while (i + cnt < j && (long long)h[i + cnt].z - 1 > r0) ++cnt;
      if (cnt == 0) break;
      bd.count.push_back((int)cnt);
    }
    bands->push_back(std::move(bd));
    i = j;
  }
}

int32_t build_tiles(mprof_ctx* c, const Grid& g, long long k_lo, long long k_hi, long long R,
                    long long l_old, bool near_block, bool rc, long long* ntiles) {
  const long long key[10] = {g.L, k_lo, k_hi, R, g.exact ? -g.g0 : g.g0, g.row_hi, g.m, g.S, l_old,
                             (near_block ? 1 : 0) | (rc ? 2 : 0)};
  mprof_ctx::TileSlot* lru = &c->tile_slot[0];
  for (auto& sl : c->tile_slot) {
    if (std::equal(key, key + 10, sl.key)) {
      sl.used = ++c->tile_clock;
      c->tiles = &sl;
      *ntiles = (long long)sl.h.size();
      return MPROF_OK;
    }
    if (sl.used < lru->used) lru = &sl;
  }
  // replace the least recently used table (stream-ordered upload: kernels still reading the old
  // table of this slot were enqueued earlier on the same stream; ensure()'s cudaFree synchronizes)
  mprof_ctx::TileSlot& sl = *lru;
  std::fill(sl.key, sl.key + 10, -1LL);
  tile_list(g, k_lo, k_hi, R, sl.h, nullptr, l_old);
  arrange_tiles(g, near_block, rc, sl.h, &sl.n_near, &sl.n_legacy, &sl.bands);
  const size_t need = sl.h.size() * sizeof(int4);
  void* p = sl.d;
  int32_t st = ensure(&p, &sl.cap, std::max<size_t>(need, 16));
  sl.d = static_cast<int4*>(p);
  if (st != MPROF_OK) return st;
  CK(cudaMemcpyAsync(sl.d, sl.h.data(), need, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));  // the pageable host table may be rebuilt by a later call
  std::copy(key, key + 10, sl.key);
  sl.used = ++c->tile_clock;
  c->tiles = &sl;
  *ntiles = (long long)sl.h.size();
  return MPROF_OK;
}

// __launch_bounds__ minimum CTAs per SM: the policy's own choice if it has one, else the build's.
template <class P>
constexpr int min_blocks() {
  if constexpr (requires { P::kMinWarps; }) return std::max(1, P::kMinWarps * 32 / kT);
  else return MPROF_MIN_BLOCKS;
}

// Thresholds from diagonal k1 (FP64 direct evaluation), before the tiles.
template <class P>
int32_t launch_first_diag(mprof_ctx* c, const SweepParams& prm, int k1, uint32_t* launches) {
  if (k1 > prm.L - 1) return MPROF_OK;
  k_first_diag<P><<<grid_for((prm.L - k1 + 15) / 16, 128), 128, 0, c->stream>>>(prm, k1);  // >= 1 warp per 32 runs
  k_first_diag_cols<<<grid_for(prm.L - k1), 256, 0, c->stream>>>(prm, k1);
  CK(cudaGetLastError());
  *launches += 2;
  return MPROF_OK;
}

// Rows per shared-memory stage of the policy's kernel: the policy's own choice if it has one,
// else the build's (longer stages halve the per-stage barrier/threshold-refresh overhead; only
// the policies where that measured faster ask for them).
template <class P>
constexpr int stage_rows() {
  if constexpr (requires { P::kStageRows; }) return P::kStageRows;
  else return kS;
}

// Tiles [t0, t0 + nt) of the tile table on stream s.
template <class P>
int32_t launch_tiles(SweepParams prm, long long t0, long long nt, cudaStream_t s, uint32_t* launches) {
  if (nt <= 0) return MPROF_OK;
  constexpr int S = stage_rows<P>();
  using SM = SweepSmem<P, kD, kT, S>;
  const size_t smem = sizeof(SM);
  auto kern = sweep_kernel<P, kD, kT, S, min_blocks<P>()>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  prm.tiles += t0;
  kern<<<(unsigned)nt, kT, smem, s>>>(prm);
  CK(cudaGetLastError());
  ++*launches;
  return MPROF_OK;
}

// Calls f.template operator()<P>() with the sweep policy of (precision, family, p, exact, filter).
template <class F>
int32_t with_policy(const mprof_ctx* c, const mprof_config* cfg, F&& f) {
  const double p = cfg->p;
  const bool l2 = cfg->family == MPROF_EUCLIDEAN || (cfg->family == MPROF_PNORM && p == 2.0);
  if (cfg->precision == MPROF_FP32) {
    if (cfg->family == MPROF_ZNORMALIZED)
      return c->zn_colscale ? f.template operator()<ZnormF32<true>>()
                            : f.template operator()<ZnormF32<false>>();
    if (l2) return f.template operator()<EuclidF32>();
    if (p == 1.0) return f.template operator()<PnormF32<1>>();
    if (p == 3.0) return f.template operator()<PnormF32<3>>();
    if (p == 4.0) return f.template operator()<PnormF32<4>>();
    return f.template operator()<PnormF32<0>>();
  }
  const bool ex0 = cfg->exact != 0;
  if (c->dense && !ex0) {  // noise-like series: no block filter (plan_series)
    if (cfg->family == MPROF_ZNORMALIZED) return f.template operator()<Dense<Znorm<true>>>();
    if (l2) return f.template operator()<Dense<Euclid<false>>>();
    if (p == 1.0) return f.template operator()<Dense<Pnorm<1, false>>>();
    if (p == 3.0) return f.template operator()<Dense<Pnorm<3, false>>>();
  }
  if (cfg->family == MPROF_ZNORMALIZED) {
    if (c->zn_colscale) return f.template operator()<Znorm<true>>();
    return c->wide ? f.template operator()<Wide<Znorm<false>>>() : f.template operator()<Znorm<false>>();
  }
  const bool ex = cfg->exact != 0;
  if (l2 && !ex && c->aamp_cov)
    return c->wide ? f.template operator()<Wide<EuclidCov>>() : f.template operator()<EuclidCov>();
  if (l2) return ex ? f.template operator()<Euclid<true>>() : f.template operator()<Euclid<false>>();
  if (p == 1.0) return ex ? f.template operator()<Pnorm<1, true>>() : f.template operator()<Pnorm<1, false>>();
  if (p == 3.0) return ex ? f.template operator()<Pnorm<3, true>>() : f.template operator()<Pnorm<3, false>>();
  if (p == 4.0) return ex ? f.template operator()<Pnorm<4, true>>() : f.template operator()<Pnorm<4, false>>();
  if (ex) return f.template operator()<Pnorm<0, true>>();
  if (p == 1.5) return f.template operator()<Pnorm<-3, false>>();
  if (p == 2.5) return f.template operator()<Pnorm<-5, false>>();
  if (p == 3.5) return f.template operator()<Pnorm<-7, false>>();
  return f.template operator()<Pnorm<0, false>>();
}

// Side stream + fork/join events (created on first use).
int32_t ensure_side(mprof_ctx* c) {
  if (c->side) return MPROF_OK;
  CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  return MPROF_OK;
}

// The sweep of one tile table: optional first-diagonal prepass, then the tiles. Tiles
// [0, n_near) (the diagonal block next to the exclusion zone) run with the column-scaled z-norm
// filter on a side stream, concurrently with the rest: there correlations are ~1 and the
// covariance-only bound (block-wide 1/B extrema) passes nearly every block, whose replays
// would make those tiles the sweep's critical path.
// The covariance-form AAMP filter's block bound uses block extrema of S and mu; on series whose
// nearest-neighbour distances are small against that slack (near-periodic signals with a low
// noise floor) most blocks pass and replay, and the (delta, sigma) kernel is several times
// faster (C3's sinusoid at m = 1024: 53 vs 17 ms). The window-scale spread test cannot see that,
// so the choice is confirmed on the series itself: kProbeTiles short tiles spread over the
// band's diagonal blocks and rows are swept with the covariance kernel (after the first-diagonal
// pass, so the thresholds are the real ones) with a replay counter. The probe cells are genuine
// cells of the band (offers are exact minima, so sweeping them again later changes nothing).
// The sample's geometry is taken on the quantized profile length (quantize_len), so a series that
// grows a little (an EngineState extension) samples the same tiles and keeps its decision.
int32_t probe_form(mprof_ctx* c, bool zn, const SweepParams& prm, int kb_lo, uint32_t* launches) {
  const int L = prm.L, k_hi = prm.k_hi, row_hi = prm.row_hi;
  const long long Lq = quantize_len(L);
  const long long nblk = (Lq - kb_lo + kK - 1) / kK;
  if (nblk <= 0) return MPROF_OK;
  std::vector<int4> pt;
  double cells = 0.0;
  for (int q = 0; q < kProbeTiles; ++q) {
    const long long kb = kb_lo + kK * ((long long)q * nblk / kProbeTiles);
    const long long rend = std::min<long long>(L - kb, row_hi);
    if (kb >= k_hi || rend <= 0) continue;
    const long long span = std::max<long long>(1, Lq - kb - kProbeRows);
    const long long ra = (long long)(((unsigned long long)q * 2654435761ull) % (unsigned long long)span);
    if (ra >= rend) continue;
    const long long re = std::min<long long>(ra + kProbeRows, rend);
    pt.push_back(make_int4((int)kb, (int)ra, (int)re, (int)std::min<long long>(kb + kK, k_hi)));
    cells += (double)(re - ra) * (double)std::min<long long>(kK, k_hi - kb);
  }
  if (pt.empty() || cells <= 0.0) return MPROF_OK;
  if (!c->probe_d) CK(cudaMalloc(&c->probe_d, kProbeTiles * sizeof(int4)));
  if (!c->probe_cnt) CK(cudaMalloc(&c->probe_cnt, 2 * sizeof(unsigned long long)));
  CK(cudaMemcpyAsync(c->probe_d, pt.data(), pt.size() * sizeof(int4), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemsetAsync(c->probe_cnt, 0, 2 * sizeof(unsigned long long), c->stream));
  SweepParams pp = prm;
  pp.tiles = c->probe_d;
  pp.stats = c->probe_cnt;
  int32_t st = zn ? launch_tiles<Znorm<false>>(pp, 0, (long long)pt.size(), c->stream, launches)
                  : launch_tiles<EuclidCov>(pp, 0, (long long)pt.size(), c->stream, launches);
  if (st != MPROF_OK) return st;
  unsigned long long h[2];
  CK(cudaMemcpyAsync(h, c->probe_cnt, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->probe_replays = h[0];
  c->probe_cells = cells;
  const bool keep = (double)h[0] <= (zn ? kProbeMaxReplaysZ : kProbeMaxReplays) * cells;
  if (zn) c->zn_colscale = !keep;
  else c->aamp_cov = keep;
  c->wide = keep && (double)h[0] <= kProbeWideMaxReplays * cells;
  if (knobs().tile_debug)
    fprintf(stderr, "[mprof probe] %s: %zu tiles, %.3g cells, %llu replays -> %s\n",
            zn ? "z-norm" : "AAMP", pt.size(), cells, h[0],
            keep ? "covariance-only form" : zn ? "column-scaled form" : "(delta, sigma) kernel");
  return MPROF_OK;
}

// The constant-row kernel of the sweep policy (sweep_rc.h), or -1: FP64 fast-mode covariance-only
// forms whose rows per tile are whole windows.
int rc_policy_of(const mprof_ctx* c, const mprof_config* cfg, long long R) {
  // (anytime sweeps run many small chunks: the legacy kernel's single launch per chunk)
  if (!c->rowconst || cfg->exact || c->dense || c->progress) return -1;
  if (R <= 0) return -1;
  // FP32 mode: the covariance-only z-norm kernel (FFMA R, R, UR, R); the FP32 AAMP kernel is the
  // (delta, sigma) slide with in-loop value keys and keeps the tile kernel
  if (cfg->precision == MPROF_FP32)
    return (cfg->family == MPROF_ZNORMALIZED && !c->zn_colscale) ? mpg::kRcZnormF32 : -1;
  if (cfg->precision != MPROF_FP64) return -1;
  // Every covariance-only form: the replay-heavy ones (hit groups of 2, e.g. C5) stash their
  // accumulators per hit group, so a deferred replay restarts at its own group (sweep_rc.cu):
  // C5 2100 -> 1805 ms, random walk n = 2^20, m = 512 ACAMP 131.7 -> 114.4 ms; small sweeps
  // (n = 2^17, m = 512: 3.29 vs 3.34 ms) are neutral.
  if (cfg->family == MPROF_ZNORMALIZED)
    return c->zn_colscale ? -1 : (c->wide ? mpg::kRcWideZnorm : mpg::kRcZnorm);
  const bool l2 = cfg->family == MPROF_EUCLIDEAN || (cfg->family == MPROF_PNORM && cfg->p == 2.0);
  if (l2 && c->aamp_cov) return c->wide ? mpg::kRcWideEuclidCov : mpg::kRcEuclidCov;
  return -1;
}

// Pinned host mirror of `pairs` (count entries), refreshed when the operands were rebuilt.
int32_t rc_host_pairs(mprof_ctx* c, const void* pairs, size_t bytes, const void** out) {
  if (c->rc_host_src != pairs || c->rc_host_gen != c->op_gen || c->rc_host_cap < bytes) {
    if (c->rc_host_cap < bytes) {
      if (c->rc_host) cudaFreeHost(c->rc_host);
      c->rc_host = nullptr;
      c->rc_host_cap = 0;
      CK(cudaMallocHost(&c->rc_host, bytes));
      c->rc_host_cap = bytes;
    }
    CK(cudaMemcpyAsync(c->rc_host, pairs, bytes, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->rc_host_src = pairs;
    c->rc_host_gen = c->op_gen;
  }
  *out = c->rc_host;
  return MPROF_OK;
}

// Sweeps a tile table arranged by arrange_tiles: tiles [0, n_near) on the side stream with the
// side kernel, [n_near, n_legacy) with the policy's legacy kernel, the row bands with the
// constant-row kernel (rc_policy >= 0).
int32_t dispatch_sweep(mprof_ctx* c, const mprof_config* cfg, const SweepParams& prm,
                       long long ntiles, long long n_near, long long n_legacy,
                       const std::vector<mpg::RcBand>& bands, int rc_policy,
                       const void* host_pairs, int k1, bool first_diag, uint32_t* launches,
                       float* ms, uint32_t* rc_launches, mpg::RcGraph* rc_graph = nullptr) {
  int32_t st = MPROF_OK;
  if (n_legacy < ntiles && !host_pairs) {  // before the timed region: the mirror needs a sync
    if (rc_policy < 0 || bands.empty()) return fail(MPROF_E_CUDA, "internal: row bands without a kernel");
    st = rc_host_pairs(c, mpg::rc_pairs(rc_policy, prm),
                       (size_t)std::max(prm.L - 1, 1) * mpg::rc_pair_bytes(rc_policy), &host_pairs);
    if (st != MPROF_OK) return st;
  }
  if (first_diag && !cfg->exact) {
    st = with_policy(c, cfg, [&]<class P>() { return launch_first_diag<P>(c, prm, k1, launches); });
    if (st != MPROF_OK) return st;
  }
  if (ntiles > INT_MAX) return fail(MPROF_E_TOO_LARGE, "too many tiles");
  *ms = 0.f;
  if (ntiles == 0) return MPROF_OK;
  if (c->timing) CK(cudaEventRecord(c->ev0, c->stream));
  n_near = std::min(n_near, ntiles);
  if (n_near > 0) {
    st = ensure_side(c);
    if (st != MPROF_OK) return st;
    CK(cudaEventRecord(c->ev_fork, c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    // near block: the column-scaled z-norm form, or the (delta, sigma) AAMP kernel
    if (cfg->family != MPROF_ZNORMALIZED) st = launch_tiles<Euclid<false>>(prm, 0, n_near, c->side, launches);
    else if (cfg->precision == MPROF_FP32) st = launch_tiles<ZnormF32<true>>(prm, 0, n_near, c->side, launches);
    else st = launch_tiles<Znorm<true>>(prm, 0, n_near, c->side, launches);
    if (st != MPROF_OK) return st;
    CK(cudaEventRecord(c->ev_join, c->side));
  }
  n_legacy = std::min(std::max(n_legacy, n_near), ntiles);
  st = with_policy(c, cfg, [&]<class P>() {
    return launch_tiles<P>(prm, n_near, n_legacy - n_near, c->stream, launches);
  });
  if (st != MPROF_OK) return st;
  if (n_legacy < ntiles) {
    if (rc_policy < 0 || bands.empty()) return fail(MPROF_E_CUDA, "internal: row bands without a kernel");
    uint32_t nl = 0;
    const cudaError_t e = mpg::rc_sweep(rc_policy, prm, bands, c->rc, c->stream, host_pairs, &nl,
                                        rc_graph);
    if (e != cudaSuccess) return cuda_fail(e, "constant-row sweep");
    *launches += nl;
    if (rc_launches) *rc_launches += nl;
  }
  if (n_near > 0) CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  if (c->timing) {
    CK(cudaEventRecord(c->ev1, c->stream));
    CK(cudaEventSynchronize(c->ev1));
    CK(cudaEventElapsedTime(ms, c->ev0, c->ev1));
  }
  return MPROF_OK;
}

// Resident sweep CTAs per SM of the policy's kernel (registers + shared memory), >= 1.
int sweep_blocks_per_sm(const mprof_ctx* c, const mprof_config* cfg) {
  int nb = 1;
  with_policy(c, cfg, [&]<class P>() {
    using SM = SweepSmem<P, kD, kT, stage_rows<P>()>;
    auto kern = sweep_kernel<P, kD, kT, stage_rows<P>(), min_blocks<P>()>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SM)) ==
            cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kT, sizeof(SM)) != cudaSuccess)
      nb = 1;
    cudaGetLastError();
    return 0;
  });
  return std::max(1, nb);
}

int stage_rows_for(const mprof_ctx* c, const mprof_config* cfg) {
  return with_policy(c, cfg, [&]<class P>() { return stage_rows<P>(); });
}

int32_t check_config(uint64_t n, const mprof_config* cfg) {
  // validate_config (/root/reference/proj/src/core.cpp:21-40), same order and codes
  if (cfg->m < 1 || cfg->m > n - 1)
    return fail(MPROF_E_BAD_SUBSEQ_LEN, "subsequence length %llu outside [1, %llu] for series of length %llu",
                (unsigned long long)cfg->m, (unsigned long long)(n - 1), (unsigned long long)n);
  if (cfg->family == MPROF_PNORM && !(cfg->p >= 1.0))
    return fail(MPROF_E_BAD_P, "p-norm exponent must be >= 1, got %f", cfg->p);
  if (cfg->exclusion < 1 || cfg->exclusion > n - cfg->m)
    return fail(MPROF_E_BAD_EXCLUSION, "exclusion %llu outside [1, %llu]",
                (unsigned long long)cfg->exclusion, (unsigned long long)(n - cfg->m));
  if (!(cfg->flat_threshold >= 0.0)) return fail(MPROF_E_BAD_THRESHOLD, "flat_threshold must be >= 0");
  if (cfg->family < 0 || cfg->family > 2) return fail(MPROF_E_BAD_ARG, "unknown distance family %d", cfg->family);
  if (cfg->precision != MPROF_FP64 && cfg->precision != MPROF_FP32)
    return fail(MPROF_E_BAD_ARG, "unknown precision %d", cfg->precision);
  if (n >= (uint64_t)INT_MAX - 2 * (uint64_t)kK) return fail(MPROF_E_TOO_LARGE, "series too long for 32-bit positions");
  return MPROF_OK;
}

int32_t check_series(const double* t, uint64_t n) {
  // make_time_series (/root/reference/proj/src/core.cpp:7-19): NonFinite first, then TooShort
  for (uint64_t i = 0; i < n; ++i)
    if (!std::isfinite(t[i])) return fail(MPROF_E_NON_FINITE, "sample %llu is not finite", (unsigned long long)i);
  if (n < 2) return fail(MPROF_E_TOO_SHORT, "time series needs at least 2 samples, got %llu", (unsigned long long)n);
  return MPROF_OK;
}

// ---- sweep phases ---------------------------------------------------------------------------
// (1) operands of series d_t: z-norm statistics, operand pairs (FP64 and FP32), filter form
int32_t prepare_operands(mprof_ctx* c, const double* d_t, int n, const mprof_config* cfg,
                         const Workspace& w, uint32_t* launches) {
  const int m = (int)cfg->m;
  const int L = n - m + 1;
  const int g = grid_for(L);
  int32_t st = MPROF_OK;
  const bool zn = cfg->family == MPROF_ZNORMALIZED;
  ++c->op_gen;  // the operand arrays are rebuilt: host mirrors of them are stale
  if (zn) {
    c->stats_t = nullptr;  // force: the series bytes behind d_t may have changed
    st = ensure_znorm_stats(c, d_t, (uint64_t)n, cfg, w);
    if (st != MPROF_OK) return st;
    k_znorm_pairs<<<g, 256, 0, c->stream>>>(d_t, w.mu, w.A, L, m);
    *launches += 2;
    // filter form for this series (mprof_ctx_set_form, then MPROF_ZN_FILTER=cov|col, override
    // the measured choice)
    if (c->form == MPROF_FORM_COV || c->form == MPROF_FORM_WIDE) {
      c->zn_colscale = false;
    } else if (c->form == MPROF_FORM_ALT || c->form == MPROF_FORM_DENSE) {
      c->zn_colscale = true;
    } else if (knobs().zn_filter == 1) {
      c->zn_colscale = false;
    } else if (knobs().zn_filter == 2) {
      c->zn_colscale = true;
    } else {
      if (!c->d_spread) CK(cudaMalloc(&c->d_spread, 3 * sizeof(double)));
      CK(cudaMemsetAsync(c->d_spread, 0, 2 * sizeof(double), c->stream));
      k_bspread<<<grid_for(L / (2 * kD) + 1), 256, 0, c->stream>>>(w.B, L, c->d_spread);
      double h[2];
      CK(cudaMemcpyAsync(h, c->d_spread, sizeof h, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      ++*launches;
      c->zn_colscale = !(h[1] > 0.0 && h[0] / h[1] >= kZnCovFilterMinSpread);
    }
  } else {
    // the fast Euclidean policy slides (delta, sigma) pairs; everything else the raw pairs
    const bool ds = !cfg->exact && (cfg->family == MPROF_EUCLIDEAN ||
                                    (cfg->family == MPROF_PNORM && cfg->p == 2.0));
    k_build_pairs<<<g, 256, 0, c->stream>>>(d_t, w.A, L, m, ds ? kPairsDeltaSum : kPairsRaw);
    ++*launches;
    c->aamp_cov = false;
    const bool forced = c->form != MPROF_FORM_AUTO;
    if (ds && cfg->precision == MPROF_FP64 && c->form != MPROF_FORM_ALT && c->form != MPROF_FORM_DENSE &&
        (forced || knobs().aamp_cov != 0)) {
      // covariance form (EuclidCov) when the window scales vary little inside the filter
      // blocks (the same spread test as the z-norm filter form; MPROF_AAMP_COV=0|1 overrides)
      if (!c->d_spread) CK(cudaMalloc(&c->d_spread, 3 * sizeof(double)));
      CK(cudaMemsetAsync(c->d_spread, 0, 3 * sizeof(double), c->stream));
      unsigned int* d_oor = reinterpret_cast<unsigned int*>(c->d_spread + 2);
      k_euclid_stats<<<ws_grid(L), kWsT, 0, c->stream>>>(d_t, L, m, w.emu, w.S, w.SB, w.cv, d_oor);
      k_bspread<<<grid_for(L / (2 * kD) + 1), 256, 0, c->stream>>>(w.cv, L, c->d_spread);
      *launches += 2;
      double h[3];
      CK(cudaMemcpyAsync(h, c->d_spread, sizeof h, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      unsigned int oor;
      std::memcpy(&oor, &h[2], sizeof oor);
      bool use = forced || knobs().aamp_cov == 1 || (h[1] > 0.0 && h[0] / h[1] >= kAampCovMinSpread);
      if (oor) use = false;  // values beyond the float tables' range: (delta, sigma) kernel
      if (use) {
        k_znorm_pairs<<<g, 256, 0, c->stream>>>(d_t, w.emu, w.A2, L, m);
        ++*launches;
        c->aamp_cov = true;
      }
    }
  }
  if (cfg->precision == MPROF_FP32) {
    if (zn) {
      k_znorm_pairs32<<<g, 256, 0, c->stream>>>(w.A, w.B, w.A32, w.B32, L);
      ++*launches;
    } else {
      CK(cudaMemsetAsync(w.scalars, 0, sizeof(double), c->stream));
      k_mean<<<grid_for(n), 256, 0, c->stream>>>(d_t, n, w.scalars);
      const bool ds32 = cfg->family == MPROF_EUCLIDEAN || cfg->p == 2.0;
      k_build_pairs32<<<g, 256, 0, c->stream>>>(d_t, w.A32, L, m, ds32 ? kPairsDeltaSum : kPairsRaw,
                                                w.scalars);
      *launches += 2;
    }
  }
  CK(cudaGetLastError());
  return MPROF_OK;
}

// (2) the tiles of diagonals [k_lo, k_hi) x rows [0, row_hi) into w.best (initialised by the
// caller)
struct SweepOut {
  float ms = 0.f;
  long long ntiles = 0, R = 0;
  uint32_t rc_launches = 0;  // window launches of the constant-row kernel
};

SweepParams make_params(const mprof_ctx* c, const double* d_t, int n, const mprof_config* cfg,
                        const Workspace& w, int k_hi, int row_hi) {
  SweepParams prm;
  prm.t = d_t;
  prm.A = w.A;
  prm.B = w.B;
  prm.A32 = w.A32;
  prm.B32 = w.B32;
  prm.mu = c->aamp_cov && cfg->family != MPROF_ZNORMALIZED ? w.emu : w.mu;
  prm.A2 = w.A2;
  prm.SB = w.SB;
  prm.S = w.S;
  prm.best = w.best;
  prm.tiles = nullptr;
  prm.n = n;
  prm.m = (int)cfg->m;
  prm.L = n - (int)cfg->m + 1;
  prm.k_hi = k_hi;
  prm.R = 0;
  prm.row_hi = row_hi;
  prm.p = cfg->p;
  prm.stats = nullptr;
  prm.scratch = w.cv;
  return prm;
}

Grid grid_of(const mprof_ctx* c, const mprof_config* cfg, int L, int row_hi) {
  return Grid{L, (long long)cfg->exclusion + (cfg->exact ? 0 : 1), row_hi, cfg->exact != 0,
              (int)cfg->m, stage_rows_for(c, cfg)};
}

// Per-series decisions, taken once before any band / chunk is swept so that they are the same
// for every band of a multi-GPU run and every chunk of an anytime run:
//  * the filter form: an automatically chosen covariance-only form (AAMP or z-norm) is confirmed
//    on the series itself when the WHOLE sweep has >= kProbeMinCells cells: the first-diagonal
//    thresholds, then the probe over the whole diagonal range (probe_form);
//  * the rows per tile (choose_R on the whole range).
struct SeriesPlan {
  long long R = 0;
  bool first_diag_done = false;  // the prepass of diagonal `exclusion` already ran
};

int32_t plan_series(mprof_ctx* c, const double* d_t, int n, const mprof_config* cfg,
                    const Workspace& w, int row_hi, uint32_t* launches, SeriesPlan* out) {
  const int L = n - (int)cfg->m + 1;
  c->wide = c->form == MPROF_FORM_WIDE;  // else set by the form probe below
  c->probe_replays = 0;
  c->probe_cells = 0.0;
  const bool zn = cfg->family == MPROF_ZNORMALIZED;
  const bool auto_cov = c->form == MPROF_FORM_AUTO &&
                        (zn ? (!c->zn_colscale && knobs().zn_filter == 0)
                            : (c->aamp_cov && knobs().aamp_cov == -1));
  const long long g0 = (long long)cfg->exclusion + 1;
  const bool big = row_hi == L && L - g0 > 2 * kK &&
                   (double)mprof_band_cells((uint64_t)n, cfg->m, (uint64_t)g0, (uint64_t)L) >= kProbeMinCells;
  if (auto_cov && !cfg->exact && cfg->precision == MPROF_FP64 && !big) {
    // Below the probe size the covariance-only forms are not used: their block bound's slack is
    // unconfirmed and small sweeps measured slower with them (random walk n = 2^16, m = 256:
    // EuclidCov 1.76 ms vs (delta, sigma) 0.76 ms; Znorm<0> 0.33 vs Znorm<1> 0.12 ms at n = 2^14).
    if (zn) c->zn_colscale = true;
    else c->aamp_cov = false;
  }
  // Dense<P> (no block filter): forced, or chosen by the noise test for noise-like series
  const bool fast64 = !cfg->exact && cfg->precision == MPROF_FP64;
  const bool dense_ok = fast64 && (zn || cfg->family == MPROF_EUCLIDEAN ||
                                   (cfg->family == MPROF_PNORM && (cfg->p == 1.0 || cfg->p == 2.0 || cfg->p == 3.0)));
  c->dense = dense_ok && c->form == MPROF_FORM_DENSE;
  if (kNoiseDenseFrac <= 1.0 && dense_ok && c->form == MPROF_FORM_AUTO && row_hi == L &&
      L - (long long)cfg->exclusion > 1 && knobs().zn_filter == 0 && knobs().aamp_cov == -1) {
    const SweepParams prm = make_params(c, d_t, n, cfg, w, L, L);
    int32_t st = with_policy(c, cfg, [&]<class P>() {
      return launch_first_diag<P>(c, prm, (int)cfg->exclusion, launches);
    });
    if (st != MPROF_OK) return st;
    out->first_diag_done = true;
    if (!c->noise_cnt) CK(cudaMalloc(&c->noise_cnt, sizeof(unsigned int)));
    CK(cudaMemsetAsync(c->noise_cnt, 0, sizeof(unsigned int), c->stream));
    st = with_policy(c, cfg, [&]<class P>() {
      k_noise_test<P><<<grid_for(32LL * kNoiseSamples, 256), 256, 0, c->stream>>>(
          prm, (int)cfg->exclusion, kNoiseSamples, c->noise_cnt);
      return MPROF_OK;
    });
    ++*launches;
    unsigned int cnt = 0;
    CK(cudaMemcpyAsync(&cnt, c->noise_cnt, sizeof cnt, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->noise_frac = (double)cnt / kNoiseSamples;
    c->dense = c->noise_frac > kNoiseDenseFrac;
    if (knobs().tile_debug)
      fprintf(stderr, "[mprof noise] %u of %d random pairs pass the first-diagonal thresholds -> %s\n",
              cnt, kNoiseSamples, c->dense ? "dense" : "filtered");
  }
  if (c->dense) {  // the dense kernels are the (delta, sigma) / column-scaled / p-norm slides
    if (zn) c->zn_colscale = true;
    else c->aamp_cov = false;
  }
  if (!c->dense && auto_cov && fast64 && big) {
    const SweepParams prm = make_params(c, d_t, n, cfg, w, L, L);
    int32_t st = MPROF_OK;
    if (!out->first_diag_done) {
      st = with_policy(c, cfg, [&]<class P>() {
        return launch_first_diag<P>(c, prm, (int)cfg->exclusion, launches);
      });
      if (st != MPROF_OK) return st;
      out->first_diag_done = true;
    }
    st = probe_form(c, zn, prm, (int)(g0 + kK), launches);
    if (st != MPROF_OK) return st;
  }
  const Grid g = grid_of(c, cfg, L, row_hi);
  long long pbits;
  std::memcpy(&pbits, &cfg->p, sizeof pbits);
  const int slots = c->num_sms * sweep_blocks_per_sm(c, cfg);
  const long long key[9] = {L, g.g0, row_hi, (long long)cfg->m, cfg->exact,
                            (long long)cfg->refresh_interval,
                            ((long long)cfg->family << 8) | (cfg->precision << 4) | (c->zn_colscale ? 1 : 0) |
                                (c->aamp_cov ? 2 : 0) | (c->wide ? 4 : 0) | (c->dense ? 8 : 0),
                            pbits, slots};
  out->R = 0;
  for (const auto& rc : c->R_cache)
    if (std::equal(key, key + 9, rc.key)) out->R = rc.R;
  if (!out->R) {
    out->R = choose_R(cfg, g, slots);
    if (!knobs().rows_per_tile) {
      if (c->R_cache.size() >= 16) c->R_cache.erase(c->R_cache.begin());
      mprof_ctx::RChoice rc;
      std::copy(key, key + 9, rc.key);
      rc.R = out->R;
      c->R_cache.push_back(rc);
    }
  }
  c->plan_R = out->R;
  return MPROF_OK;
}

// The per-series decisions that fix every cell's arithmetic: rows per tile and kernel forms.
int plan_flags(const mprof_ctx* c) {
  return (c->aamp_cov ? 1 : 0) | (c->zn_colscale ? 2 : 0) | (c->wide ? 4 : 0) | (c->dense ? 8 : 0);
}

// The tiles of diagonals [k_lo, k_hi) x rows [0, row_hi) into w.best (initialised by the caller),
// R rows per tile (plan_series).
// first_diag: seed the filter thresholds with diagonal `exclusion` (evaluated directly) first.
// Those are genuine cells even when the band starts further out, so band profiles still merge
// exactly, and every band starts from near-final thresholds (random walks: ~all nearest
// neighbours at k = 1). In the fast mode diagonal `exclusion` belongs to that prepass, never to
// the tiles (tile grid origin exclusion + 1): sweeping it again would re-offer values equal to
// the thresholds it set (every block of those lanes replays and pays L2 round trips).
int32_t sweep_tiles(mprof_ctx* c, const double* d_t, int n, const mprof_config* cfg,
                    const Workspace& w, int k_lo, int k_hi, int row_hi, bool first_diag,
                    long long R, long long l_old, uint32_t* launches, SweepOut* out) {
  const int L = n - (int)cfg->m + 1;
  if (k_lo >= k_hi || row_hi <= 0) return MPROF_OK;
  first_diag = first_diag && !cfg->exact;
  const int k_tile = (!cfg->exact && k_lo == (int)cfg->exclusion) ? k_lo + 1 : k_lo;
  SweepParams prm = make_params(c, d_t, n, cfg, w, k_hi, row_hi);
  const Grid g = grid_of(c, cfg, L, row_hi);
  out->R = R;
  // the global block next to the exclusion zone runs the side kernel (dispatch_sweep)
  const bool cov_main = (cfg->family == MPROF_ZNORMALIZED && !c->zn_colscale) ||
                        (cfg->family != MPROF_ZNORMALIZED && c->aamp_cov);
  const bool near_block = cov_main && !cfg->exact && !knobs().zn_no_near;
  const int rc_policy = rc_policy_of(c, cfg, R);
  int32_t st = build_tiles(c, g, k_tile, k_hi, R, l_old, near_block, rc_policy >= 0, &out->ntiles);
  if (st != MPROF_OK) return st;
  prm.tiles = c->tiles->d;
  prm.R = (int)std::min<long long>(R, INT_MAX);
  const bool want_stats = knobs().stats;
  if (want_stats) {
    CK(cudaMallocAsync(&prm.stats, 2 * sizeof(unsigned long long), c->stream));
    CK(cudaMemsetAsync(prm.stats, 0, 2 * sizeof(unsigned long long), c->stream));
  }
  st = dispatch_sweep(c, cfg, prm, out->ntiles, c->tiles->n_near, c->tiles->n_legacy,
                      c->tiles->bands, rc_policy, nullptr, (int)cfg->exclusion, first_diag, launches,
                      &out->ms, &out->rc_launches);
  if (st != MPROF_OK) return st;
  if (want_stats) {
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, prm.stats, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFreeAsync(prm.stats, c->stream);
    fprintf(stderr, "[mprof stats] family %d L %d tiles %lld R %lld: replays %llu offers %llu\n",
            cfg->family, L, out->ntiles, R, h[0], h[1]);
  }
  return MPROF_OK;
}

// (3) z-norm flat windows of the band (original coordinates): final entries
int32_t flat_fix(mprof_ctx* c, const double* B, int L, int k_lo, int k_hi, const Workspace& w,
                 BestEntry* best, uint32_t* launches) {
  if (k_lo >= k_hi) return MPROF_OK;
  const int nch = (L + kChunk - 1) / kChunk;
  k_flat_chunk_min<<<nch, 256, 0, c->stream>>>(B, L, w.cmin);
  k_flat_fix<<<grid_for(L), 256, 0, c->stream>>>(B, L, k_lo, k_hi, w.cmin, best);
  *launches += 2;
  CK(cudaGetLastError());
  return MPROF_OK;
}

void fill_info(mprof_ctx* c, const mprof_config* cfg, uint64_t cells, long long diagonals,
               const SweepOut& so, uint32_t launches, mprof_run_info* info) {
  if (!info) return;
  // FP64-pipe instructions per cell of the hot loop (SASS-audited)
  float ops = 4.f;
  if (cfg->family == MPROF_ZNORMALIZED) ops = c->zn_colscale ? 3.125f : 2.f;
  else if (cfg->exact) ops = (cfg->family == MPROF_PNORM && cfg->p != 1.0 && cfg->p != 2.0) ? 8.f : 6.f;
  else if (cfg->family == MPROF_EUCLIDEAN || cfg->p == 2.0) ops = c->aamp_cov ? 2.f : 3.f;
  else if (cfg->p == 1.0) ops = 4.f;
  else if (cfg->p == 3.0 || cfg->p == 4.0) ops = 6.f;
  else ops = 0.f;  // generic pow: library call, not a fixed count
  if (cfg->precision == MPROF_FP32) {
    info->fp64_ops_per_cell = 0.f;
    info->fp32_ops_per_cell = ops;
  } else {
    info->fp64_ops_per_cell = ops;
    info->fp32_ops_per_cell = 0.f;
  }
  info->cells = cells;
  info->diagonals = diagonals > 0 ? (uint64_t)diagonals : 0;
  info->tiles = (uint64_t)so.ntiles;
  info->rows_per_tile = (uint64_t)so.R;
  info->kernel_launches = launches;
  info->row_windows = so.rc_launches;
  info->reserved = 0;
  info->sweep_ms = so.ms;
  std::memset(info->policy, 0, sizeof info->policy);
  with_policy(c, cfg, [&]<class P>() {
    std::snprintf(info->policy, sizeof info->policy, "%s", policy_name<P>());
    info->hit_group = hit_group_for<P>();
    return 0;
  });
  info->probe_replays = (uint32_t)std::min<unsigned long long>(c->probe_replays, UINT32_MAX);
  info->probe_cells = (uint64_t)c->probe_cells;
}

int32_t sweep_impl(mprof_ctx* c, const double* d_t, uint64_t n64, const mprof_config* cfg,
                   uint64_t k_lo64, uint64_t k_hi64, double* d_cmp, int64_t* d_idx,
                   mprof_run_info* info) {
  int32_t st = check_config(n64, cfg);
  if (st != MPROF_OK) return st;
  if (cfg->precision == MPROF_FP32 && cfg->exact)
    return fail(MPROF_E_BAD_ARG, "the exact (parity) mode is FP64 only");
  const int n = (int)n64, m = (int)cfg->m;
  const int L = n - m + 1;
  // band: [max(k_lo, excl), min(k_hi, L)) ; 0,0 = everything
  long long k_lo = (long long)cfg->exclusion, k_hi = L;
  if (!(k_lo64 == 0 && k_hi64 == 0)) {
    k_lo = std::max<long long>(k_lo, (long long)k_lo64);
    k_hi = std::min<long long>(k_hi, (long long)k_hi64);
  }
  Workspace w;
  st = carve(c, L, &w);
  if (st != MPROF_OK) return st;
  uint32_t launches = 0;
  const bool zn = cfg->family == MPROF_ZNORMALIZED;
  st = prepare_operands(c, d_t, n, cfg, w, &launches);
  if (st != MPROF_OK) return st;
  k_init_best<<<grid_for(L), 256, 0, c->stream>>>(w.best, zn ? w.B : nullptr, L);
  ++launches;
  SweepOut so;
  long long k_done = k_hi;
  SeriesPlan plan;
  st = plan_series(c, d_t, n, cfg, w, L, &launches, &plan);
  if (st != MPROF_OK) return st;
  if (!c->progress || k_lo >= k_hi) {
    st = sweep_tiles(c, d_t, n, cfg, w, (int)k_lo, (int)k_hi, L, !plan.first_diag_done, plan.R, 0,
                     &launches, &so);
    if (st != MPROF_OK) return st;
  } else {
    // Anytime mode (scan_diagonals' observer, /root/reference/proj/src/detail/diag_scan.hpp:
    // 210-226): the band is swept in ascending chunks of diagonals, the observer sees
    // (diagonals done, total) after each; false cancels, leaving the exact minimum over the
    // completed diagonals. Chunks of max(1, total/256) diagonals (one diagonal for small runs).
    const long long total = k_hi - k_lo;
    const long long chunk = std::max<long long>(1, (total + 255) / 256);
    for (long long a = k_lo; a < k_hi; a += chunk) {
      const long long b = std::min(k_hi, a + chunk);
      SweepOut part;
      st = sweep_tiles(c, d_t, n, cfg, w, (int)a, (int)b, L, a == k_lo && !plan.first_diag_done,
                       plan.R, 0, &launches, &part);
      if (st != MPROF_OK) return st;
      so.ms += part.ms;
      so.rc_launches += part.rc_launches;
      so.ntiles += part.ntiles;
      so.R = part.R;
      CK(cudaStreamSynchronize(c->stream));
      if (!c->progress((uint64_t)(b - k_lo), (uint64_t)total, c->progress_user)) {
        k_done = b;
        break;
      }
    }
  }
  if (zn) {
    st = flat_fix(c, w.B, L, (int)k_lo, (int)k_done, w, w.best, &launches);
    if (st != MPROF_OK) return st;
  }
  k_hi = k_done;
  k_split<<<grid_for(L), 256, 0, c->stream>>>(w.best, d_cmp, d_idx, L);
  ++launches;
  CK(cudaGetLastError());
  const uint64_t cells = k_lo < k_hi ? mprof_band_cells(n64, cfg->m, (uint64_t)k_lo, (uint64_t)k_hi) : 0;
  fill_info(c, cfg, cells, k_hi - k_lo, so, launches, info);
  return MPROF_OK;
}

int32_t host_entry(mprof_ctx* in, const double* t, uint64_t n, const mprof_config* cfg,
                   int32_t family_required, double* P, int64_t* I, mprof_run_info* info) {
  if (!t || !cfg || !P || !I) return fail(MPROF_E_BAD_ARG, "null argument");
  int32_t st = check_series(t, n);
  if (st != MPROF_OK) return st;
  st = check_config(n, cfg);
  if (st != MPROF_OK) return st;
  if (cfg->family != family_required) {
    static const char* msg[] = {"aamp computes Euclidean profiles only",
                                "aamp_pnorm requires a p-norm distance kind",
                                "acamp requires the z-normalized distance kind"};
    return fail(MPROF_E_BAD_KIND, "%s", msg[family_required]);
  }
  mprof_ctx* c = nullptr;
  st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  const uint64_t L = n - cfg->m + 1;
  const size_t nt = align_up(n * sizeof(double)), nl = align_up(L * sizeof(double));
  st = ensure(&c->io, &c->io_bytes, nt + 3 * nl);
  if (st != MPROF_OK) return st;
  char* base = static_cast<char*>(c->io);
  double* d_t = reinterpret_cast<double*>(base);
  double* d_cmp = reinterpret_cast<double*>(base + nt);
  int64_t* d_idx = reinterpret_cast<int64_t*>(base + nt + nl);
  double* d_P = reinterpret_cast<double*>(base + nt + 2 * nl);
  CK(cudaMemcpyAsync(d_t, t, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  st = sweep_impl(c, d_t, n, cfg, 0, 0, d_cmp, d_idx, info);
  if (st != MPROF_OK) return st;
  st = mprof_finalize_device(c, d_t, n, d_cmp, d_idx, cfg, d_P);
  if (st != MPROF_OK) return st;
  if (info) info->kernel_launches += 1;
  CK(cudaMemcpyAsync(P, d_P, L * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(I, d_idx, L * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return MPROF_OK;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// C ABI

extern "C" {

int32_t mprof_abi_version(void) { return MPROF_GPU_ABI_VERSION; }

const char* mprof_status_string(int32_t s) {
  switch (s) {
    case MPROF_OK: return "ok";
    case MPROF_E_NON_FINITE: return "NonFinite";
    case MPROF_E_TOO_SHORT: return "TooShort";
    case MPROF_E_EMPTY_INPUT: return "EmptyInput";
    case MPROF_E_PARSE_ERROR: return "ParseError";
    case MPROF_E_BAD_SUBSEQ_LEN: return "BadSubseqLen";
    case MPROF_E_BAD_P: return "BadP";
    case MPROF_E_BAD_EXCLUSION: return "BadExclusion";
    case MPROF_E_BAD_THRESHOLD: return "BadThreshold";
    case MPROF_E_BAD_KIND: return "BadKind";
    case MPROF_E_OUT_OF_RANGE: return "OutOfRange";
    case MPROF_E_DEGENERATE: return "Degenerate";
    case MPROF_E_INCOMPLETE_STATE: return "IncompleteState";
    case MPROF_E_IO: return "Io";
    case MPROF_E_CUDA: return "Cuda";
    case MPROF_E_OOM: return "OutOfMemory";
    case MPROF_E_BAD_ARG: return "BadArgument";
    case MPROF_E_TOO_LARGE: return "TooLarge";
    default: return "unknown";
  }
}

const char* mprof_last_error(void) { return g_last_error.c_str(); }

void mprof_config_init(mprof_config* cfg, uint64_t m, int32_t family, double p) {
  std::memset(cfg, 0, sizeof *cfg);
  cfg->m = m;
  cfg->family = family;
  cfg->p = (family == MPROF_PNORM) ? p : 2.0;
  cfg->exclusion = 1;
  cfg->order = MPROF_ORDER_ASCENDING;
  cfg->order_seed = 0;
  cfg->refresh_interval = 0;
  cfg->flat_threshold = 1e-12 * (double)m;  // default_flat_threshold (core.hpp:78-80)
  cfg->precision = MPROF_FP64;
  cfg->exact = 0;
}

int32_t mprof_validate(const double* t, uint64_t n, const mprof_config* cfg) {
  if (!t || !cfg) return fail(MPROF_E_BAD_ARG, "null argument");
  int32_t st = check_series(t, n);
  if (st != MPROF_OK) return st;
  return check_config(n, cfg);
}

uint64_t mprof_profile_length(uint64_t n, uint64_t m) { return n - m + 1; }

int32_t mprof_ctx_create(int32_t device, mprof_ctx** out) {
  if (!out) return fail(MPROF_E_BAD_ARG, "null out");
  *out = nullptr;
  int count = 0;
  CK(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return fail(MPROF_E_CUDA, "no CUDA device %d (%d present)", device, count);
  CK(cudaSetDevice(device));
  mprof_ctx* c = new mprof_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete c; return cuda_fail(e, "cudaStreamCreate"); }
  c->own_stream = true;
  cudaEventCreate(&c->ev0);
  cudaEventCreate(&c->ev1);
  *out = c;
  return MPROF_OK;
}

void mprof_ctx_destroy(mprof_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->ws) cudaFree(c->ws);
  if (c->io) cudaFree(c->io);
  for (auto& sl : c->tile_slot)
    if (sl.d) cudaFree(sl.d);
  mpg::rc_release(c->rc);
  if (c->rc_host) cudaFreeHost(c->rc_host);
  if (c->d_spread) cudaFree(c->d_spread);
  if (c->probe_d) cudaFree(c->probe_d);
  if (c->probe_cnt) cudaFree(c->probe_cnt);
  if (c->noise_cnt) cudaFree(c->noise_cnt);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
  }
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  for (auto it = g_default_ctx.by_device.begin(); it != g_default_ctx.by_device.end(); ++it)
    if (it->second == c) { g_default_ctx.by_device.erase(it); break; }
  delete c;
}

int32_t mprof_ctx_set_stream(mprof_ctx* in, void* stream) {
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
    c->own_stream = false;
  } else {
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  return MPROF_OK;
}

int32_t mprof_ctx_set_timing(mprof_ctx* in, int32_t enabled) {
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  c->timing = enabled != 0;
  return MPROF_OK;
}

int32_t mprof_aamp(mprof_ctx* ctx, const double* t, uint64_t n, const mprof_config* cfg, double* P,
                   int64_t* I, mprof_run_info* info) {
  return host_entry(ctx, t, n, cfg, MPROF_EUCLIDEAN, P, I, info);
}

int32_t mprof_aamp_pnorm(mprof_ctx* ctx, const double* t, uint64_t n, const mprof_config* cfg,
                         double* P, int64_t* I, mprof_run_info* info) {
  return host_entry(ctx, t, n, cfg, MPROF_PNORM, P, I, info);
}

int32_t mprof_acamp(mprof_ctx* ctx, const double* t, uint64_t n, const mprof_config* cfg,
                    int32_t variant, double* P, int64_t* I, mprof_run_info* info) {
  if (variant != MPROF_ACAMP_FSCORE && variant != MPROF_ACAMP_SQUARED_DISTANCE)
    return fail(MPROF_E_BAD_ARG, "unknown AcampVariant %d", variant);
  // Both variants yield the same profile (acamp.hpp:93-95); the GPU compares in 1 - corr.
  return host_entry(ctx, t, n, cfg, MPROF_ZNORMALIZED, P, I, info);
}

int32_t mprof_sweep_device(mprof_ctx* in, const double* d_t, uint64_t n, const mprof_config* cfg,
                           uint64_t k_lo, uint64_t k_hi, double* d_cmp, int64_t* d_idx,
                           mprof_run_info* info) {
  if (!d_t || !cfg || !d_cmp || !d_idx) return fail(MPROF_E_BAD_ARG, "null argument");
  if (n < 2) return fail(MPROF_E_TOO_SHORT, "time series needs at least 2 samples");
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  return sweep_impl(c, d_t, n, cfg, k_lo, k_hi, d_cmp, d_idx, info);
}

int32_t mprof_finalize_device(mprof_ctx* in, const double* d_t, uint64_t n, const double* d_cmp,
                              const int64_t* d_idx, const mprof_config* cfg, double* d_P) {
  if (!d_t || !d_cmp || !d_idx || !cfg || !d_P) return fail(MPROF_E_BAD_ARG, "null argument");
  int32_t st = check_config(n, cfg);
  if (st != MPROF_OK) return st;
  mprof_ctx* c = nullptr;
  st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  const int L = (int)(n - cfg->m + 1);
  Workspace w;
  st = carve(c, L, &w);
  if (st != MPROF_OK) return st;
  if (cfg->family == MPROF_ZNORMALIZED) {
    st = ensure_znorm_stats(c, d_t, n, cfg, w);
    if (st != MPROF_OK) return st;
  }
  k_finalize_range<<<grid_for(32LL * L), 256, 0, c->stream>>>(d_t, d_cmp, d_idx, w.mu, w.B, d_P, 0, L,
                                                                (int)cfg->m, cfg->family, cfg->p,
                                                                cfg->exact ? 1 : 0);
  CK(cudaGetLastError());
  return MPROF_OK;
}

int32_t mprof_finalize_range_device(mprof_ctx* in, const double* d_t, uint64_t n,
                                    const double* d_cmp, const int64_t* d_idx,
                                    const mprof_config* cfg, double* d_P, uint64_t lo,
                                    uint64_t hi) {
  if (!d_t || !d_cmp || !d_idx || !cfg || !d_P) return fail(MPROF_E_BAD_ARG, "null argument");
  int32_t st = check_config(n, cfg);
  if (st != MPROF_OK) return st;
  const uint64_t L = n - cfg->m + 1;
  if (hi > L) hi = L;
  if (lo >= hi) return MPROF_OK;
  mprof_ctx* c = nullptr;
  st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  Workspace w;
  st = carve(c, (int)L, &w);
  if (st != MPROF_OK) return st;
  if (cfg->family == MPROF_ZNORMALIZED) {
    st = ensure_znorm_stats(c, d_t, n, cfg, w);
    if (st != MPROF_OK) return st;
  }
  // entries [lo, hi): shift the per-entry arrays; the series / statistics stay absolute
  k_finalize_range<<<grid_for(32LL * (long long)(hi - lo)), 256, 0, c->stream>>>(
      d_t, d_cmp, d_idx, w.mu, w.B, d_P, (int)lo, (int)hi, (int)cfg->m, cfg->family, cfg->p,
      cfg->exact ? 1 : 0);
  CK(cudaGetLastError());
  return MPROF_OK;
}

int32_t mprof_ipc_alloc(mprof_ctx* in, uint64_t bytes, void** d_ptr, mprof_ipc_handle* h) {
  if (!d_ptr || !h || bytes == 0) return fail(MPROF_E_BAD_ARG, "null argument or zero size");
  static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(mprof_ipc_handle), "IPC handle size");
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return fail(MPROF_E_OOM, "cudaMalloc(%llu) failed", (unsigned long long)bytes);
  CK(cudaMemset(p, 0, bytes));
  cudaIpcMemHandle_t ih;
  if (cudaIpcGetMemHandle(&ih, p) != cudaSuccess) {
    cudaFree(p);
    return fail(MPROF_E_CUDA, "cudaIpcGetMemHandle failed");
  }
  memcpy(h->bytes, &ih, sizeof(ih));
  *d_ptr = p;
  return MPROF_OK;
}

int32_t mprof_ipc_free(mprof_ctx* in, void* d_ptr) {
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  CK(cudaFree(d_ptr));
  return MPROF_OK;
}

int32_t mprof_ipc_open(mprof_ctx* in, const mprof_ipc_handle* h, void** d_ptr) {
  if (!h || !d_ptr) return fail(MPROF_E_BAD_ARG, "null argument");
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  cudaIpcMemHandle_t ih;
  memcpy(&ih, h->bytes, sizeof(ih));
  const cudaError_t e = cudaIpcOpenMemHandle(d_ptr, ih, cudaIpcMemLazyEnablePeerAccess);
  if (e == cudaErrorInvalidValue || e == cudaErrorInvalidResourceHandle || e == cudaErrorDeviceUninitialized) {
    cudaGetLastError();
    return fail(MPROF_E_BAD_ARG, "cudaIpcOpenMemHandle: %s (own or stale handle?)", cudaGetErrorString(e));
  }
  CK(e);
  return MPROF_OK;
}

int32_t mprof_ipc_close(mprof_ctx* in, void* d_ptr) {
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  CK(cudaIpcCloseMemHandle(d_ptr));
  return MPROF_OK;
}

int32_t mprof_merge_finalize_peers(mprof_ctx* in, const double* d_t, uint64_t n,
                                   const mprof_config* cfg, const double* const* peer_cmp,
                                   const int64_t* const* peer_idx, uint32_t nin,
                                   double* const* out_P, int64_t* const* out_I, uint32_t nout,
                                   uint64_t lo, uint64_t hi) {
  if (!d_t || !cfg || !peer_cmp || !peer_idx || !out_P || !out_I)
    return fail(MPROF_E_BAD_ARG, "null argument");
  if (nin < 1 || nin > MPROF_MAX_PEERS || nout < 1 || nout > MPROF_MAX_PEERS)
    return fail(MPROF_E_BAD_ARG, "peer counts must be in [1, %d]", MPROF_MAX_PEERS);
  PeerSet ps{};
  for (uint32_t r = 0; r < nin; ++r) {
    if (!peer_cmp[r] || !peer_idx[r]) return fail(MPROF_E_BAD_ARG, "null peer buffer %u", r);
    ps.cmp[r] = peer_cmp[r];
    ps.idx[r] = peer_idx[r];
  }
  for (uint32_t r = 0; r < nout; ++r) {
    if (!out_P[r] || !out_I[r]) return fail(MPROF_E_BAD_ARG, "null output buffer %u", r);
    ps.P[r] = out_P[r];
    ps.I[r] = out_I[r];
  }
  ps.nin = (int)nin;
  ps.nout = (int)nout;
  int32_t st = check_config(n, cfg);
  if (st != MPROF_OK) return st;
  const uint64_t L = n - cfg->m + 1;
  if (hi > L) hi = L;
  if (lo >= hi) return MPROF_OK;
  mprof_ctx* c = nullptr;
  st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  Workspace w;
  st = carve(c, (int)L, &w);
  if (st != MPROF_OK) return st;
  if (cfg->family == MPROF_ZNORMALIZED) {
    st = ensure_znorm_stats(c, d_t, n, cfg, w);
    if (st != MPROF_OK) return st;
  }
  k_merge_finalize_peers<<<grid_for(32LL * (long long)(hi - lo)), 256, 0, c->stream>>>(
      d_t, ps, w.mu, w.B, (int)lo, (int)hi, (int)cfg->m, cfg->family, cfg->p, cfg->exact ? 1 : 0);
  CK(cudaGetLastError());
  return MPROF_OK;
}

int32_t mprof_merge_device(mprof_ctx* in, double* d_cmp, int64_t* d_idx, const double* d_ocmp,
                           const int64_t* d_oidx, uint64_t L) {
  if (!d_cmp || !d_idx || !d_ocmp || !d_oidx) return fail(MPROF_E_BAD_ARG, "null argument");
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  k_merge<<<grid_for((long long)L), 256, 0, c->stream>>>(d_cmp, d_idx, d_ocmp, d_oidx, (int)L);
  CK(cudaGetLastError());
  return MPROF_OK;
}

int32_t mprof_profile_multi(const int32_t* devices, uint32_t ndev, int32_t engine, const double* t,
                            uint64_t n, const mprof_config* cfg, double* P, int64_t* I,
                            mprof_run_info* info) {
  if (!devices || ndev == 0 || !t || !cfg || !P || !I) return fail(MPROF_E_BAD_ARG, "null argument");
  if (engine < 0 || engine > 2) return fail(MPROF_E_BAD_ARG, "unknown engine %d", engine);
  if (ndev > MPROF_MAX_PEERS) return fail(MPROF_E_BAD_ARG, "at most %d bands (devices listed)", MPROF_MAX_PEERS);
  int32_t st = check_series(t, n);
  if (st != MPROF_OK) return st;
  st = check_config(n, cfg);
  if (st != MPROF_OK) return st;
  static const int32_t fam[] = {MPROF_EUCLIDEAN, MPROF_PNORM, MPROF_ZNORMALIZED};
  static const char* msg[] = {"aamp computes Euclidean profiles only",
                              "aamp_pnorm requires a p-norm distance kind",
                              "acamp requires the z-normalized distance kind"};
  if (cfg->family != fam[engine]) return fail(MPROF_E_BAD_KIND, "%s", msg[engine]);
  int count = 0, caller_dev = 0;
  CK(cudaGetDeviceCount(&count));
  CK(cudaGetDevice(&caller_dev));
  for (uint32_t g = 0; g < ndev; ++g)
    if (devices[g] < 0 || devices[g] >= count)
      return fail(MPROF_E_CUDA, "no CUDA device %d (%d present)", devices[g], count);
  const uint64_t L = n - cfg->m + 1;
  std::vector<uint64_t> cuts(ndev + 1);
  st = mprof_band_cuts(n, cfg->m, cfg->exclusion, ndev, cuts.data());
  if (st != MPROF_OK) return st;

  // one context, stream and buffer set per band (a device listed twice gets two contexts)
  struct Part {
    int dev = 0;
    mprof_ctx* ctx = nullptr;
    double* d_t = nullptr;
    double* d_cmp = nullptr;
    int64_t* d_idx = nullptr;
    mprof_run_info info{};
    int32_t st = MPROF_OK;
    std::string err;
  };
  std::vector<Part> parts(ndev);
  auto release = [&]() {
    for (auto& q : parts) {
      if (!q.ctx) continue;
      cudaSetDevice(q.dev);
      cudaStreamSynchronize(q.ctx->stream);
      cudaFree(q.d_t);
      cudaFree(q.d_cmp);
      cudaFree(q.d_idx);
      mprof_ctx_destroy(q.ctx);
      q.ctx = nullptr;
    }
  };
  auto work = [&](uint32_t g) {
    Part& q = parts[g];
    q.dev = devices[g];
    q.st = [&]() -> int32_t {
      int32_t s = mprof_ctx_create(q.dev, &q.ctx);
      if (s != MPROF_OK) return s;
      CK(cudaMalloc(&q.d_t, n * sizeof(double)));
      CK(cudaMalloc(&q.d_cmp, L * sizeof(double)));
      CK(cudaMalloc(&q.d_idx, L * sizeof(int64_t)));
      CK(cudaMemcpyAsync(q.d_t, t, n * sizeof(double), cudaMemcpyHostToDevice, q.ctx->stream));
      if (cuts[g] >= cuts[g + 1]) {  // empty band: an all-empty partial profile
        k_split_empty<<<grid_for((long long)L), 256, 0, q.ctx->stream>>>(q.d_cmp, q.d_idx, (int)L);
        CK(cudaGetLastError());
      } else {
        s = sweep_impl(q.ctx, q.d_t, n, cfg, cuts[g], cuts[g + 1], q.d_cmp, q.d_idx, &q.info);
        if (s != MPROF_OK) return s;
      }
      CK(cudaStreamSynchronize(q.ctx->stream));
      return MPROF_OK;
    }();
    if (q.st != MPROF_OK) q.err = g_last_error;
  };
  {
    std::vector<std::thread> pool;
    for (uint32_t g = 1; g < ndev; ++g) pool.emplace_back(work, g);
    work(0);
    for (auto& th : pool) th.join();
  }
  for (auto& q : parts)
    if (q.st != MPROF_OK) {
      const int32_t s = q.st;
      const std::string e = q.err;
      release();
      g_last_error = e;
      cudaSetDevice(caller_dev);
      return s;
    }
  // merge + finalize on the first device in ONE kernel that reads every band's partial (cmp, idx)
  // in place over NVLink peer access (k_merge_finalize_peers, MinBuffer::absorb + finalize, the
  // same kernel the multi-process path uses); without peer access between two of the devices the
  // partials are first copied to the first device (cudaMemcpyPeer) and merged from there
  Part& p0 = parts[0];
  mprof_ctx* c0 = p0.ctx;
  auto finish = [&]() -> int32_t {
    CK(cudaSetDevice(p0.dev));
    std::vector<void*> owned;  // device-0 copies of partials without peer access, d_P, d_I
    auto dev_alloc = [&](size_t bytes) -> void* {
      void* q = nullptr;
      if (cudaMalloc(&q, bytes) != cudaSuccess) return nullptr;
      owned.push_back(q);
      return q;
    };
    std::vector<const double*> in_cmp(ndev);
    std::vector<const int64_t*> in_idx(ndev);
    int32_t s = MPROF_OK;
    for (uint32_t g = 0; g < ndev && s == MPROF_OK; ++g) {
      const Part& q = parts[g];
      in_cmp[g] = q.d_cmp;
      in_idx[g] = q.d_idx;
      if (q.dev == p0.dev) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, p0.dev, q.dev);
      if (can) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(q.dev, 0);
        if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
          continue;
        }
        cudaGetLastError();
      }
      double* cc = static_cast<double*>(dev_alloc(L * sizeof(double)));
      int64_t* ci = static_cast<int64_t*>(dev_alloc(L * sizeof(int64_t)));
      if (!cc || !ci) return fail(MPROF_E_OOM, "merge staging");
      CK(cudaMemcpyPeerAsync(cc, p0.dev, q.d_cmp, q.dev, L * sizeof(double), c0->stream));
      CK(cudaMemcpyPeerAsync(ci, p0.dev, q.d_idx, q.dev, L * sizeof(int64_t), c0->stream));
      in_cmp[g] = cc;
      in_idx[g] = ci;
    }
    double* d_P = static_cast<double*>(dev_alloc(L * sizeof(double)));
    int64_t* d_I = static_cast<int64_t*>(dev_alloc(L * sizeof(int64_t)));
    if (!d_P || !d_I) s = fail(MPROF_E_OOM, "merge output");
    if (s == MPROF_OK)
      s = mprof_merge_finalize_peers(c0, p0.d_t, n, cfg, in_cmp.data(), in_idx.data(), ndev, &d_P,
                                     &d_I, 1, 0, L);
    if (s == MPROF_OK) {
      CK(cudaMemcpyAsync(P, d_P, L * sizeof(double), cudaMemcpyDeviceToHost, c0->stream));
      CK(cudaMemcpyAsync(I, d_I, L * sizeof(int64_t), cudaMemcpyDeviceToHost, c0->stream));
      CK(cudaStreamSynchronize(c0->stream));
    }
    for (void* q : owned) cudaFree(q);
    return s;
  };
  st = finish();
  if (st == MPROF_OK && info) {
    *info = parts[0].info;
    info->cells = 0;
    info->tiles = 0;
    info->kernel_launches = 0;
    info->sweep_ms = 0.f;
    for (const auto& q : parts) {
      info->cells += q.info.cells;
      info->tiles += q.info.tiles;
      info->kernel_launches += q.info.kernel_launches;
      info->sweep_ms = std::max(info->sweep_ms, q.info.sweep_ms);
    }
    info->diagonals = L - cfg->exclusion;
    info->kernel_launches += 1;  // the fused merge + finalize
  }
  const std::string keep = g_last_error;
  release();
  g_last_error = keep;
  cudaSetDevice(caller_dev);
  return st;
}

uint64_t mprof_band_cells(uint64_t n, uint64_t m, uint64_t k_lo, uint64_t k_hi) {
  const uint64_t L = n - m + 1;
  if (k_hi > L) k_hi = L;
  if (k_lo >= k_hi) return 0;
  // sum_{k=k_lo}^{k_hi-1} (L - k)
  const uint64_t cnt = k_hi - k_lo;
  const uint64_t first = L - k_lo, last = L - (k_hi - 1);
  return (first + last) * cnt / 2;
}

int32_t mprof_band_cuts(uint64_t n, uint64_t m, uint64_t exclusion, uint32_t parts, uint64_t* cuts) {
  if (!cuts || parts == 0) return fail(MPROF_E_BAD_ARG, "bad arguments");
  if (m < 1 || m > n - 1) return fail(MPROF_E_BAD_SUBSEQ_LEN, "bad m");
  if (exclusion < 1 || exclusion > n - m) return fail(MPROF_E_BAD_EXCLUSION, "bad exclusion");
  const uint64_t L = n - m + 1;
  const long double total = (long double)mprof_band_cells(n, m, exclusion, L);
  cuts[0] = exclusion;
  cuts[parts] = L;
  uint64_t lo = exclusion;
  for (uint32_t g = 1; g < parts; ++g) {
    const long double target = total * g / parts;
    // smallest K >= lo with cells(exclusion, K) >= target (binary search)
    uint64_t a = lo, b = L;
    while (a < b) {
      const uint64_t mid = a + (b - a) / 2;
      if ((long double)mprof_band_cells(n, m, exclusion, mid) >= target) b = mid; else a = mid + 1;
    }
    // align to whole diagonal blocks of the tile grid (first tile diagonal exclusion + 1, the
    // prepass sweeps `exclusion`): a band's last block would otherwise be a thin, slow tile row
    const uint64_t base = exclusion + 1;
    if (a > base && a < L) {
      const uint64_t q = (a - base + kK / 2) / kK;
      a = std::min<uint64_t>(L, std::max<uint64_t>(lo, base + q * kK));
    }
    cuts[g] = a;
    lo = a;
  }
  return MPROF_OK;
}

// ---- EngineState ---------------------------------------------------------------------------

int32_t mprof_state_build(mprof_ctx* in, const double* t, uint64_t n, const mprof_config* cfg,
                          mprof_state** out, mprof_run_info* info) {
  if (!t || !cfg || !out) return fail(MPROF_E_BAD_ARG, "null argument");
  *out = nullptr;
  int32_t st = check_series(t, n);
  if (st != MPROF_OK) return st;
  st = check_config(n, cfg);
  if (st != MPROF_OK) return st;
  mprof_ctx* caller = nullptr;
  st = resolve_ctx(in, &caller);
  if (st != MPROF_OK) return st;
  // the state owns its context (stream + workspace): it may be extended or cloned from any thread
  // while the caller's context is in use elsewhere, and it outlives the caller's thread
  mprof_ctx* c = nullptr;
  st = state_ctx(caller, &c);
  if (st != MPROF_OK) return st;
  c->progress = caller->progress;  // a cancelled build leaves an incomplete state
  c->progress_user = caller->progress_user;
  mprof_state* S = new mprof_state();
  S->ctx = c;
  S->cfg = *cfg;
  S->n = n;
  const uint64_t L = n - cfg->m + 1;
  st = ensure(reinterpret_cast<void**>(&S->t), &S->t_bytes, n * sizeof(double));
  if (st == MPROF_OK) st = ensure(reinterpret_cast<void**>(&S->cmp), &S->cmp_bytes, L * sizeof(double));
  if (st == MPROF_OK) st = ensure(reinterpret_cast<void**>(&S->idx), &S->idx_bytes, L * sizeof(int64_t));
  if (st != MPROF_OK) { mprof_state_destroy(S); return st; }
  cudaError_t e = cudaMemcpyAsync(S->t, t, n * sizeof(double), cudaMemcpyHostToDevice, c->stream);
  if (e != cudaSuccess) { mprof_state_destroy(S); return cuda_fail(e, "cudaMemcpyAsync"); }
  mprof_run_info local{};
  st = sweep_impl(c, S->t, n, cfg, 0, 0, S->cmp, S->idx, info ? info : &local);
  c->progress = nullptr;
  c->progress_user = nullptr;
  if (st != MPROF_OK) { mprof_state_destroy(S); return st; }
  S->done = (info ? info : &local)->diagonals;
  S->plan_R = c->plan_R;
  S->plan_flags = plan_flags(c);
  trim_ctx(c);
  *out = S;
  return MPROF_OK;
}

int32_t mprof_state_extend(mprof_state* S, const double* samples, uint64_t count,
                           mprof_run_info* info) {
  if (!S) return fail(MPROF_E_BAD_ARG, "null state");
  if (S->done != state_total(S))  // engine_state.cpp:56-58: checked before anything else
    return fail(MPROF_E_INCOMPLETE_STATE,
                "cannot extend a partially computed profile (%llu of %llu diagonals done)",
                (unsigned long long)S->done, (unsigned long long)state_total(S));
  if (count == 0) {
    if (info) std::memset(info, 0, sizeof *info);
    return MPROF_OK;  // extend_profile with an empty span returns the state unchanged
  }
  if (!samples) return fail(MPROF_E_BAD_ARG, "null samples");
  for (uint64_t i = 0; i < count; ++i)
    if (!std::isfinite(samples[i]))
      return fail(MPROF_E_NON_FINITE, "appended sample %llu is not finite", (unsigned long long)i);
  mprof_ctx* c = S->ctx;
  CK(cudaSetDevice(c->device));
  const mprof_config* cfg = &S->cfg;
  const uint64_t n_old = S->n, n_new = n_old + count;
  int32_t st = check_config(n_new, cfg);
  if (st != MPROF_OK) return st;
  const int m = (int)cfg->m;
  const int L_old = (int)(n_old - m + 1), L_new = (int)(n_new - m + 1);
  const int dL = L_new - L_old;
  // series: grow (device copy of the old samples), append the new ones
  if (S->t_bytes < n_new * sizeof(double)) {
    double* nt = nullptr;
    size_t cap = 0;
    st = ensure(reinterpret_cast<void**>(&nt), &cap, std::max<size_t>(n_new * sizeof(double), 2 * S->t_bytes));
    if (st != MPROF_OK) return st;
    CK(cudaMemcpyAsync(nt, S->t, n_old * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(S->t);
    S->t = nt;
    S->t_bytes = cap;
  }
  CK(cudaMemcpyAsync(S->t + n_old, samples, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  // The extended series is planned exactly as a fresh build would plan it (operands, form probe,
  // rows per tile). When that plan equals the one the stored profile was swept with, every old
  // cell already has its fresh-sweep value: the old entries seed the profile and only the fresh
  // sweep's tiles that hold a new window's cells run (tile_list, l_old), so the result is
  // bit-identical to a fresh profile of the extended series (extend_profile's contract,
  // /root/reference/proj/include/mprof/engine_state.hpp:47-52). Otherwise the whole extended
  // series is swept.
  uint32_t launches = 0;
  Workspace w;
  st = carve(c, L_new, &w);
  if (st != MPROF_OK) return st;
  const bool zn = cfg->family == MPROF_ZNORMALIZED;
  st = prepare_operands(c, S->t, (int)n_new, cfg, w, &launches);
  if (st != MPROF_OK) return st;
  k_init_best<<<grid_for(L_new), 256, 0, c->stream>>>(w.best, zn ? w.B : nullptr, L_new);
  ++launches;
  SeriesPlan plan;
  st = plan_series(c, S->t, (int)n_new, cfg, w, L_new, &launches, &plan);
  if (st != MPROF_OK) return st;
  const bool incremental = plan.R == S->plan_R && plan_flags(c) == S->plan_flags;
  if (incremental) {
    k_seed_prev<<<grid_for(L_old), 256, 0, c->stream>>>(w.best, zn ? w.B : nullptr, S->cmp, S->idx, L_old);
    ++launches;
  }
  SweepOut so;
  const int k_lo = (int)cfg->exclusion;
  st = sweep_tiles(c, S->t, (int)n_new, cfg, w, k_lo, L_new, L_new, !plan.first_diag_done, plan.R,
                   incremental ? L_old : 0, &launches, &so);
  if (st != MPROF_OK) return st;
  if (zn) {
    st = flat_fix(c, w.B, L_new, k_lo, L_new, w, w.best, &launches);
    if (st != MPROF_OK) return st;
  }
  st = ensure(reinterpret_cast<void**>(&S->cmp), &S->cmp_bytes, (size_t)L_new * sizeof(double));
  if (st == MPROF_OK) st = ensure(reinterpret_cast<void**>(&S->idx), &S->idx_bytes, (size_t)L_new * sizeof(int64_t));
  if (st != MPROF_OK) return st;
  k_split<<<grid_for(L_new), 256, 0, c->stream>>>(w.best, S->cmp, S->idx, L_new);
  ++launches;
  CK(cudaGetLastError());
  S->n = n_new;
  S->done = state_total(S);
  S->plan_R = plan.R;
  S->plan_flags = plan_flags(c);
  // cells swept: the tiles' cells (incremental) or the whole extended series
  uint64_t cells = 0;
  if (incremental) {
    for (const int4& tl : c->tiles->h)
      cells += (uint64_t)tile_cells(L_new, tl.x, tl.w, L_new, tl.y, tl.z - tl.y);
  } else {
    cells = mprof_band_cells(n_new, cfg->m, cfg->exclusion, (uint64_t)L_new);
  }
  fill_info(c, cfg, cells, L_new - k_lo, so, launches, info);
  trim_ctx(c);
  return MPROF_OK;
}

int32_t mprof_state_clone(const mprof_state* S, mprof_state** out) {
  if (!S || !out) return fail(MPROF_E_BAD_ARG, "null argument");
  mprof_ctx* c = nullptr;
  int32_t st0 = state_ctx(S->ctx, &c);
  if (st0 != MPROF_OK) return st0;
  CK(cudaStreamSynchronize(S->ctx->stream));  // S's pending work (build / extend) is complete
  mprof_state* R = new mprof_state();
  R->ctx = c;
  R->cfg = S->cfg;
  R->n = S->n;
  R->done = S->done;
  R->plan_R = S->plan_R;
  R->plan_flags = S->plan_flags;
  const uint64_t L = S->n - S->cfg.m + 1;
  int32_t st = ensure(reinterpret_cast<void**>(&R->t), &R->t_bytes, S->n * sizeof(double));
  if (st == MPROF_OK) st = ensure(reinterpret_cast<void**>(&R->cmp), &R->cmp_bytes, L * sizeof(double));
  if (st == MPROF_OK) st = ensure(reinterpret_cast<void**>(&R->idx), &R->idx_bytes, L * sizeof(int64_t));
  if (st != MPROF_OK) { mprof_state_destroy(R); return st; }
  cudaMemcpyAsync(R->t, S->t, S->n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
  cudaMemcpyAsync(R->cmp, S->cmp, L * sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
  cudaMemcpyAsync(R->idx, S->idx, L * sizeof(int64_t), cudaMemcpyDeviceToDevice, c->stream);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) { mprof_state_destroy(R); return cuda_fail(e, "clone"); }
  *out = R;
  return MPROF_OK;
}

uint64_t mprof_state_series_length(const mprof_state* S) { return S ? S->n : 0; }

int32_t mprof_state_profile(mprof_state* S, double* P, int64_t* I, double* cmp) {
  if (!S) return fail(MPROF_E_BAD_ARG, "null state");
  mprof_ctx* c = S->ctx;
  CK(cudaSetDevice(c->device));
  const uint64_t L = S->n - S->cfg.m + 1;
  if (P) {
    int32_t st = ensure(reinterpret_cast<void**>(&S->P), &S->P_bytes, L * sizeof(double));
    if (st != MPROF_OK) return st;
    st = mprof_finalize_device(c, S->t, S->n, S->cmp, S->idx, &S->cfg, S->P);
    if (st != MPROF_OK) return st;
    CK(cudaMemcpyAsync(P, S->P, L * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  if (I) CK(cudaMemcpyAsync(I, S->idx, L * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  if (cmp) CK(cudaMemcpyAsync(cmp, S->cmp, L * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  trim_ctx(c);
  return MPROF_OK;
}

int32_t mprof_state_series(const mprof_state* S, double* t) {
  if (!S || !t) return fail(MPROF_E_BAD_ARG, "null argument");
  CK(cudaSetDevice(S->ctx->device));
  CK(cudaMemcpyAsync(t, S->t, S->n * sizeof(double), cudaMemcpyDeviceToHost, S->ctx->stream));
  CK(cudaStreamSynchronize(S->ctx->stream));
  return MPROF_OK;
}

void mprof_state_destroy(mprof_state* S) {
  if (!S) return;
  if (S->ctx) cudaSetDevice(S->ctx->device);
  if (S->ctx && S->ctx->stream) cudaStreamSynchronize(S->ctx->stream);
  cudaFree(S->t);
  cudaFree(S->cmp);
  cudaFree(S->idx);
  cudaFree(S->P);
  mprof_ctx_destroy(S->ctx);
  delete S;
}

uint64_t mprof_state_completed_diagonals(const mprof_state* S) { return S ? S->done : 0; }

int32_t mprof_state_tail(const mprof_state* S, double* acc) {
  if (!S || !acc) return fail(MPROF_E_BAD_ARG, "null argument");
  if (S->done == 0) return MPROF_OK;
  mprof_ctx* c = S->ctx;
  CK(cudaSetDevice(c->device));
  const int sums = S->cfg.family == MPROF_ZNORMALIZED ? 5 : 1;
  const size_t bytes = (size_t)S->done * sums * sizeof(double);
  double* d = nullptr;
  CK(cudaMallocAsync(&d, bytes, c->stream));
  k_tail<<<grid_for(32LL * (long long)S->done), 256, 0, c->stream>>>(
      S->t, (int)(S->n - S->cfg.m + 1), (int)S->cfg.m, (int)S->cfg.exclusion, (int)S->done,
      S->cfg.family, S->cfg.p, d);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(acc, d, bytes, cudaMemcpyDeviceToHost, c->stream);
  cudaFreeAsync(d, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(e, "mprof_state_tail");
  return MPROF_OK;
}

int32_t mprof_ctx_set_progress(mprof_ctx* in, mprof_progress_fn fn, void* user) {
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  c->progress = fn;
  c->progress_user = user;
  return MPROF_OK;
}

void mprof_plan_destroy(mprof_plan* P) {
  if (!P) return;
  // the context may already be gone (it is borrowed): cudaFree itself waits for the device
  cudaSetDevice(P->device);
  cudaFree(P->ws);
  cudaFree(P->tiles);
  if (P->host_pairs) cudaFreeHost(P->host_pairs);
  mpg::rc_graph_release(P->rc_graph);
  delete P;
}

int32_t mprof_plan_create(mprof_ctx* in, const double* d_t, uint64_t n64, const mprof_config* cfg,
                          uint64_t k_lo64, uint64_t k_hi64, mprof_plan** out) {
  if (!d_t || !cfg || !out) return fail(MPROF_E_BAD_ARG, "null argument");
  *out = nullptr;
  if (n64 < 2) return fail(MPROF_E_TOO_SHORT, "time series needs at least 2 samples");
  int32_t st = check_config(n64, cfg);
  if (st != MPROF_OK) return st;
  if (cfg->precision == MPROF_FP32 && cfg->exact)
    return fail(MPROF_E_BAD_ARG, "the exact (parity) mode is FP64 only");
  mprof_ctx* c = nullptr;
  st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  const int n = (int)n64, L = n - (int)cfg->m + 1;
  mprof_plan* P = new mprof_plan();
  P->ctx = c;
  P->device = c->device;
  P->t = d_t;
  P->n = n64;
  P->cfg = *cfg;
  P->k_lo = (long long)cfg->exclusion;
  P->k_hi = L;
  if (!(k_lo64 == 0 && k_hi64 == 0)) {
    P->k_lo = std::max<long long>(P->k_lo, (long long)k_lo64);
    P->k_hi = std::min<long long>(P->k_hi, (long long)k_hi64);
  }
  auto bail = [&](int32_t s2) { mprof_plan_destroy(P); return s2; };
  if (cudaMalloc(&P->ws, workspace_bytes(L)) != cudaSuccess) {
    cudaGetLastError();
    return bail(fail(MPROF_E_OOM, "plan workspace of %zu bytes", workspace_bytes(L)));
  }
  Workspace w;
  carve_at(static_cast<char*>(P->ws), L, &w);
  uint32_t launches = 0;
  st = prepare_operands(c, d_t, n, cfg, w, &launches);
  c->stats_t = nullptr;  // the statistics live in the plan's workspace, not the context's
  if (st != MPROF_OK) return bail(st);
  const bool zn = cfg->family == MPROF_ZNORMALIZED;
  k_init_best<<<grid_for(L), 256, 0, c->stream>>>(w.best, zn ? w.B : nullptr, L);
  SeriesPlan sp;
  st = plan_series(c, d_t, n, cfg, w, L, &launches, &sp);
  if (st != MPROF_OK) return bail(st);
  P->R = sp.R;
  P->aamp_cov = c->aamp_cov;
  P->zn_colscale = c->zn_colscale;
  P->wide = c->wide;
  P->dense = c->dense;
  P->probe_replays = c->probe_replays;
  P->probe_cells = c->probe_cells;
  if (P->k_lo < P->k_hi) {
    const int k_tile = (!cfg->exact && P->k_lo == (long long)cfg->exclusion) ? (int)P->k_lo + 1 : (int)P->k_lo;
    const Grid g = grid_of(c, cfg, L, L);
    std::vector<int4> tl;
    tile_list(g, k_tile, P->k_hi, P->R, tl, nullptr);
    P->ntiles = (long long)tl.size();
    const bool cov_main = zn ? !c->zn_colscale : c->aamp_cov;
    P->rc_policy = rc_policy_of(c, cfg, P->R);
    arrange_tiles(g, cov_main && !cfg->exact && !knobs().zn_no_near, P->rc_policy >= 0, tl,
                  &P->n_near, &P->n_legacy, &P->bands);
    if (!P->bands.empty()) {  // the window launches' row operands: one host mirror per plan
      const SweepParams pp = make_params(c, d_t, n, cfg, w, L, L);
      const size_t cnt = (size_t)std::max(L - 1, 1);
      const size_t pbytes = cnt * mpg::rc_pair_bytes(P->rc_policy);
      if (cudaMallocHost(&P->host_pairs, pbytes) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(MPROF_E_OOM, "plan operand mirror"));
      }
      const cudaError_t e = cudaMemcpyAsync(P->host_pairs, mpg::rc_pairs(P->rc_policy, pp),
                                            pbytes, cudaMemcpyDeviceToHost, c->stream);
      if (e != cudaSuccess) return bail(cuda_fail(e, "plan operand mirror"));
    }
    if (!tl.empty()) {
      if (cudaMalloc(&P->tiles, tl.size() * sizeof(int4)) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(MPROF_E_OOM, "plan tile table"));
      }
      const cudaError_t e = cudaMemcpyAsync(P->tiles, tl.data(), tl.size() * sizeof(int4),
                                            cudaMemcpyHostToDevice, c->stream);
      if (e != cudaSuccess) return bail(cuda_fail(e, "plan tile table upload"));
    }
  }
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return bail(cuda_fail(e, "mprof_plan_create"));
  *out = P;
  return MPROF_OK;
}

int32_t mprof_plan_sweep(mprof_plan* P, double* d_cmp, int64_t* d_idx, mprof_run_info* info) {
  if (!P || !d_cmp || !d_idx) return fail(MPROF_E_BAD_ARG, "null argument");
  mprof_ctx* c = P->ctx;
  CK(cudaSetDevice(c->device));
  const mprof_config* cfg = &P->cfg;
  const int n = (int)P->n, L = n - (int)cfg->m + 1;
  const bool zn = cfg->family == MPROF_ZNORMALIZED;
  c->aamp_cov = P->aamp_cov;  // with_policy / make_params read the form from the context
  c->zn_colscale = P->zn_colscale;
  c->wide = P->wide;
  c->dense = P->dense;
  c->probe_replays = P->probe_replays;
  c->probe_cells = P->probe_cells;
  Workspace w;
  carve_at(static_cast<char*>(P->ws), L, &w);
  uint32_t launches = 0;
  k_init_best<<<grid_for(L), 256, 0, c->stream>>>(w.best, zn ? w.B : nullptr, L);
  ++launches;
  SweepOut so;
  so.R = P->R;
  so.ntiles = P->ntiles;
  if (P->k_lo < P->k_hi) {
    SweepParams prm = make_params(c, P->t, n, cfg, w, (int)P->k_hi, L);
    prm.tiles = P->tiles;
    prm.R = (int)std::min<long long>(P->R, INT_MAX);
    int32_t st = dispatch_sweep(c, cfg, prm, P->ntiles, P->n_near, P->n_legacy, P->bands,
                                P->rc_policy, P->host_pairs, (int)cfg->exclusion, true, &launches,
                                &so.ms, &so.rc_launches, knobs().no_graph ? nullptr : &P->rc_graph);
    if (st != MPROF_OK) return st;
    if (zn) {
      st = flat_fix(c, w.B, L, (int)P->k_lo, (int)P->k_hi, w, w.best, &launches);
      if (st != MPROF_OK) return st;
    }
  }
  k_split<<<grid_for(L), 256, 0, c->stream>>>(w.best, d_cmp, d_idx, L);
  ++launches;
  CK(cudaGetLastError());
  const uint64_t cells = P->k_lo < P->k_hi ? mprof_band_cells(P->n, cfg->m, (uint64_t)P->k_lo, (uint64_t)P->k_hi) : 0;
  fill_info(c, cfg, cells, P->k_hi - P->k_lo, so, launches, info);
  return MPROF_OK;
}

int32_t mprof_ctx_set_form(mprof_ctx* in, int32_t form) {
  if (form < MPROF_FORM_AUTO || form > MPROF_FORM_DENSE) return fail(MPROF_E_BAD_ARG, "unknown form %d", form);
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  c->form = form;
  c->R_cache.clear();  // keyed on the form flags, not on the override
  return MPROF_OK;
}

int32_t mprof_ctx_set_row_const(mprof_ctx* in, int32_t enabled) {
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  c->rowconst = enabled != 0;
  return MPROF_OK;
}

int32_t mprof_brute_profile(mprof_ctx* in, const double* t, uint64_t n, const mprof_config* cfg,
                            double* P, int64_t* I) {
  if (!t || !cfg || !P || !I) return fail(MPROF_E_BAD_ARG, "null argument");
  int32_t st = check_series(t, n);
  if (st != MPROF_OK) return st;
  st = check_config(n, cfg);  // brute_profile validates but accepts every family
  if (st != MPROF_OK) return st;
  mprof_ctx* c = nullptr;
  st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  const uint64_t L = n - cfg->m + 1;
  const size_t nt = align_up(n * sizeof(double)), nl = align_up(L * sizeof(double));
  st = ensure(&c->io, &c->io_bytes, nt + 4 * nl);
  if (st != MPROF_OK) return st;
  char* base = static_cast<char*>(c->io);
  double* d_t = reinterpret_cast<double*>(base);
  double* d_P = reinterpret_cast<double*>(base + nt);
  int64_t* d_I = reinterpret_cast<int64_t*>(base + nt + nl);
  double* d_mean = reinterpret_cast<double*>(base + nt + 2 * nl);
  double* d_var = reinterpret_cast<double*>(base + nt + 3 * nl);
  CK(cudaMemcpyAsync(d_t, t, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (cfg->family == MPROF_ZNORMALIZED)
    k_moments<<<grid_for((long long)L), 256, 0, c->stream>>>(d_t, (int)L, (int)cfg->m, d_mean, d_var);
  k_brute<<<(unsigned)std::min<uint64_t>(L, 148ull * 64), 256, 0, c->stream>>>(
      d_t, (int)L, (int)cfg->m, (int)cfg->exclusion, cfg->family, cfg->p, cfg->flat_threshold,
      d_mean, d_var, d_P, d_I, nullptr, 0);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(P, d_P, L * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(I, d_I, L * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return MPROF_OK;
}

int32_t mprof_brute_rows(mprof_ctx* in, const double* t, uint64_t n, const mprof_config* cfg,
                         const int64_t* rows, uint64_t nrows, double* P, int64_t* I) {
  if (!t || !cfg || (nrows && (!rows || !P || !I))) return fail(MPROF_E_BAD_ARG, "null argument");
  int32_t st = check_series(t, n);
  if (st != MPROF_OK) return st;
  st = check_config(n, cfg);
  if (st != MPROF_OK) return st;
  const uint64_t L = n - cfg->m + 1;
  for (uint64_t r = 0; r < nrows; ++r)
    if (rows[r] < 0 || (uint64_t)rows[r] >= L)
      return fail(MPROF_E_BAD_ARG, "row %lld outside [0, %llu)", (long long)rows[r], (unsigned long long)L);
  if (nrows == 0) return MPROF_OK;
  if (nrows > (uint64_t)INT_MAX) return fail(MPROF_E_TOO_LARGE, "too many rows");
  mprof_ctx* c = nullptr;
  st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  const size_t nt = align_up(n * sizeof(double)), nl = align_up(L * sizeof(double)),
               nr = align_up(nrows * sizeof(double));
  st = ensure(&c->io, &c->io_bytes, nt + 2 * nl + 3 * nr);
  if (st != MPROF_OK) return st;
  char* base = static_cast<char*>(c->io);
  double* d_t = reinterpret_cast<double*>(base);
  double* d_mean = reinterpret_cast<double*>(base + nt);
  double* d_var = reinterpret_cast<double*>(base + nt + nl);
  int64_t* d_rows = reinterpret_cast<int64_t*>(base + nt + 2 * nl);
  double* d_P = reinterpret_cast<double*>(base + nt + 2 * nl + nr);
  int64_t* d_I = reinterpret_cast<int64_t*>(base + nt + 2 * nl + 2 * nr);
  CK(cudaMemcpyAsync(d_t, t, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(d_rows, rows, nrows * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
  if (cfg->family == MPROF_ZNORMALIZED)
    k_moments<<<grid_for((long long)L), 256, 0, c->stream>>>(d_t, (int)L, (int)cfg->m, d_mean, d_var);
  k_brute<<<(unsigned)std::min<uint64_t>(nrows, 148ull * 64), 256, 0, c->stream>>>(
      d_t, (int)L, (int)cfg->m, (int)cfg->exclusion, cfg->family, cfg->p, cfg->flat_threshold,
      d_mean, d_var, d_P, d_I, d_rows, (int)nrows);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(P, d_P, nrows * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(I, d_I, nrows * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return MPROF_OK;
}

int32_t mprof_fp64_peak(mprof_ctx* in, double* gflops, float* ms_out) {
  mprof_ctx* c = nullptr;
  int32_t st = resolve_ctx(in, &c);
  if (st != MPROF_OK) return st;
  double* d = nullptr;
  CK(cudaMalloc(&d, sizeof(double)));
  const int blocks = c->num_sms * 8, threads = 256, iters = 4096;
  k_dfma_peak<<<blocks, threads, 0, c->stream>>>(d, 64);  // warm-up
  CK(cudaEventRecord(c->ev0, c->stream));
  k_dfma_peak<<<blocks, threads, 0, c->stream>>>(d, iters);
  CK(cudaEventRecord(c->ev1, c->stream));
  CK(cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  cudaFree(d);
  const double flops = 2.0 * 8 * 4 * (double)iters * blocks * threads;
  if (gflops) *gflops = flops / (ms * 1e-3) / 1e9;
  if (ms_out) *ms_out = ms;
  return MPROF_OK;
}

}  // extern "C"
