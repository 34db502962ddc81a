// sweep_rc.cu — the constant-row sweep kernels (see sweep_rc.h for the design).
//
// The kernel is the legacy tile kernel (sweep.cuh: sweep_kernel / run_stage) with three changes:
//  * the tile's rows are cut into windows of kRcW row transitions; launch w sweeps window w of
//    every tile of one row band, seeding the accumulators directly in window 0 (exactly as the
//    legacy kernel seeds its tile) and carrying them through `acc` otherwise;
//  * the row operand pair of transition i comes from the kernel parameter space (RcParams::rows,
//    constant bank 0) through uniform registers instead of shared memory; the stage loop keeps
//    every per-thread address on bumped pointers so that its counters stay uniform (ptxas then
//    emits LDCU + DFMA R, R, UR, R);
//  * replays read their row operands from the operand array in global memory.
// Reference hot loop replaced: /root/reference/proj/src/diag_scan.cpp:7-85.
#include "sweep_rc.h"

#include <algorithm>
#include <cstring>

namespace mpg {

struct RcParams {
  int w;         // window index within the band's tiles
  int zero;      // 0, opaque to the compiler (run_stage_rc's per-thread replay offsets)
  double* acc;   // accumulator carry of the launch's chain: [tile][K]
  double* stash;          // replay stash pool: [SM][kRcSmSlots][super-group][d][thread]
  unsigned* stash_bits;   // per SM bitmap of taken stash slots
  double2 rows[kRcW];  // operand pairs of the window's row transitions
};
static_assert(sizeof(SweepParams) + sizeof(RcParams) <= 32764, "kernel parameter space");

#ifndef MPROF_RC_MINB
#define MPROF_RC_MINB 3
#endif

// Rows per shared-memory stage of the constant-row kernels (their own choice: the window length is
// a multiple of it, and the per-series rows-per-tile plan keeps using the legacy kernel's).
#ifndef MPROF_RC_STAGE
#define MPROF_RC_STAGE 384
#endif
template <class P>
constexpr int rc_stage_rows_of() {
  return MPROF_RC_STAGE;
}

// Shared memory of the constant-row kernel: the legacy layout plus the stash of the accumulators
// at the start of every super-group of kRcSuper blocks (the deferred replays restart there).
#ifndef MPROF_RC_SUPER
#define MPROF_RC_SUPER 8
#endif
constexpr int kRcSuper = MPROF_RC_SUPER;  // blocks per stash (policies with long hit groups)
// Blocks per stash of policy P: MPROF_RC_SUPER_FINE blocks (at least its hit group) when its hit
// group is shorter than kRcSuper: a passing group is then replayed from a stash at most
// MPROF_RC_SUPER_FINE - hit group blocks before it instead of fast-forwarding through up to 7
// blocks -- what the replay-heavy forms (hit groups of 2) need; 0 keeps kRcSuper.
#ifndef MPROF_RC_SUPER_FINE
#define MPROF_RC_SUPER_FINE 2
#endif
template <class P>
constexpr int rc_super_of() {
  constexpr int hg = hit_group_for<P>();
  if constexpr (MPROF_RC_SUPER_FINE == 0 || hg >= kRcSuper) return kRcSuper;
  else return hg > MPROF_RC_SUPER_FINE ? hg : MPROF_RC_SUPER_FINE;
}
// MPROF_RC_STASH_GLOBAL = 1 (default) keeps the stash in global memory instead (64 bytes stored
// per thread per 512 cells), which frees 32 KB of shared memory per CTA at 256-row stages: 3 CTAs
// per SM instead of 2 (C4 AAMP 94.6 -> 90.0 ms). A CTA takes its S / 64 x 8 KB from a pool with
// kRcSmSlots slots per SM (claimed in the SM's bitmap at the start, released at the end), so the
// stash is 148 x 8 x 48 KB = 57 MB that live in L2; a stash per tile of every chain (0.8 GB at C4)
// was written back to HBM as the chains evicted each other: 23 MB per window launch.
#ifndef MPROF_RC_STASH_GLOBAL
#define MPROF_RC_STASH_GLOBAL 1
#endif
template <class P, int D, int T, int S>
constexpr int rc_stash_doubles() { return S / (rc_super_of<P>() * D) * D * T; }
template <class P, int D, int T, int S>
struct RcSmem {
  SweepSmem<P, D, T, S, false> base;
  double stash[MPROF_RC_STASH_GLOBAL ? 1 : rc_stash_doubles<P, D, T, S>()];  // [super-group][d][thread]
};

// The slide of one block without any cell test (bit-identical to the hot loop's and to
// replay_block's arithmetic): fast-forward over a group that did not pass, inside a replayed
// super-group.
template <class P, int D, bool GUARD>
__device__ __forceinline__ Acc<P, D> skip_block(Acc<P, D> acc, int s, int cnt, double p,
                                                const typename P::V2* cA1,
                                                const typename P::V2* cA2,
                                                const typename P::V2* rowA) {
  using V2 = typename P::V2;
#pragma unroll
  for (int u = 0; u < D; ++u) {
    if (GUARD && s + u >= cnt) break;
    const V2 r = rowA[s + u];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int e = u + d;
      acc.a[d] = P::step(acc.a[d], r, e < D ? cA1[e] : cA2[e - D], p);
    }
  }
  return acc;
}

// One stage of S (or cnt < S) row transitions, covariance-only filters (raw covariance keys).
// Same arithmetic, keys, block bounds and exact replays as run_stage, restructured for the
// uniform datapath. What ptxas needs to keep the constant row operands in uniform registers
// (LDCU + DFMA R, R, UR, R; found by inspecting the SASS of each variant, sm_100a, CUDA 12.9):
//  * the constant index is ONE running variable (ci, carried across stages) plus compile-time
//    offsets -- a sum of two loop counters falls back to LDC into vector registers;
//  * no per-thread address is formed from the loop counters: the ring position, the block-table
//    pointers and the replay offsets are per-thread variables bumped alongside;
//  * the loop nest that holds the constant loads contains no atomic, volatile access or trap,
//    not even in a called function: the group loop only records which groups passed (hmask), and
//    the exact replays run after it, restarting from the accumulators stashed in shared memory at
//    the start of each super-group of kRcSuper blocks.
// crow = the window's row operands (kernel parameter space), ci = index in it of the stage's
// first row operand, rowA_g = the same operands in global memory (replays), svz = 0 (opaque to
// the compiler).
template <class P, int D, int T, int S, bool GUARD>
__device__ __forceinline__ void run_stage_rc(RcSmem<P, D, T, S>& rsm, int b, int X0,
                                             typename P::V (&acc)[D], int i0, int cnt, int kt,
                                             int kend, int L, BestEntry* best, double p,
                                             unsigned long long* stats,
                                             const typename P::V2* crow, int& ci,
                                             const typename P::V2* rowA_g, int svz,
                                             typename P::V* gstash) {
  using G = Geo<D, T, S>;
  using V2 = typename P::V2;
  using SMT = SweepSmem<P, D, T, S, false>;
  SMT& sm = rsm.base;
  constexpr bool EQ = SMT::EQ;
  static_assert(SMT::ZQ || SMT::EQ, "constant-row sweep: covariance-only filters");
  constexpr int HG = hit_group_for<P>();
  constexpr int SUP = rc_super_of<P>();      // blocks per stash
  static_assert(SUP % HG == 0 && S % (SUP * D) == 0, "super-groups are whole hit groups");
  constexpr int GPS = SUP / HG;              // hit groups per super-group
  constexpr int NSG = S / (SUP * D);         // super-groups per stage
  static_assert(NSG * GPS <= 32, "one hit bit per group");
  constexpr int RP = G::RING / D * (D + 1);  // padded ring length
  const int xb = threadIdx.x * D;
  V2 cA[D];
  const int q0 = G::pad((X0 + xb) % G::RING);  // padded ring slot of the stage's first operand
  int qc = q0;
#pragma unroll
  for (int d = 0; d < D; ++d) cA[d] = sm.colA[qc + d];
  const float md_f = static_cast<float>(EQ ? g_cell_ctx.md : 0.0);
  // block bound as a raw covariance word (hit <=> max raw(cov) >= bound), INT_MIN = any cell may
  // pass: run_stage's block_theta_cov on explicit table entries
  auto theta_e = [&](const float4 rq, const float4 cq) {
    const float gap = fmaxf(0.f, fmaxf(__fsub_rd(cq.y, rq.z), __fsub_rd(rq.y, cq.z)));
    const float ss = __fmaf_rd(__fmul_rd(md_f, gap), gap, __fadd_rd(rq.x, cq.x));
    const float th = 0.5f * __fsub_rd(__fmul_rd(ss, 1.f - 0x1p-20f), fmaxf(rq.w, cq.w));
    return th > 0.f ? P::cov_bound_raw_f(th) : INT_MIN;
  };
  auto theta_z = [&](const float2 rq, const float2 cq) {
    const float th = fminf(__fmul_rd(rq.x, cq.y), __fmul_rd(cq.x, rq.y));
    return th > 0.f ? P::cov_bound_raw_f(th) : INT_MIN;
  };
  // table pointers, bumped once per super-group (the row tables have a spare entry after the
  // stage's last block: the bound computed from it is never used)
  const float4* ect = &sm.ecol[EQ ? threadIdx.x : 0];
  const float2* zct = &sm.zcol[EQ ? 0 : threadIdx.x];
  const float4* ert = &sm.erow[0];
  const float2* zrt = &sm.zrow[0];
  using V = typename P::V;
  V* stash = (MPROF_RC_STASH_GLOBAL ? gstash : reinterpret_cast<V*>(rsm.stash)) + threadIdx.x;
  unsigned hmask = 0;  // bit (sg * GPS + group): the group passed its block bounds
  int theta_nx;
  if constexpr (EQ) theta_nx = theta_e(ert[0], ect[0]);
  else theta_nx = theta_z(zrt[0], zct[0]);
  const int lim = GUARD ? cnt : S;  // full stages: a compile-time trip count
  int sg = 0;
#pragma unroll 1
  for (int s0 = 0; s0 < lim; s0 += SUP * D, ++sg) {
#pragma unroll
    for (int d = 0; d < D; ++d) stash[(sg * D + d) * T] = acc[d];
#pragma unroll
    for (int gg = 0; gg < GPS; ++gg) {
      bool hit = false;
#pragma unroll
      for (int g = gg * HG; g < (gg + 1) * HG; ++g) {
        const int s = s0 + g * D;
        if (GUARD && s >= cnt) break;
        int qn = qc + (D + 1);
        if (qn >= RP) qn -= RP;
        MPG_CHECK(qn + D <= G::RINGP);
        const V2* nA = &sm.colA[qn];
        const int theta = theta_nx;
        if constexpr (EQ) theta_nx = theta_e(ert[g + 1], ect[g + 1]);
        else theta_nx = theta_z(zrt[g + 1], zct[g + 1]);
        int hmax = INT_MIN;
#pragma unroll
        for (int u = 0; u < D; ++u) {
          if (GUARD && s + u >= cnt) break;
          const V2 r = crow[ci + g * D + u];
          const int row = i0 + s + u + 1;
          int hu = INT_MIN;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            acc[d] = P::step(acc[d], r, cA[(d + u) % D], p);
            int h = P::cov_raw(acc[d]);
            if (GUARD && !((kt + d < kend) && (row + kt + d <= L - 1))) h = INT_MIN;
            hu = max(hu, h);
          }
          hmax = max(hmax, hu);
          cA[u] = nA[u];
        }
        hit |= hmax >= theta;
        qc = qn;
      }
      hmask |= (hit ? 1u : 0u) << (sg * GPS + gg);
    }
    ci += SUP * D;
    if constexpr (EQ) {
      ect += SUP;
      ert += SUP;
    } else {
      zct += SUP;
      zrt += SUP;
    }
  }
  if (hmask == 0) return;
  // ---- deferred exact replays (rare): per super-group with a passing group, restart from its
  // stash; passing groups are replayed block by block, the others fast-forwarded ----
  int* colT = sm.colT[b];
  int sv = svz;  // block offset within the stage, per-thread copy
  int q1 = q0;
#pragma unroll 1
  for (int g2 = 0; g2 < NSG; ++g2) {
    const unsigned bits = (hmask >> (g2 * GPS)) & ((1u << GPS) - 1u);
    if (bits == 0) {
      sv += SUP * D;
      q1 += SUP * (D + 1);
      if (q1 >= RP) q1 -= RP;
      continue;
    }
    Acc<P, D> a0;
#pragma unroll
    for (int d = 0; d < D; ++d) a0.a[d] = stash[(g2 * D + d) * T];
#pragma unroll 1
    for (int g = 0; g < SUP; ++g) {
      if (GUARD && sv >= cnt) break;
      int q2 = q1 + (D + 1);
      if (q2 >= RP) q2 -= RP;
      if ((bits >> (g / HG)) & 1u) {
        a0 = replay_block<P, D, GUARD>(a0, sv, cnt, i0, kt, kend, L, p, &sm.colA[q1], &sm.colA[q2],
                                       &sm.colB[q1], &sm.colB[q2], &colT[G::pad(sv + xb)],
                                       &colT[G::pad(sv + xb + D)], rowA_g, sm.rowB[b], sm.rowT[b],
                                       best, stats);
      } else {
        a0 = skip_block<P, D, GUARD>(a0, sv, cnt, p, &sm.colA[q1], &sm.colA[q2], rowA_g);
      }
      sv += D;
      q1 = q2;
    }
  }
}

template <class P, int D, int T, int S, int MINB>
__global__ void __launch_bounds__(T, MINB)
    sweep_kernel_rc(const SweepParams prm, const __grid_constant__ RcParams rc) {
  using G = Geo<D, T, S>;
  using SM = SweepSmem<P, D, T, S, false>;
  using V = typename P::V;
  using VB = typename P::VB;
  static_assert(kRcW % S == 0, "a window is whole stages");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RcSmem<P, D, T, S>& rsm = *reinterpret_cast<RcSmem<P, D, T, S>*>(smem_raw);
  SM& sm = rsm.base;

  const int4 tl = prm.tiles[blockIdx.x];
  const int kb = tl.x;
  const int ra = tl.y + rc.w * kRcW;  // first row transition of this window
  const int L = prm.L;
  const int m = prm.m;
  const int kt = kb + static_cast<int>(threadIdx.x) * D;
  const int kend = min(min(tl.w, kb + G::K), prm.k_hi);
  // the tile's transitions are [tl.y, tl.z - 1); this window takes at most kRcW of them
  const int left = tl.z - 1 - ra;
  if (rc.w > 0 && left <= 0) return;
  const int steps = min(left, kRcW);
  MPG_CHECK(kb >= 1 && tl.y >= 0 && tl.y < tl.z && tl.z <= L - kb && tl.z <= prm.row_hi &&
            tl.w > kb && tl.w <= L);
  if constexpr (is_euclid_cov<P>()) {
    if (threadIdx.x == 0) g_cell_ctx = CellCtx{prm.S, prm.mu, static_cast<double>(m)};
    __syncthreads();
  }
  // (the carry and the stash are sized for doubles; the FP32 policy uses the front of each part)
  V* carry = reinterpret_cast<V*>(rc.acc) + (static_cast<size_t>(blockIdx.x) * G::K + threadIdx.x * D);
  V acc[D];
  if (rc.w == 0) {
    // ---- seed (FP64): direct length-m sum for the pair (ra, ra + kt + d), as sweep_kernel ----
    double sacc[D];
    double muc[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      sacc[d] = 0.0;
      const int j = ra + kt + d;
      muc[d] = (j < L) ? prm.mu[j] : 0.0;
    }
    {
      constexpr int SL = 2 * S;
      static_assert(sizeof(SM) >= sizeof(double) * (SL + G::pad(G::K + SL)), "seed scratch");
      double* srow = reinterpret_cast<double*>(smem_raw);
      double* scol = srow + SL;
      const double mur = prm.mu[ra];
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
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = static_cast<V>(sacc[d]);
    // the seed cells (ra, ra + k): exact merge
    {
      const VB* Bs = scales_of<P>(prm);
      Cells<D> c;
      unsigned valid = 0;
      const VB rb = Bs[ra];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int k = kt + d;
        const bool ok = (k < kend) && (ra + k <= L - 1);
        const VB cb = ok ? Bs[ra + k] : VB{};
        c.v[d] = ok ? cell_value<P>(acc[d], rb, cb, ra, ra + k) : 0.0;
        valid |= (ok ? 1u : 0u) << d;
      }
      resolve_seed<D>(c, valid, ra, ra + kt, prm.best);
    }
    if (steps <= 0) return;
    __syncthreads();  // seed scratch reuse
  } else {
    if constexpr (sizeof(V) == 8) {  // 16-byte loads
      const double2* cp = reinterpret_cast<const double2*>(carry);
#pragma unroll
      for (int d = 0; d < D; d += 2) {
        const double2 v = __ldcg(cp + d / 2);
        acc[d] = v.x;
        acc[d + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] = __ldcg(carry + d);
    }
  }

  // ---- the CTA's replay stash: a slot of the per-SM pool (claimed in the SM's bitmap, released
  // at the end; the pool has more slots per SM than CTAs can be resident) ----
  V* gstash = nullptr;
  if constexpr (MPROF_RC_STASH_GLOBAL) {
    __shared__ int s_slot;
    if (threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      int got = -1;
      while (got < 0) {
        for (int bsl = 0; bsl < kRcSmSlots && got < 0; ++bsl) {
          const unsigned bit = 1u << bsl;
          if (!(atomicOr(&rc.stash_bits[smid], bit) & bit)) got = bsl;
        }
      }
      s_slot = static_cast<int>(smid) * kRcSmSlots + got;
    }
    __syncthreads();
    gstash = reinterpret_cast<V*>(rc.stash) + static_cast<size_t>(s_slot) * rc_stash_doubles<P, D, T, S>();
  }

  // ---- stage pipeline over the window's row transitions (sweep_kernel's, rows from rc.rows) --
  const typename P::V2* A = pairs_of<P>(prm);
  const int nst = (steps + S - 1) / S;
  load_stage<P, D, T, S, false>(sm, prm, 0, ra, kb);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  stage_block_max<P, D, T, S, false>(sm, 0, 0);
  if (nst > 1) load_stage<P, D, T, S, false>(sm, prm, 1, ra, kb);
  cp_async_commit();
  __syncthreads();
  int ci = 0;  // running index in rc.rows of the next stage's first row operand
  for (int st = 0; st < nst; ++st) {
    const int s0 = st * S;
    const int cnt = min(S, steps - s0);
    const int i0 = ra + s0;
    const bool full = (cnt == S) && (kb + G::K <= kend) && (i0 + cnt + kb + G::K - 1 <= L - 1);
    if (full) {
      run_stage_rc<P, D, T, S, false>(rsm, st & 1, s0, acc, i0, cnt, kt, kend, L, prm.best, prm.p,
                                      prm.stats, reinterpret_cast<const typename P::V2*>(rc.rows), ci,
                                      A + i0, rc.zero, gstash);
    } else {
      run_stage_rc<P, D, T, S, true>(rsm, st & 1, s0, acc, i0, cnt, kt, kend, L, prm.best, prm.p,
                                     prm.stats, reinterpret_cast<const typename P::V2*>(rc.rows), ci,
                                      A + i0, rc.zero, gstash);
    }
    if (st + 1 == nst) break;
    cp_async_wait<0>();
    __syncthreads();
    stage_block_max<P, D, T, S, false>(sm, (st + 1) & 1, s0 + S);
    if (st + 2 < nst) load_stage<P, D, T, S, false>(sm, prm, st + 2, ra, kb);
    cp_async_commit();
    __syncthreads();
  }
  if constexpr (MPROF_RC_STASH_GLOBAL) {
    __syncthreads();  // every thread is done with the stash
    if (threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      const int bsl = (static_cast<int>((gstash - reinterpret_cast<V*>(rc.stash)) / rc_stash_doubles<P, D, T, S>())) % kRcSmSlots;
      atomicAnd(&rc.stash_bits[smid], ~(1u << bsl));
    }
  }
  // more transitions of this tile follow in the next window: carry the accumulators
  if (left > kRcW) {
    if constexpr (sizeof(V) == 8) {
      double2* cp = reinterpret_cast<double2*>(carry);
#pragma unroll
      for (int d = 0; d < D; d += 2) __stcg(cp + d / 2, make_double2(acc[d], acc[d + 1]));
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) __stcg(carry + d, acc[d]);
    }
  }
}

namespace {

constexpr int kD = 8, kT = 128;

template <class P>
auto rc_kernel() {
  return sweep_kernel_rc<P, kD, kT, rc_stage_rows_of<P>(), MPROF_RC_MINB>;
}

template <class P>
size_t rc_smem() {
  return sizeof(RcSmem<P, kD, kT, rc_stage_rows_of<P>()>);
}

template <class F>
auto with_rc_policy(int policy, F&& f) {
#ifdef RC_ONLY_WZ  // experiments: one instantiation for quick SASS checks
  return f.template operator()<Wide<Znorm<false>>>();
#else
  switch (policy) {
    case kRcZnorm: return f.template operator()<Znorm<false>>();
    case kRcWideZnorm: return f.template operator()<Wide<Znorm<false>>>();
    case kRcEuclidCov: return f.template operator()<EuclidCov>();
    case kRcZnormF32: return f.template operator()<ZnormF32<false>>();
    default: return f.template operator()<Wide<EuclidCov>>();
  }
#endif
}

cudaError_t ensure_res(RcRes& res, size_t tiles, size_t per_tile, size_t stash_doubles) {
  cudaError_t e;
  if (!res.fork) {
    if ((e = cudaEventCreateWithFlags(&res.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
    for (int s = 0; s < kRcSlots; ++s) {
      if ((e = cudaStreamCreateWithFlags(&res.st[s], cudaStreamNonBlocking)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&res.join[s], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
  }
  // grow-only: a pool sized for the largest slot serves every policy (each kernel strides the pool
  // by its own slot size), so alternating policies on one context do not reallocate
  if (stash_doubles > 0 && (stash_doubles > res.stash_slot_doubles || !res.stash)) {
    int dev = 0, sms = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if (res.stash) cudaFree(res.stash);
    if (res.stash_bits) cudaFree(res.stash_bits);
    res.stash = nullptr;
    res.stash_bits = nullptr;
    if ((e = cudaMalloc(&res.stash, sizeof(double) * stash_doubles * sms * kRcSmSlots)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&res.stash_bits, sizeof(unsigned) * sms)) != cudaSuccess) return e;
    if ((e = cudaMemset(res.stash_bits, 0, sizeof(unsigned) * sms)) != cudaSuccess) return e;
    res.stash_slot_doubles = stash_doubles;
    res.stash_sms = sms;
  }
  if (tiles * per_tile > res.acc_tiles * res.acc_per_tile || per_tile != res.acc_per_tile) {
    if (res.acc) cudaFree(res.acc);
    res.acc = nullptr;
    res.acc_tiles = 0;
    if ((e = cudaMalloc(&res.acc, sizeof(double) * per_tile * tiles * kRcSlots)) != cudaSuccess) return e;
    res.acc_tiles = tiles;
    res.acc_per_tile = per_tile;
  }
  return cudaSuccess;
}

}  // namespace

int rc_stage_rows(int policy) {
  return with_rc_policy(policy, [&]<class P>() { return rc_stage_rows_of<P>(); });
}

int rc_blocks_per_sm(int policy) {
  return with_rc_policy(policy, [&]<class P>() {
    int nb = 1;
    auto kern = rc_kernel<P>();
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rc_smem<P>()) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kT, rc_smem<P>()) != cudaSuccess)
      nb = 1;
    cudaGetLastError();
    return std::max(1, nb);
  });
}

namespace {

// Enqueues the window chain: fork from `main`, the bands' window launches round-robin over the
// chain streams, join back into `main`.
template <class P>
cudaError_t rc_issue(const SweepParams& prm, const std::vector<RcBand>& bands, RcRes& res,
                     cudaStream_t main, const unsigned char* host_pairs, size_t per_tile,
                     uint32_t* launches) {
  auto kern = rc_kernel<P>();
  const size_t smem = rc_smem<P>();
  cudaError_t e2;
  if ((e2 = cudaEventRecord(res.fork, main)) != cudaSuccess) return e2;
  for (int s = 0; s < kRcSlots; ++s)
    if ((e2 = cudaStreamWaitEvent(res.st[s], res.fork, 0)) != cudaSuccess) return e2;
  // band i runs on chain i % kRcSlots; the chains are issued round-robin, one window launch at
  // a time, so the streams advance together
  size_t next_band[kRcSlots];
  int next_w[kRcSlots];
  for (int s = 0; s < kRcSlots; ++s) {
    next_band[s] = (size_t)s;
    next_w[s] = 0;
  }
  RcParams rc;
  rc.zero = 0;
  for (bool any = true; any;) {
    any = false;
    for (int s = 0; s < kRcSlots; ++s) {
      while (next_band[s] < bands.size() && next_w[s] >= (int)bands[next_band[s]].count.size()) {
        next_band[s] += kRcSlots;
        next_w[s] = 0;
      }
      if (next_band[s] >= bands.size()) continue;
      any = true;
      const RcBand& bd = bands[next_band[s]];
      const int w = next_w[s]++;
      const int nt = bd.count[w];
      if (nt <= 0) continue;
      const long long r0 = (long long)bd.ra + (long long)w * kRcW;
      const long long rows = std::min<long long>(kRcW, (long long)prm.L - 1 - r0);
      if (rows > 0)
        std::memcpy(rc.rows, host_pairs + (size_t)r0 * sizeof(typename P::V2),
                    (size_t)rows * sizeof(typename P::V2));
      SweepParams q = prm;
      q.tiles = prm.tiles + bd.off;
      rc.w = w;
      rc.acc = res.acc + (size_t)s * res.acc_tiles * per_tile;
      rc.stash = res.stash;
      rc.stash_bits = res.stash_bits;
      kern<<<(unsigned)nt, kT, smem, res.st[s]>>>(q, rc);
      if ((e2 = cudaGetLastError()) != cudaSuccess) return e2;
      ++*launches;
    }
  }
  for (int s = 0; s < kRcSlots; ++s) {
    if ((e2 = cudaEventRecord(res.join[s], res.st[s])) != cudaSuccess) return e2;
    if ((e2 = cudaStreamWaitEvent(main, res.join[s], 0)) != cudaSuccess) return e2;
  }
  return cudaSuccess;
}

}  // namespace

const void* rc_pairs(int policy, const SweepParams& prm) {
  if (policy == kRcZnormF32) return prm.A32;
  return (policy == kRcEuclidCov || policy == kRcWideEuclidCov) ? prm.A2 : prm.A;
}

size_t rc_pair_bytes(int policy) { return policy == kRcZnormF32 ? sizeof(float2) : sizeof(double2); }

void rc_graph_release(RcGraph& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  g = RcGraph{};
}

cudaError_t rc_sweep(int policy, const SweepParams& prm, const std::vector<RcBand>& bands,
                     RcRes& res, cudaStream_t main, const void* host_pairs_v, uint32_t* launches,
                     RcGraph* graph) {
  const unsigned char* host_pairs = static_cast<const unsigned char*>(host_pairs_v);
  if (bands.empty()) return cudaSuccess;
  size_t most = 0;
  for (const RcBand& bd : bands)
    if (!bd.count.empty()) most = std::max<size_t>(most, (size_t)bd.count[0]);
  if (most == 0) return cudaSuccess;
  return with_rc_policy(policy, [&]<class P>() -> cudaError_t {
    constexpr size_t per_tile = (size_t)kD * kT;
    constexpr size_t stash_doubles = MPROF_RC_STASH_GLOBAL ? rc_stash_doubles<P, kD, kT, rc_stage_rows_of<P>()>() : 0;
    cudaError_t e = ensure_res(res, most, per_tile, stash_doubles);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(rc_kernel<P>(), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rc_smem<P>());
    if (e != cudaSuccess) return e;
    if (graph && !prm.stats) {
      // a graph is valid for the buffers its launches were captured with
      if (graph->exec && (graph->acc != res.acc || graph->stash != res.stash ||
                          graph->tiles != prm.tiles || graph->best != prm.best))
        rc_graph_release(*graph);
      if (!graph->exec) {
        cudaGraph_t g = nullptr;
        uint32_t n = 0;
        if (cudaStreamBeginCapture(main, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
          const cudaError_t ei = rc_issue<P>(prm, bands, res, main, host_pairs, per_tile, &n);
          const cudaError_t ec = cudaStreamEndCapture(main, &g);
          if (ei == cudaSuccess && ec == cudaSuccess && g &&
              cudaGraphInstantiate(&graph->exec, g, 0) == cudaSuccess) {
            graph->acc = res.acc;
            graph->stash = res.stash;
            graph->tiles = prm.tiles;
            graph->best = prm.best;
            graph->launches = n;
          } else {
            graph->exec = nullptr;
          }
          if (g) cudaGraphDestroy(g);
        }
        cudaGetLastError();  // a stream that cannot be captured: direct launches below
      }
      if (graph->exec) {
        if ((e = cudaGraphLaunch(graph->exec, main)) != cudaSuccess) return e;
        *launches += graph->launches;
        return cudaSuccess;
      }
    }
    return rc_issue<P>(prm, bands, res, main, host_pairs, per_tile, launches);
  });
}

void rc_release(RcRes& res) {
  for (int s = 0; s < kRcSlots; ++s) {
    if (res.st[s]) {
      cudaStreamSynchronize(res.st[s]);
      cudaStreamDestroy(res.st[s]);
      res.st[s] = nullptr;
    }
    if (res.join[s]) {
      cudaEventDestroy(res.join[s]);
      res.join[s] = nullptr;
    }
  }
  if (res.fork) {
    cudaEventDestroy(res.fork);
    res.fork = nullptr;
  }
  if (res.acc) cudaFree(res.acc);
  res.acc = nullptr;
  res.acc_tiles = 0;
  if (res.stash) cudaFree(res.stash);
  if (res.stash_bits) cudaFree(res.stash_bits);
  res.stash = nullptr;
  res.stash_bits = nullptr;
  res.stash_slot_doubles = 0;
}

}  // namespace mpg
