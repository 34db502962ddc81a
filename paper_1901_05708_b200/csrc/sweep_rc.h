// sweep_rc.h — host interface of the constant-row sweep (csrc/sweep_rc.cu).
//
// The covariance-only FP64 sweeps (Znorm<0>, EuclidCov and their Wide<> forms) are bound by the
// register-file reads of their DFMAs: with the row operand in a vector register every second DFMA
// reads three 64-bit registers and dispatches in 3 cycles against its 2-cycle pipe slot
// (DESIGN.md §4). The row operand is the same for every thread of the grid that works on the same
// row, so this path puts it in the CONSTANT bank: the sweep runs as a sequence of row WINDOWS of
// kRcW rows, one launch per window, whose row operands travel as a KERNEL PARAMETER (30 KB of the
// 32 KB parameter space, bank 0; the host keeps a pinned copy of the operand array); the kernel
// reads them with LDCU into uniform registers and its DFMAs take a uniform-register operand
// (DFMA R, R, UR, R: two vector register reads). A tile (1024 diagonals x R rows, the legacy
// kernel's CTA) becomes ceil(R / kRcW) consecutive window launches that carry their accumulators
// through a global buffer; the tiles that start at the same row form a band whose windows are
// chained on one stream, and the bands run concurrently on kRcSlots streams (each launch has at
// most L / 1024 CTAs: the chains fill each other's tails). Every cell keeps the arithmetic of the
// legacy kernel (same seeds on the same row grid, same slide order), so the two paths give
// bit-identical profiles (tests/test_gpu_rowconst.py).
// (A __constant__ array refilled by stream-ordered device copies was measured first: 64 KB hold
// only 2 x 2048 or 8 x 512 rows, i.e. few chains or short windows: C4 AAMP 114.7 / 102.5 ms.)
//
// Reference hot loop replaced: EuclidScan / ZnormScan driven by scan_diagonals
// (/root/reference/proj/src/diag_scan.cpp:7-85, src/detail/diag_scan.hpp:193-259).
#pragma once

#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "sweep.cuh"

namespace mpg {

// Rows per window (operand pairs of 16 bytes in the kernel parameter space, which holds 32 764
// bytes in all; 1920 = 5 stages of 384 rows) and concurrent band chains (streams). Measured on C4
// (sweep ms AAMP / ACAMP): 1920-row windows of 128-row stages, 8 chains 96.2 / 97.2, 16 chains
// 95.0 / 96.3; 1792-row windows of 256-row stages (stash in global memory, 3 CTAs/SM), 8 chains
// 91.7 / 92.4, 16 chains 90.0 / 91.5; 1920-row windows of 384-row stages (the longest stage that
// keeps 3 CTAs/SM: 72 KB of shared memory without row-operand buffers), 16 chains 87.8 / 88.6.
// 32 chains (one per row band at C4) measure the same on one GPU (86.6 / 86.8) but matter when a
// GPU sweeps 1/8 of the diagonals: its launches have ~100 CTAs, a chain's windows run one after
// the other, and with 16 chains the 36 windows per chain (~300 us each) bound the band at
// 12.7-14.3 ms; with 32 chains the slowest of 8 bands takes 11.8 / 11.6 ms (92 % / 94 % of 1/8).
#ifndef MPROF_RC_W
#define MPROF_RC_W 1920
#endif
#ifndef MPROF_RC_CHAINS
#define MPROF_RC_CHAINS 32
#endif
constexpr int kRcW = MPROF_RC_W;
constexpr int kRcSlots = MPROF_RC_CHAINS;
constexpr int kRcSmSlots = 4;   // stash slots per SM (>= resident CTAs per SM: 3)
static_assert(kRcW * 16 <= 30720, "the row window must fit the kernel parameter space");

// (kRcZnormF32: the FP32 mode's covariance-only z-norm kernel; its FFMAs take the row operand from
// a uniform register the same way)
enum RcPolicy { kRcZnorm = 0, kRcWideZnorm = 1, kRcEuclidCov = 2, kRcWideEuclidCov = 3, kRcZnormF32 = 4 };

// One row band of the tile grid: the tiles that start at row `ra` (ascending first diagonal, so
// their row ends are non-increasing and the tiles still alive in window w are a prefix), at
// offset `off` of the device tile table; count[w] = tiles with a row transition in window w
// (windows of kRcW rows from `ra`; count[0] = every tile: window 0 also merges the seed cells).
struct RcBand {
  int off = 0;
  int ra = 0;
  std::vector<int> count;
};

// Streams, events and the accumulator carry buffer of one context.
struct RcRes {
  cudaStream_t st[kRcSlots] = {};
  cudaEvent_t fork = nullptr;
  cudaEvent_t join[kRcSlots] = {};
  double* acc = nullptr;     // kRcSlots (chains) x acc_tiles x K doubles
  size_t acc_tiles = 0;
  size_t acc_per_tile = 0;   // doubles per tile: the carry (K)
  // replay stash pool: one slot per resident CTA (kRcSmSlots per SM, claimed in a per-SM bitmap),
  // so the stash stays a few tens of MB that live in L2 whatever the number of tiles
  double* stash = nullptr;
  unsigned* stash_bits = nullptr;   // per SM: bit b set = slot b taken
  size_t stash_slot_doubles = 0;
  int stash_sms = 0;
};

// A captured window chain (planned sweeps): the ~600 launches of a sweep, each with 30 KB of
// parameters, cost the host ~20 us apiece, which binds a GPU that sweeps only 1/8 of the
// diagonals; a plan captures its chain once in a CUDA graph and replays it with one launch.
struct RcGraph {
  cudaGraphExec_t exec = nullptr;
  const double* acc = nullptr;   // the carry buffer the graph's launches point into
  const double* stash = nullptr; // and the stash pool
  const int4* tiles = nullptr;   // and their tile table
  BestEntry* best = nullptr;
  uint32_t launches = 0;
};
void rc_graph_release(RcGraph& g);

// Rows per shared-memory stage of the policy's constant-row kernel.
int rc_stage_rows(int policy);

// Resident CTAs per SM of the policy's constant-row kernel.
int rc_blocks_per_sm(int policy);

// Sweeps the bands' tiles (prm.tiles = device table the band offsets index) with the constant-row
// kernel of `policy`: window launches chained per band on the context's chain streams, forked
// from and joined to `main`. host_pairs = host copy of the policy's operand pairs (prm.A, or
// prm.A2 for the covariance-form AAMP), L - 1 entries. Adds the kernel launches to *launches.
// graph != nullptr: replay (or first capture) the chain as a CUDA graph; falls back to direct
// launches when the stream cannot be captured.
cudaError_t rc_sweep(int policy, const SweepParams& prm, const std::vector<RcBand>& bands,
                     RcRes& res, cudaStream_t main, const void* host_pairs, uint32_t* launches,
                     RcGraph* graph = nullptr);

// Device pointer of the policy's operand pairs in prm (what host_pairs must mirror).
const void* rc_pairs(int policy, const SweepParams& prm);
// Bytes of one operand pair of the policy (double2, or float2 in FP32 mode).
size_t rc_pair_bytes(int policy);

void rc_release(RcRes& res);

}  // namespace mpg
