/*
 * mprof_gpu.h — C ABI of the B200 matrix-profile engine (AAMP / p-norm AAMP / ACAMP).
 *
 * This is the drop-in boundary for the reference's hot path. The reference exposes a C++
 * API (no C ABI); each entry point below replaces one reference symbol and keeps its
 * argument meaning, validation order and error codes:
 *
 *   mprof_aamp        <- mprof::aamp        /root/reference/proj/include/mprof/aamp.hpp:59-60,
 *                                           /root/reference/proj/src/aamp.cpp:7-15
 *   mprof_aamp_pnorm  <- mprof::aamp_pnorm  /root/reference/proj/include/mprof/aamp.hpp:64-65,
 *                                           /root/reference/proj/src/aamp.cpp:17-25
 *   mprof_acamp       <- mprof::acamp       /root/reference/proj/include/mprof/acamp.hpp:100-102,
 *                                           /root/reference/proj/src/acamp.cpp:29-36
 *   mprof_validate    <- mprof::make_time_series + mprof::validate_config
 *                                           /root/reference/proj/src/core.cpp:7-40
 *   mprof_config_init <- mprof::ProfileConfig(m, kind) defaults
 *                                           /root/reference/proj/include/mprof/core.hpp:78-93
 *   mprof_sweep_device / mprof_finalize_device
 *                     <- mprof::detail::run_engine split at its two phases (scan_diagonals,
 *                        then the comparison->distance conversion)
 *                                           /root/reference/proj/src/diag_scan.cpp:89-140
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary. Host entry points
 * take HOST buffers (the series, and caller-allocated P/I of length n-m+1); *_device entry
 * points take DEVICE pointers and run on the context's CUDA stream.
 * There is no CPU fallback: without a CUDA device every compute call returns MPROF_E_CUDA.
 */
#ifndef MPROF_GPU_H
#define MPROF_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPROF_GPU_ABI_VERSION 3

/* Status codes. 1..13 are mprof::ErrorCode + 1 in declaration order
 * (/root/reference/proj/include/mprof/core.hpp:16-30); >= 100 are device-side failures. */
typedef enum mprof_status {
  MPROF_OK = 0,
  MPROF_E_NON_FINITE = 1,
  MPROF_E_TOO_SHORT = 2,
  MPROF_E_EMPTY_INPUT = 3,
  MPROF_E_PARSE_ERROR = 4,
  MPROF_E_BAD_SUBSEQ_LEN = 5,
  MPROF_E_BAD_P = 6,
  MPROF_E_BAD_EXCLUSION = 7,
  MPROF_E_BAD_THRESHOLD = 8,
  MPROF_E_BAD_KIND = 9,
  MPROF_E_OUT_OF_RANGE = 10,
  MPROF_E_DEGENERATE = 11,
  MPROF_E_INCOMPLETE_STATE = 12,
  MPROF_E_IO = 13,
  MPROF_E_CUDA = 100,
  MPROF_E_OOM = 101,
  MPROF_E_BAD_ARG = 102,
  MPROF_E_TOO_LARGE = 103
} mprof_status;

/* mprof::DistanceFamily (core.hpp:64) */
enum { MPROF_EUCLIDEAN = 0, MPROF_PNORM = 1, MPROF_ZNORMALIZED = 2 };
/* mprof::DiagonalOrder (core.hpp:75) — accepted, result is order-independent */
enum { MPROF_ORDER_ASCENDING = 0, MPROF_ORDER_RANDOM = 1 };
/* mprof::AcampVariant (acamp.hpp:95) */
enum { MPROF_ACAMP_SQUARED_DISTANCE = 0, MPROF_ACAMP_FSCORE = 1 };
/* GPU-side additions */
enum { MPROF_FP64 = 0, MPROF_FP32 = 1 };

/* Mirrors mprof::ProfileConfig + DistanceKind (core.hpp:66-93), plus the GPU-only fields
 * `precision` and `exact`. Use mprof_config_init for the reference defaults. */
typedef struct mprof_config {
  uint64_t m;                /* subsequence length */
  int32_t family;            /* MPROF_EUCLIDEAN / MPROF_PNORM / MPROF_ZNORMALIZED */
  int32_t order;             /* DiagonalOrder; ignored by the GPU sweep */
  double p;                  /* p-norm exponent (PNorm only), >= 1 */
  uint64_t exclusion;        /* minimum admissible |i - j|, default 1 */
  uint64_t order_seed;       /* ignored */
  uint64_t refresh_interval; /* incremental steps between direct recomputations, 0 = never */
  double flat_threshold;     /* variance floor for z-normalization, default 1e-12*m */
  int32_t precision;         /* MPROF_FP64 (default) or MPROF_FP32 */
  int32_t exact;             /* 1: parity build — reference arithmetic (no FMA, clamp, runs
                                aligned to refresh_interval) for bit-exact AAMP / p-norm */
} mprof_config;

/* Result-free metadata of one sweep (filled when the pointer is non-null). */
typedef struct mprof_run_info {
  uint64_t cells;            /* admissible cells swept = sum over diagonals of (L - k) */
  uint64_t diagonals;        /* diagonals swept */
  uint64_t tiles;            /* CTAs launched for the sweep kernel */
  uint64_t rows_per_tile;    /* run length R of each tile (seeded directly at its start) */
  uint32_t kernel_launches;  /* kernels launched by this call */
  float sweep_ms;            /* CUDA-event time of the sweep kernel alone (0 if not timed) */
  float fp64_ops_per_cell;   /* FP64-pipe instructions the sweep kernel issues per cell */
  float fp32_ops_per_cell;   /* FP32 instructions per cell (FP32 mode) */
  /* the sweep kernel's policy ("Wide<EuclidCov>", "Znorm<0>", "Euclid", "Pnorm<3>", ...; the
   * diagonal block next to the exclusion zone of a covariance-form sweep runs "Euclid" /
   * "Znorm<1>" on a side stream) and its blocks per hit test */
  char policy[32];
  int32_t hit_group;
  /* form probe (covariance-form sweeps of >= 4e9 cells): replayed blocks / cells of its sample;
   * 0 / 0 when no probe ran */
  uint32_t probe_replays;
  uint64_t probe_cells;
  /* window launches of the constant-row kernel (0: the sweep ran the legacy tile kernel only) */
  uint32_t row_windows;
  uint32_t reserved;
} mprof_run_info;

typedef struct mprof_ctx mprof_ctx;

/* ---- metadata ---------------------------------------------------------------------------- */
int32_t mprof_abi_version(void);
const char* mprof_status_string(int32_t status);
/* Thread-local message of the last failing call (empty if none). */
const char* mprof_last_error(void);

/* ---- configuration ----------------------------------------------------------------------- */
/* ProfileConfig(m, kind) defaults: exclusion 1, ascending, seed 0, refresh 0,
 * flat_threshold 1e-12*m, fp64, exact 0. */
void mprof_config_init(mprof_config* cfg, uint64_t m, int32_t family, double p);
/* make_time_series (NonFinite, TooShort) then validate_config (BadSubseqLen, BadP,
 * BadExclusion, BadThreshold), in the reference's order. */
int32_t mprof_validate(const double* t, uint64_t n, const mprof_config* cfg);
/* Length of the profile, n - m + 1 (core.hpp:99). */
uint64_t mprof_profile_length(uint64_t n, uint64_t m);

/* ---- contexts ---------------------------------------------------------------------------- */
/* A context owns one device's workspace and CUDA stream. ctx == NULL in the calls below means
 * the calling thread's default context on the current device. */
int32_t mprof_ctx_create(int32_t device, mprof_ctx** out);
void mprof_ctx_destroy(mprof_ctx* ctx);
/* Run the context's work on an external stream (cudaStream_t as void*); NULL = own stream. */
int32_t mprof_ctx_set_stream(mprof_ctx* ctx, void* stream);
/* Time the sweep kernel with CUDA events on the launching stream (fills sweep_ms). */
int32_t mprof_ctx_set_timing(mprof_ctx* ctx, int32_t enabled);
/* Anytime observer (ProgressFn, /root/reference/proj/include/mprof/core.hpp:112): when set, the
 * sweeps of this context run in ascending chunks of diagonals (max(1, total/256) per chunk) and
 * fn(diagonals_done, diagonals_total, user) is called after each; returning 0 cancels and the
 * profile holds the exact minimum over the completed diagonals. NULL disables (one launch). */
typedef int32_t (*mprof_progress_fn)(uint64_t done, uint64_t total, void* user);
int32_t mprof_ctx_set_progress(mprof_ctx* ctx, mprof_progress_fn fn, void* user);
/* Filter form of the FP64 fast-mode Euclidean and z-normalized sweeps. AUTO (default): chosen per
 * series (window-scale spread test + form probe). COV: covariance-only filter (EuclidCov /
 * Znorm<0>) with its own hit groups; WIDE: the same with the long hit groups (Wide<...>);
 * ALT: the (delta, sigma) Euclidean kernel / the column-scaled z-norm filter; DENSE: no block
 * filter at all (every cell compared exactly; chosen automatically for noise-like series, also
 * for p-norm p = 1, 2, 3). Every form gives the exact minimum under the same parity rules; this
 * selects which kernel decides it (tests, experiments). Exact and FP32 sweeps ignore it. */
enum { MPROF_FORM_AUTO = 0, MPROF_FORM_COV = 1, MPROF_FORM_WIDE = 2, MPROF_FORM_ALT = 3,
       MPROF_FORM_DENSE = 4 };
int32_t mprof_ctx_set_form(mprof_ctx* ctx, int32_t form);
/* Constant-row sweep (nonzero, the default): the FP64 covariance-only forms (EuclidCov, Znorm<0>
 * and their Wide<> variants, i.e. the sweeps of >= 4e9 cells the form probe confirms) run as a
 * sequence of row-window launches (1920 rows each) with the row operands passed as kernel
 * parameters, i.e. in the constant bank (uniform-register DFMA operands); 0 keeps the
 * single-launch tile kernel. Both paths do the same arithmetic per cell: identical P and I
 * (tests/test_gpu_rowconst.py). Anytime sweeps (a progress observer) use the tile kernel. */
int32_t mprof_ctx_set_row_const(mprof_ctx* ctx, int32_t enabled);

/* ---- reference entry points (host buffers) ------------------------------------------------ */
/* P[L] and I[L], L = n - m + 1, caller-allocated. `threads` (reference: CPU workers) selects
 * nothing on the GPU and is accepted for signature parity. */
int32_t mprof_aamp(mprof_ctx* ctx, const double* t, uint64_t n, const mprof_config* cfg,
                   double* P, int64_t* I, mprof_run_info* info);
int32_t mprof_aamp_pnorm(mprof_ctx* ctx, const double* t, uint64_t n, const mprof_config* cfg,
                         double* P, int64_t* I, mprof_run_info* info);
int32_t mprof_acamp(mprof_ctx* ctx, const double* t, uint64_t n, const mprof_config* cfg,
                    int32_t variant, double* P, int64_t* I, mprof_run_info* info);

/* Brute-force profile (mprof::brute_profile, /root/reference/proj/src/oracle.cpp:95-132): direct
 * distances for every admissible pair with the reference's evaluation order, ties to the smallest
 * j; any family. O(L^2 m) on the GPU — the CLI's `--engine oracle` and an exact checker. */
int32_t mprof_brute_profile(mprof_ctx* ctx, const double* t, uint64_t n, const mprof_config* cfg,
                            double* P, int64_t* I);
/* Brute-force nearest neighbours of selected rows only (same arithmetic as mprof_brute_profile):
 * row rows[r] into P[r], I[r], r < nrows; a row outside [0, L) is MPROF_E_BAD_ARG. Used for full
 * exact-argmin checks of sampled rows at sizes where a whole brute-force profile is too slow. */
int32_t mprof_brute_rows(mprof_ctx* ctx, const double* t, uint64_t n, const mprof_config* cfg,
                         const int64_t* rows, uint64_t nrows, double* P, int64_t* I);

/* ---- device-resident pipeline ------------------------------------------------------------- */
/* Sweeps diagonals k in [k_lo, k_hi) ∩ [exclusion, n - m] of series d_t (device, n doubles) and
 * writes the partial profile in COMPARISON space: d_cmp[L] (double, +inf = untouched) and
 * d_idx[L] (int64, -1 = untouched). k_lo = k_hi = 0 sweeps every admissible diagonal.
 * Comparison spaces: Euclidean D^2; p-norm sum |x-y|^p; z-normalized 1 - Pearson correlation.
 * Partial profiles of disjoint bands merge by the lexicographic (cmp, idx) minimum
 * (MinBuffer::absorb, /root/reference/proj/src/detail/diag_scan.hpp:45-52). No validation of
 * the series values is done here (the host entry points do it). */
int32_t mprof_sweep_device(mprof_ctx* ctx, const double* d_t, uint64_t n, const mprof_config* cfg,
                           uint64_t k_lo, uint64_t k_hi, double* d_cmp, int64_t* d_idx,
                           mprof_run_info* info);
/* Planned band sweeps: mprof_plan_create takes every per-series decision of the sweep of band
 * [k_lo, k_hi) (0, 0 = all) of series d_t ONCE, synchronously -- operand statistics, the filter
 * form (spread test, form probe), rows per tile, the band's tile table -- into a plan that owns
 * its workspace; mprof_plan_sweep then only enqueues kernels on the context's stream (no host
 * synchronisation unless the context times the sweep), so repeated sweeps of a fixed series can
 * be captured in a CUDA graph. Results are identical to mprof_sweep_device's. The series must not
 * change while the plan is used; one plan must not be swept concurrently from two threads. */
typedef struct mprof_plan mprof_plan;
int32_t mprof_plan_create(mprof_ctx* ctx, const double* d_t, uint64_t n, const mprof_config* cfg,
                          uint64_t k_lo, uint64_t k_hi, mprof_plan** out);
int32_t mprof_plan_sweep(mprof_plan* plan, double* d_cmp, int64_t* d_idx, mprof_run_info* info);
void mprof_plan_destroy(mprof_plan* plan);

/* Distances d_P[L] of a (merged) comparison-space profile of series d_t (n samples), the
 * finalization of run_engine (to_distance / f_to_dz, /root/reference/proj/src/detail/diag_scan.hpp:
 * 153-167). Default mode: the distance of each chosen pair (i, d_idx[i]) is recomputed directly
 * (no sliding drift; exact zeros for identical z-normalized windows). exact = 1: the reference's
 * conversion of the comparison value. Untouched entries (idx -1) stay +inf. */
int32_t mprof_finalize_device(mprof_ctx* ctx, const double* d_t, uint64_t n, const double* d_cmp,
                              const int64_t* d_idx, const mprof_config* cfg, double* d_P);
/* Entries [lo, hi) only (d_P indexed absolutely): ranks of a multi-GPU run finalize disjoint
 * slices of the merged profile and all-gather them. */
int32_t mprof_finalize_range_device(mprof_ctx* ctx, const double* d_t, uint64_t n,
                                    const double* d_cmp, const int64_t* d_idx,
                                    const mprof_config* cfg, double* d_P, uint64_t lo,
                                    uint64_t hi);
/* Lexicographic (cmp, idx) merge of two partial profiles in place into (d_cmp, d_idx):
 * the fused peer-memory alternative to the two-pass ncclMin merge. d_other_* may be peer
 * pointers (NVLink) when peer access is enabled. */
int32_t mprof_merge_device(mprof_ctx* ctx, double* d_cmp, int64_t* d_idx,
                           const double* d_other_cmp, const int64_t* d_other_idx, uint64_t L);

/* ---- several processes, several GPUs: fused merge over peer memory ------------------------ */
/* One process per GPU (torch.distributed plumbing): each rank sweeps its band into buffers it
 * allocated with mprof_ipc_alloc, the ranks exchange the 64-byte handles (any host channel) and
 * map each other's buffers with mprof_ipc_open (NVLink peer memory; also works between two
 * processes on one GPU). After a host barrier (every partial complete), rank g calls
 * mprof_merge_finalize_peers on its slice [lo, hi): one kernel loads the W partial (cmp, idx)
 * entries over NVLink, takes their lexicographic minimum (MinBuffer::absorb,
 * /root/reference/proj/src/detail/diag_scan.hpp:45-52), finalizes the distance (as
 * mprof_finalize_range_device) and stores (P, I) into every rank's output buffers. After a
 * second barrier every rank holds the whole profile: this replaces the ncclMin all-reduces,
 * the separate finalize and the all-gather (the scan_diagonals merge of
 * /root/reference/proj/src/detail/diag_scan.hpp:228-256 across processes). */
#define MPROF_MAX_PEERS 16
typedef struct mprof_ipc_handle {
  unsigned char bytes[64]; /* cudaIpcMemHandle_t */
} mprof_ipc_handle;
/* bytes of device memory on the context's device (cudaMalloc, zero-filled) and its handle. */
int32_t mprof_ipc_alloc(mprof_ctx* ctx, uint64_t bytes, void** d_ptr, mprof_ipc_handle* handle);
int32_t mprof_ipc_free(mprof_ctx* ctx, void* d_ptr);
/* Maps another process's allocation; BadArg for a handle of this process's own allocation. */
int32_t mprof_ipc_open(mprof_ctx* ctx, const mprof_ipc_handle* handle, void** d_ptr);
int32_t mprof_ipc_close(mprof_ctx* ctx, void* d_ptr);
/* nin partial profiles (peer_cmp[r], peer_idx[r], each L entries) -> entries [lo, hi) of the
 * merged, finalized (P, I) written into nout output buffer pairs (out_P[r], out_I[r], each L
 * entries, indexed absolutely). 1 <= nin, nout <= MPROF_MAX_PEERS. Asynchronous on the context's
 * stream. */
int32_t mprof_merge_finalize_peers(mprof_ctx* ctx, const double* d_t, uint64_t n,
                                   const mprof_config* cfg, const double* const* peer_cmp,
                                   const int64_t* const* peer_idx, uint32_t nin,
                                   double* const* out_P, int64_t* const* out_I, uint32_t nout,
                                   uint64_t lo, uint64_t hi);

/* ---- streaming extension: EngineState ---------------------------------------------------- */
/* build_engine_state / extend_profile (/root/reference/proj/include/mprof/engine_state.hpp:26-52,
 * /root/reference/proj/src/engine_state.cpp:11-156). The state keeps the series and the
 * comparison-space profile on the device. extend sweeps ONLY the cells that involve an appended
 * window — on the time-reversed series those are rows [0, dL) of every diagonal — and merges
 * them into the stored profile; the result equals a from-scratch profile of the extended series
 * (parity tolerance; the reference's bit-exact cursor replay is CPU arithmetic). */
typedef struct mprof_state mprof_state;
int32_t mprof_state_build(mprof_ctx* ctx, const double* t, uint64_t n, const mprof_config* cfg,
                          mprof_state** out, mprof_run_info* info);
/* NonFinite for a bad sample (nothing changes); count == 0 leaves the state unchanged. */
int32_t mprof_state_extend(mprof_state* st, const double* samples, uint64_t count,
                           mprof_run_info* info);
int32_t mprof_state_clone(const mprof_state* st, mprof_state** out);
uint64_t mprof_state_series_length(const mprof_state* st);
/* P, I (and optionally cmp) of length n - m + 1 to host buffers; any pointer may be NULL. */
int32_t mprof_state_profile(mprof_state* st, double* P, int64_t* I, double* cmp);
/* The state's series (n samples) to a host buffer. */
int32_t mprof_state_series(const mprof_state* st, double* t);
/* Diagonals the build completed, ascending from exclusion (EngineState::completed_diagonals,
 * /root/reference/proj/include/mprof/engine_state.hpp:33): n - m - exclusion + 1 for a complete
 * state; fewer when the build's progress observer cancelled. mprof_state_extend refuses an
 * incomplete state with MPROF_E_INCOMPLETE_STATE (src/engine_state.cpp:56-58). */
uint64_t mprof_state_completed_diagonals(const mprof_state* st);
/* Tail state of every completed diagonal k = exclusion + r at its last cell (pos = n - m - k),
 * evaluated directly on the GPU (EngineState::tail_cursors / znorm_cursors, engine_state.hpp:
 * 34-35): Euclidean / p-norm acc[r] = the comparison-space accumulator; z-normalized
 * acc[5r .. 5r+4] = (sum_left, sum_right, sumsq_left, sumsq_right, dot). */
int32_t mprof_state_tail(const mprof_state* st, double* acc);
void mprof_state_destroy(mprof_state* st);

/* ---- one process, several GPUs ------------------------------------------------------------ */
/* The entry points above on `ndev` devices: the admissible diagonals are split into equal-area
 * bands (mprof_band_cuts), device devices[g] sweeps band g from its own host thread and context,
 * the partial profiles are merged on devices[0] (the lexicographic merge = MinBuffer::absorb,
 * /root/reference/proj/src/detail/diag_scan.hpp:45-52) and finalized there. engine: 0 =
 * mprof_aamp, 1 = mprof_aamp_pnorm, 2 = mprof_acamp (same
 * validation and BadKind rule; both AcampVariants give the same profile). A device may be listed
 * more than once (at most MPROF_MAX_PEERS entries). The partials are merged and finalized by one
 * kernel on devices[0] that reads them over NVLink peer access (copies where peer access is
 * unavailable). This replaces the reference's `threads` worker split
 * (/root/reference/proj/src/detail/diag_scan.hpp:228-256) with a device split; progress
 * observers are not called. */
int32_t mprof_profile_multi(const int32_t* devices, uint32_t ndev, int32_t engine, const double* t,
                            uint64_t n, const mprof_config* cfg, double* P, int64_t* I,
                            mprof_run_info* info);

/* ---- multi-GPU partition (host-side math, no device needed) ------------------------------ */
/* Equal-area cut of the diagonal range [exclusion, n-m] into `parts` contiguous bands; writes
 * parts+1 boundaries (cuts[0] = exclusion, cuts[parts] = n-m+1). Area(k) = L - k cells. Interior
 * cuts are rounded to the nearest exclusion + 1 + multiple of 1024 (whole tile-grid diagonal
 * blocks), which moves at most 512 diagonals. */
int32_t mprof_band_cuts(uint64_t n, uint64_t m, uint64_t exclusion, uint32_t parts,
                        uint64_t* cuts);
/* Cells of band [k_lo, k_hi): sum_{k} (L - k). */
uint64_t mprof_band_cells(uint64_t n, uint64_t m, uint64_t k_lo, uint64_t k_hi);

/* ---- measurement --------------------------------------------------------------------------- */
/* Measured FP64 peak of the current device: independent DFMA chains on every SM, timed with
 * CUDA events. Writes GFLOP/s (DFMA = 2 flops) and the kernel time. */
int32_t mprof_fp64_peak(mprof_ctx* ctx, double* gflops, float* ms);

#ifdef __cplusplus
}
#endif

#endif /* MPROF_GPU_H */
