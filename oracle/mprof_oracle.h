/*
 * mprof_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU algorithm for the matrix-profile hot path
 * (diagonal scan + MinBuffer + comparison spaces + brute-force oracle), used as the parity
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg. Nothing in the
 * product (paper_1901_05708_b200/) may link or call it.
 *
 * Pinned by tests/test_oracle_pin.py against (a) the reference's own golden vectors and
 * known-answer tests and (b) the reference library itself built from /root/reference into
 * oracle/_ref (bit-exact comparison on seeded corpora).
 */
#ifndef MPROF_ORACLE_H
#define MPROF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_EUCLIDEAN = 0, OR_PNORM = 1, OR_ZNORM = 2 };

/* step primitives (bit-exact restatements) */
double or_abs_pow(double x, double p);
double or_incremental_euclidean_step(double acc, double oi, double oj, double ii, double ij);
double or_incremental_pnorm_step(double acc, double oi, double oj, double ii, double ij, double p);
typedef struct or_stats {
  double sum_left, sum_right, sumsq_left, sumsq_right, dot;
  uint64_t offset, pos;
} or_stats;
or_stats or_direct_stats(const double* t, uint64_t i, uint64_t j, uint64_t m);
or_stats or_advance_stats(or_stats s, double oi, double oj, double ii, double ij);
double or_f_value(const or_stats* s, double m, double scaled_flat);
double or_znorm_sq_from_stats(const or_stats* s, uint64_t m, double flat_threshold);
double or_f_to_dz(double f, uint64_t m);
double or_direct_sq_acc(const double* t, uint64_t i, uint64_t j, uint64_t m);
double or_direct_pnorm_acc(const double* t, uint64_t i, uint64_t j, uint64_t m, double p);

/* Full diagonal scan (run_engine). use_f: 1 = FScore, 0 = SquaredDistance (z-norm only).
 * Diagonals [max(k_lo, excl), min(k_hi, L)); k_lo = k_hi = 0 means all. threads >= 1.
 * Outputs (any may be NULL): cmp[L] comparison values, P[L] distances, I[L] neighbours. */
void or_scan(const double* t, uint64_t n, uint64_t m, int family, double p, uint64_t excl,
             uint64_t refresh, double flat_threshold, int use_f, uint64_t k_lo, uint64_t k_hi,
             int threads, double* cmp, double* P, int64_t* I);

/* Direct distances (oracle.cpp) and the O(n^2 m) brute profile (smallest j wins ties). */
double or_dist(const double* t, uint64_t i, uint64_t j, uint64_t m, int family, double p,
               double flat_threshold);
void or_brute_profile(const double* t, uint64_t n, uint64_t m, int family, double p,
                      uint64_t excl, double flat_threshold, double* P, int64_t* I);

/* Well-conditioned long-double distance d*(i,j) for parity rule 3: direct sum
 * for Euclidean / p-norm; two-pass centred moments for z-norm (flat rule as the reference). */
double or_dist_exact(const double* t, uint64_t i, uint64_t j, uint64_t m, int family, double p,
                     double flat_threshold);
/* d*(i, j) for many (i, j) pairs (OpenMP-free, threaded by caller count). */
void or_dist_exact_many(const double* t, uint64_t m, int family, double p, double flat_threshold,
                        const int64_t* i, const int64_t* j, uint64_t count, double* out);
/* Exact full-row argmin for sampled rows: best[r], arg[r] over all admissible j. */
void or_exact_rows(const double* t, uint64_t n, uint64_t m, int family, double p, uint64_t excl,
                   double flat_threshold, const int64_t* rows, uint64_t count, int threads,
                   double* best, int64_t* arg);

#ifdef __cplusplus
}
#endif
#endif
