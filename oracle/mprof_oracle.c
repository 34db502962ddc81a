/*
 * mprof_oracle.c — TEST INFRASTRUCTURE ONLY (see mprof_oracle.h).
 *
 * Plain-C restatement of the reference's CPU hot path. Every function cites the reference
 * lines it restates (paths relative to /root/reference/proj/). Compiled WITHOUT floating-point
 * contraction (-ffp-contract=off), like the reference's x86-64 SSE2 build, so the scan below is
 * bit-identical to mprof::aamp / aamp_pnorm / acamp (pinned by tests/test_oracle_pin.py).
 */
#include "mprof_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* --- step primitives ----------------------------------------------------------------------- */

/* include/mprof/aamp.hpp:13-20 (detail::abs_pow); identical copy in src/oracle.cpp:17-24 */
double or_abs_pow(double x, double p) {
  const double a = fabs(x);
  if (p == 1.0) return a;
  if (p == 2.0) return a * a;
  if (p == 3.0) return a * a * a;
  if (p == 4.0) return (a * a) * (a * a);
  return pow(a, p);
}

/* std::max(0.0, x) == (0.0 < x) ? x : 0.0 (NaN -> 0) */
static inline double max0(double x) { return (0.0 < x) ? x : 0.0; }
/* std::min(a, b) == (b < a) ? b : a */
static inline double minab(double a, double b) { return (b < a) ? b : a; }

/* include/mprof/aamp.hpp:37-42 */
double or_incremental_euclidean_step(double acc, double oi, double oj, double ii, double ij) {
  const double out = oi - oj;
  const double in = ii - ij;
  return max0(acc - out * out + in * in);
}

/* include/mprof/aamp.hpp:45-49 */
double or_incremental_pnorm_step(double acc, double oi, double oj, double ii, double ij, double p) {
  return max0(acc - or_abs_pow(oi - oj, p) + or_abs_pow(ii - ij, p));
}

/* src/detail/diag_scan.hpp:57-64 */
double or_direct_sq_acc(const double* t, uint64_t i, uint64_t j, uint64_t m) {
  double acc = 0.0;
  for (uint64_t l = 0; l < m; ++l) {
    const double d = t[i + l] - t[j + l];
    acc += d * d;
  }
  return acc;
}

/* src/detail/diag_scan.hpp:66-71 */
double or_direct_pnorm_acc(const double* t, uint64_t i, uint64_t j, uint64_t m, double p) {
  double acc = 0.0;
  for (uint64_t l = 0; l < m; ++l) acc += or_abs_pow(t[i + l] - t[j + l], p);
  return acc;
}

/* src/detail/diag_scan.hpp:73-87 (bit-identical to the hoisted seed, diag_scan.cpp:58-69) */
or_stats or_direct_stats(const double* t, uint64_t i, uint64_t j, uint64_t m) {
  or_stats s;
  memset(&s, 0, sizeof s);
  s.offset = j - i;
  s.pos = i;
  for (uint64_t l = 0; l < m; ++l) {
    const double a = t[i + l];
    const double b = t[j + l];
    s.sum_left += a;
    s.sum_right += b;
    s.sumsq_left += a * a;
    s.sumsq_right += b * b;
    s.dot += a * b;
  }
  return s;
}

/* include/mprof/acamp.hpp:28-37 */
or_stats or_advance_stats(or_stats s, double oi, double oj, double ii, double ij) {
  s.sum_left = s.sum_left - oi + ii;
  s.sum_right = s.sum_right - oj + ij;
  s.sumsq_left = s.sumsq_left - oi * oi + ii * ii;
  s.sumsq_right = s.sumsq_right - oj * oj + ij * ij;
  s.dot = s.dot - oi * oj + ii * ij;
  s.pos += 1;
  return s;
}

/* include/mprof/acamp.hpp:42-47 */
static inline double scaled_var_left(const or_stats* s, double m) {
  return s->sumsq_left - s->sum_left * s->sum_left / m;
}
static inline double scaled_var_right(const or_stats* s, double m) {
  return s->sumsq_right - s->sum_right * s->sum_right / m;
}

/* include/mprof/acamp.hpp:52-60 */
double or_f_value(const or_stats* s, double m, double scaled_flat) {
  const double va = scaled_var_left(s, m);
  const double vb = scaled_var_right(s, m);
  const int flat_a = va <= scaled_flat;
  const int flat_b = vb <= scaled_flat;
  if (flat_a || flat_b) return (flat_a && flat_b) ? -(m * m) : 0.0;
  const double g = s->sum_left * s->sum_right - m * s->dot;
  return g * fabs(g) / (va * vb);
}

/* include/mprof/acamp.hpp:66-76 */
double or_znorm_sq_from_stats(const or_stats* s, uint64_t m, double flat_threshold) {
  const double md = (double)m;
  const double va = scaled_var_left(s, md);
  const double vb = scaled_var_right(s, md);
  const int flat_a = va <= flat_threshold * md;
  const int flat_b = vb <= flat_threshold * md;
  if (flat_a && flat_b) return 0.0;
  if (flat_a || flat_b) return 2.0 * md;
  const double corr = (s->dot - s->sum_left * s->sum_right / md) / sqrt(va * vb);
  return max0(minab(2.0 * md * (1.0 - corr), 4.0 * md));
}

/* include/mprof/acamp.hpp:86-91 */
double or_f_to_dz(double f, uint64_t m) {
  const double md = (double)m;
  const double signed_root = f < 0.0 ? -sqrt(-f) : sqrt(f);
  const double dz_sq = max0(minab(2.0 * md + 2.0 * signed_root, 4.0 * md));
  return sqrt(dz_sq);
}

/* --- comparison spaces (src/detail/diag_scan.hpp:139-173) ---------------------------------- */

enum { SP_SQ = 0, SP_POW = 1, SP_ZSQ = 2, SP_F = 3 };

static double to_distance(double v, int space, double p, uint64_t m) {
  if (v == INFINITY) return INFINITY; /* diag_scan.hpp:154 */
  switch (space) {
    case SP_SQ:
    case SP_ZSQ: return sqrt(v);
    case SP_POW:
      if (p == 1.0) return v;
      if (p == 2.0) return sqrt(v);
      return pow(v, 1.0 / p);
    default: return or_f_to_dz(v, m);
  }
}

/* --- MinBuffer (src/detail/diag_scan.hpp:31-53) ------------------------------------------- */

typedef struct {
  double* val;
  int64_t* nn;
} minbuf;

static void mb_init(minbuf* b, uint64_t len) {
  b->val = (double*)malloc(sizeof(double) * (len ? len : 1));
  b->nn = (int64_t*)malloc(sizeof(int64_t) * (len ? len : 1));
  for (uint64_t i = 0; i < len; ++i) {
    b->val[i] = INFINITY;
    b->nn[i] = -1;
  }
}
static void mb_free(minbuf* b) {
  free(b->val);
  free(b->nn);
}
static inline void mb_update(minbuf* b, uint64_t at, double v, uint64_t neighbor) {
  const int64_t j = (int64_t)neighbor;
  if (v < b->val[at] || (v == b->val[at] && j < b->nn[at])) {
    b->val[at] = v;
    b->nn[at] = j;
  }
}
static void mb_absorb(minbuf* b, const minbuf* o, uint64_t len) {
  for (uint64_t i = 0; i < len; ++i)
    if (o->val[i] < b->val[i] || (o->val[i] == b->val[i] && o->nn[i] < b->nn[i])) {
      b->val[i] = o->val[i];
      b->nn[i] = o->nn[i];
    }
}

/* --- per-diagonal scans (src/diag_scan.cpp:7-85, advances diag_scan.hpp:93-132) ----------- */

typedef struct {
  const double* t;
  uint64_t n, m, refresh;
  int family, use_f;
  double p, flat;
  uint64_t k_begin, k_end; /* this worker's diagonals */
  minbuf buf;
} scan_job;

static void scan_one(scan_job* J, uint64_t k) {
  const double* t = J->t;
  const uint64_t n = J->n, m = J->m, R = J->refresh;
  const uint64_t last = n - m - k;
  if (J->family == OR_ZNORM) {
    or_stats s = or_direct_stats(t, 0, k, m);
    uint64_t steps = 0;
    double v = J->use_f ? or_f_value(&s, (double)m, J->flat * (double)m)
                        : or_znorm_sq_from_stats(&s, m, J->flat);
    mb_update(&J->buf, 0, v, k);
    mb_update(&J->buf, k, v, 0);
    for (uint64_t i = 1; i <= last; ++i) {
      const uint64_t j = i + k;
      if (R > 0 && steps + 1 >= R) {
        s = or_direct_stats(t, i, j, m);
        steps = 0;
      } else {
        s = or_advance_stats(s, t[i - 1], t[j - 1], t[i + m - 1], t[j + m - 1]);
        steps += 1;
      }
      v = J->use_f ? or_f_value(&s, (double)m, J->flat * (double)m)
                   : or_znorm_sq_from_stats(&s, m, J->flat);
      mb_update(&J->buf, i, v, i + k);
      mb_update(&J->buf, i + k, v, i);
    }
    return;
  }
  const int pn = J->family == OR_PNORM;
  const double p = J->p;
  double acc = pn ? or_direct_pnorm_acc(t, 0, k, m, p) : or_direct_sq_acc(t, 0, k, m);
  uint64_t steps = 0;
  mb_update(&J->buf, 0, acc, k);
  mb_update(&J->buf, k, acc, 0);
  for (uint64_t i = 1; i <= last; ++i) {
    const uint64_t j = i + k;
    if (R > 0 && steps + 1 >= R) {
      acc = pn ? or_direct_pnorm_acc(t, i, j, m, p) : or_direct_sq_acc(t, i, j, m);
      steps = 0;
    } else {
      acc = pn ? or_incremental_pnorm_step(acc, t[i - 1], t[j - 1], t[i + m - 1], t[j + m - 1], p)
               : or_incremental_euclidean_step(acc, t[i - 1], t[j - 1], t[i + m - 1], t[j + m - 1]);
      steps += 1;
    }
    mb_update(&J->buf, i, acc, i + k);
    mb_update(&J->buf, i + k, acc, i);
  }
}

static void* scan_worker(void* arg) {
  scan_job* J = (scan_job*)arg;
  for (uint64_t k = J->k_begin; k < J->k_end; ++k) scan_one(J, k);
  return NULL;
}

/* scan_diagonals + run_engine (src/detail/diag_scan.hpp:193-259, src/diag_scan.cpp:89-140):
 * workers own contiguous diagonal chunks balanced by cell count (diag_scan.hpp:233-242). */
void or_scan(const double* t, uint64_t n, uint64_t m, int family, double p, uint64_t excl,
             uint64_t refresh, double flat_threshold, int use_f, uint64_t k_lo, uint64_t k_hi,
             int threads, double* cmp, double* P, int64_t* I) {
  const uint64_t len = n - m + 1;
  uint64_t lo = excl, hi = n - m + 1; /* diagonals [lo, hi) == [exclusion, n-m] */
  if (!(k_lo == 0 && k_hi == 0)) {
    if (k_lo > lo) lo = k_lo;
    if (k_hi < hi) hi = k_hi;
  }
  const uint64_t count = hi > lo ? hi - lo : 0;
  int workers = threads < 1 ? 1 : threads;
  if ((uint64_t)workers > count) workers = count ? (int)count : 1;
  scan_job* jobs = (scan_job*)calloc((size_t)workers, sizeof(scan_job));
  /* equal-cell cuts */
  uint64_t total = 0;
  for (uint64_t k = lo; k < hi; ++k) total += len - k;
  uint64_t cut = lo, prefix = 0;
  int next = 1;
  for (int w = 0; w < workers; ++w) {
    jobs[w].t = t;
    jobs[w].n = n;
    jobs[w].m = m;
    jobs[w].refresh = refresh;
    jobs[w].family = family;
    jobs[w].use_f = use_f;
    jobs[w].p = p;
    jobs[w].flat = flat_threshold;
    jobs[w].k_begin = cut;
    if (w == workers - 1) {
      cut = hi;
    } else {
      while (cut < hi) {
        prefix += len - cut;
        ++cut;
        if (prefix * (uint64_t)workers >= total * (uint64_t)next) break;
      }
      ++next;
    }
    jobs[w].k_end = cut;
    mb_init(&jobs[w].buf, len);
  }
  if (workers == 1) {
    scan_worker(&jobs[0]);
  } else {
    pthread_t* th = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
    for (int w = 0; w < workers; ++w) pthread_create(&th[w], NULL, scan_worker, &jobs[w]);
    for (int w = 0; w < workers; ++w) pthread_join(th[w], NULL);
    free(th);
    for (int w = 1; w < workers; ++w) mb_absorb(&jobs[0].buf, &jobs[w].buf, len);
  }
  const int space = family == OR_EUCLIDEAN ? SP_SQ
                    : family == OR_PNORM   ? SP_POW
                    : (use_f ? SP_F : SP_ZSQ);
  for (uint64_t i = 0; i < len; ++i) {
    if (cmp) cmp[i] = jobs[0].buf.val[i];
    if (P) P[i] = to_distance(jobs[0].buf.val[i], space, p, m);
    if (I) I[i] = jobs[0].buf.nn[i];
  }
  for (int w = 0; w < workers; ++w) mb_free(&jobs[w].buf);
  free(jobs);
}

/* --- direct distances and brute force (src/oracle.cpp:41-132) ------------------------------ */

/* src/oracle.cpp:35-47 */
static void moments(const double* t, uint64_t start, uint64_t m, double* mean, double* var) {
  double sum = 0.0, sumsq = 0.0;
  for (uint64_t l = 0; l < m; ++l) {
    const double v = t[start + l];
    sum += v;
    sumsq += v * v;
  }
  *mean = sum / (double)m;
  double vv = sumsq / (double)m - (*mean) * (*mean);
  if (vv < 0.0) vv = 0.0;
  *var = vv;
}

/* src/oracle.cpp:51-93 */
double or_dist(const double* t, uint64_t i, uint64_t j, uint64_t m, int family, double p,
               double flat_threshold) {
  if (family == OR_EUCLIDEAN) {
    double sum = 0.0;
    for (uint64_t l = 0; l < m; ++l) {
      const double d = t[i + l] - t[j + l];
      sum += d * d;
    }
    return sqrt(sum);
  }
  if (family == OR_PNORM) {
    double sum = 0.0;
    for (uint64_t l = 0; l < m; ++l) sum += or_abs_pow(t[i + l] - t[j + l], p);
    return pow(sum, 1.0 / p);
  }
  double ma, va, mb, vb;
  moments(t, i, m, &ma, &va);
  moments(t, j, m, &mb, &vb);
  const int fa = va <= flat_threshold, fb = vb <= flat_threshold;
  if (fa && fb) return 0.0;
  if (fa || fb) return sqrt(2.0 * (double)m);
  const double ia = 1.0 / sqrt(va), ib = 1.0 / sqrt(vb);
  double sum = 0.0;
  for (uint64_t l = 0; l < m; ++l) {
    const double d = (t[i + l] - ma) * ia - (t[j + l] - mb) * ib;
    sum += d * d;
  }
  return sqrt(sum);
}

/* src/oracle.cpp:95-132 */
void or_brute_profile(const double* t, uint64_t n, uint64_t m, int family, double p,
                      uint64_t excl, double flat_threshold, double* P, int64_t* I) {
  const uint64_t len = n - m + 1;
  for (uint64_t i = 0; i < len; ++i) {
    double best = INFINITY;
    int64_t bj = -1;
    for (uint64_t j = 0; j < len; ++j) {
      const uint64_t gap = i > j ? i - j : j - i;
      if (gap < excl) continue;
      const double d = or_dist(t, i, j, m, family, p, flat_threshold);
      if (d < best) {
        best = d;
        bj = (int64_t)j;
      }
    }
    P[i] = best;
    I[i] = bj;
  }
}

/* --- well-conditioned exact distance (parity rule 3) -------------------------------------- */

double or_dist_exact(const double* t, uint64_t i, uint64_t j, uint64_t m, int family, double p,
                     double flat_threshold) {
  if (family == OR_EUCLIDEAN) {
    long double s = 0.0L;
    for (uint64_t l = 0; l < m; ++l) {
      const long double d = (long double)t[i + l] - (long double)t[j + l];
      s += d * d;
    }
    return (double)sqrtl(s);
  }
  if (family == OR_PNORM) {
    long double s = 0.0L;
    for (uint64_t l = 0; l < m; ++l) {
      const long double d = fabsl((long double)t[i + l] - (long double)t[j + l]);
      s += (p == 1.0) ? d : (p == 2.0) ? d * d : (p == 3.0) ? d * d * d : powl(d, (long double)p);
    }
    return (double)powl(s, 1.0L / (long double)p);
  }
  long double sa = 0, sb = 0;
  for (uint64_t l = 0; l < m; ++l) {
    sa += t[i + l];
    sb += t[j + l];
  }
  const long double ma = sa / m, mb = sb / m;
  long double qa = 0, qb = 0;
  for (uint64_t l = 0; l < m; ++l) {
    const long double a = t[i + l] - ma, b = t[j + l] - mb;
    qa += a * a;
    qb += b * b;
  }
  const long double va = qa / m, vb = qb / m;
  const int fa = va <= flat_threshold, fb = vb <= flat_threshold;
  if (fa && fb) return 0.0;
  if (fa || fb) return sqrt(2.0 * (double)m);
  const long double ia = 1.0L / sqrtl(va), ib = 1.0L / sqrtl(vb);
  long double s = 0;
  for (uint64_t l = 0; l < m; ++l) {
    const long double d = (t[i + l] - ma) * ia - (t[j + l] - mb) * ib;
    s += d * d;
  }
  return (double)sqrtl(s);
}

void or_dist_exact_many(const double* t, uint64_t m, int family, double p, double flat_threshold,
                        const int64_t* i, const int64_t* j, uint64_t count, double* out) {
  for (uint64_t c = 0; c < count; ++c)
    out[c] = (i[c] < 0 || j[c] < 0) ? INFINITY
                                    : or_dist_exact(t, (uint64_t)i[c], (uint64_t)j[c], m, family, p,
                                                    flat_threshold);
}

typedef struct {
  const double* t;
  uint64_t n, m, excl;
  int family;
  double p, flat;
  const int64_t* rows;
  uint64_t r0, r1;
  double* best;
  int64_t* arg;
} rows_job;

static void* rows_worker(void* a) {
  rows_job* J = (rows_job*)a;
  const uint64_t len = J->n - J->m + 1;
  for (uint64_t r = J->r0; r < J->r1; ++r) {
    const uint64_t i = (uint64_t)J->rows[r];
    double b = INFINITY;
    int64_t bj = -1;
    for (uint64_t j = 0; j < len; ++j) {
      const uint64_t gap = i > j ? i - j : j - i;
      if (gap < J->excl) continue;
      const double d = or_dist_exact(J->t, i, j, J->m, J->family, J->p, J->flat);
      if (d < b) {
        b = d;
        bj = (int64_t)j;
      }
    }
    J->best[r] = b;
    J->arg[r] = bj;
  }
  return NULL;
}

void or_exact_rows(const double* t, uint64_t n, uint64_t m, int family, double p, uint64_t excl,
                   double flat_threshold, const int64_t* rows, uint64_t count, int threads,
                   double* best, int64_t* arg) {
  int w = threads < 1 ? 1 : threads;
  if ((uint64_t)w > count) w = count ? (int)count : 1;
  rows_job* jobs = (rows_job*)calloc((size_t)w, sizeof(rows_job));
  pthread_t* th = (pthread_t*)calloc((size_t)w, sizeof(pthread_t));
  for (int k = 0; k < w; ++k) {
    rows_job J = {t, n, m, excl, family, p, flat_threshold, rows, count * k / w,
                  count * (k + 1) / w, best, arg};
    jobs[k] = J;
    pthread_create(&th[k], NULL, rows_worker, &jobs[k]);
  }
  for (int k = 0; k < w; ++k) pthread_join(th[k], NULL);
  free(th);
  free(jobs);
}
