// mprof_shim.cpp — the C++ drop-in API (include/mprof/*.hpp) over the C ABI.
// Replaces the reference's src/aamp.cpp, src/acamp.cpp, src/core.cpp, src/oracle.cpp
// (brute_profile) and src/engine_state.cpp for a GPU build: same validation order and error
// codes, MatrixProfile returned by value.
#include <algorithm>
#include <cmath>
#include <string>

#include "mprof/aamp.hpp"
#include "mprof/acamp.hpp"
#include "mprof/core.hpp"
#include "mprof/engine_state.hpp"
#include "mprof/multi_gpu.hpp"
#include "mprof/oracle.hpp"
#include "mprof_gpu.h"

namespace mprof {

namespace {

// C ABI status = ErrorCode value + 1 (device codes: Cuda = 99 <-> 100, ...)
[[noreturn]] void rethrow(int32_t status) {
  throw Error(static_cast<ErrorCode>(status - 1), mprof_last_error());
}

mprof_config to_c(const ProfileConfig& cfg) {
  mprof_config c;
  mprof_config_init(&c, cfg.m, static_cast<int32_t>(cfg.kind.family), cfg.kind.p);
  c.p = cfg.kind.p;
  c.exclusion = cfg.exclusion;
  c.order = static_cast<int32_t>(cfg.order);
  c.order_seed = cfg.order_seed;
  c.refresh_interval = cfg.refresh_interval;
  c.flat_threshold = cfg.flat_threshold;
  c.precision = cfg.precision == Precision::FP32 ? MPROF_FP32 : MPROF_FP64;
  c.exact = cfg.exact ? 1 : 0;
  return c;
}

// The observer runs on the calling thread between band launches; false cancels.
int32_t progress_trampoline(uint64_t done, uint64_t total, void* user) {
  const ProgressFn& fn = *static_cast<const ProgressFn*>(user);
  return fn(static_cast<std::size_t>(done), static_cast<std::size_t>(total)) ? 1 : 0;
}

struct ProgressScope {
  explicit ProgressScope(const ProgressFn& fn) : active(static_cast<bool>(fn)) {
    if (active) mprof_ctx_set_progress(nullptr, progress_trampoline, const_cast<ProgressFn*>(&fn));
  }
  ~ProgressScope() {
    if (active) mprof_ctx_set_progress(nullptr, nullptr, nullptr);
  }
  bool active;
};

template <class Call>
MatrixProfile run(const TimeSeries& ts, const ProfileConfig& cfg, const ProgressFn& progress,
                  Call&& call) {
  const mprof_config c = to_c(cfg);
  MatrixProfile out;
  out.m = cfg.m;
  out.kind = cfg.kind;
  const std::size_t n = ts.size();
  const std::size_t len = (cfg.m >= 1 && cfg.m <= n) ? n - cfg.m + 1 : 1;
  out.distances.resize(len);
  out.nn_index.resize(len);
  mprof_run_info info{};
  int32_t st;
  {
    ProgressScope scope(progress);
    st = call(&c, out.distances.data(), out.nn_index.data(), &info);
  }
  if (st != MPROF_OK) rethrow(st);
  return out;
}

}  // namespace

TimeSeries make_time_series(std::vector<double> samples) {
  for (std::size_t i = 0; i < samples.size(); ++i)
    if (!std::isfinite(samples[i]))
      throw Error(ErrorCode::NonFinite, "sample " + std::to_string(i) + " is not finite");
  if (samples.size() < 2)
    throw Error(ErrorCode::TooShort,
                "time series needs at least 2 samples, got " + std::to_string(samples.size()));
  return TimeSeries(std::move(samples));
}

ProfileConfig validate_config(const TimeSeries& ts, const ProfileConfig& cfg) {
  const mprof_config c = to_c(cfg);
  const int32_t st = mprof_validate(ts.data(), ts.size(), &c);
  if (st != MPROF_OK) rethrow(st);
  return cfg;
}

MatrixProfile aamp(const TimeSeries& ts, const ProfileConfig& cfg, ProgressFn progress, unsigned) {
  return run(ts, cfg, progress, [&](const mprof_config* c, double* P, int64_t* I, mprof_run_info* info) {
    return mprof_aamp(nullptr, ts.data(), ts.size(), c, P, I, info);
  });
}

MatrixProfile aamp_pnorm(const TimeSeries& ts, const ProfileConfig& cfg, ProgressFn progress,
                         unsigned) {
  return run(ts, cfg, progress, [&](const mprof_config* c, double* P, int64_t* I, mprof_run_info* info) {
    return mprof_aamp_pnorm(nullptr, ts.data(), ts.size(), c, P, I, info);
  });
}

MatrixProfile acamp(const TimeSeries& ts, const ProfileConfig& cfg, AcampVariant variant,
                    ProgressFn progress, unsigned) {
  const int32_t v = variant == AcampVariant::FScore ? MPROF_ACAMP_FSCORE : MPROF_ACAMP_SQUARED_DISTANCE;
  return run(ts, cfg, progress, [&](const mprof_config* c, double* P, int64_t* I, mprof_run_info* info) {
    return mprof_acamp(nullptr, ts.data(), ts.size(), c, v, P, I, info);
  });
}

// ---- host-side primitives of the public API ---------------------------------------------------
// The reference's direct (non-incremental) evaluations and the throwing five-sum helpers
// (/root/reference/proj/src/oracle.cpp:51-93, src/acamp.cpp:9-27). They are O(m) per call, exist
// for callers that cross-check engines, and are not on the sweep path; the summation order is the
// reference's (l = 0..m-1, no contraction), so their results match it bit for bit.

namespace {

void require_window(const TimeSeries& ts, std::size_t at, std::size_t m, const char* which) {
  if (m == 0 || at + m > ts.size())
    throw Error(ErrorCode::OutOfRange, std::string(which) + " window of length " + std::to_string(m) +
                                           " at " + std::to_string(at) + " does not fit " +
                                           std::to_string(ts.size()) + " samples");
}

// Population mean and variance from plain sums (oracle.cpp:35-47), variance floored at 0.
void window_moments(const TimeSeries& ts, std::size_t at, std::size_t m, double* mean, double* var) {
  double s = 0.0, s2 = 0.0;
  for (std::size_t l = 0; l < m; ++l) {
    const double x = ts[at + l];
    s += x;
    s2 += x * x;
  }
  const double md = static_cast<double>(m);
  *mean = s / md;
  double v = s2 / md - *mean * *mean;
  if (v < 0.0) v = 0.0;
  *var = v;
}

}  // namespace

DiagStats init_diag_stats(const TimeSeries& ts, std::size_t k, std::size_t m) {
  if (m == 0 || k + m > ts.size())
    throw Error(ErrorCode::OutOfRange, "window pair (0, " + std::to_string(k) + ") of length " +
                                           std::to_string(m) + " does not fit " +
                                           std::to_string(ts.size()) + " samples");
  DiagStats s;
  s.offset = k;
  s.pos = 0;
  for (std::size_t l = 0; l < m; ++l) {
    const double a = ts[l], b = ts[k + l];
    s.sum_left += a;
    s.sum_right += b;
    s.sumsq_left += a * a;
    s.sumsq_right += b * b;
    s.dot += a * b;
  }
  return s;
}

double f_score(const DiagStats& s, std::size_t m, double flat_threshold) {
  const double md = static_cast<double>(m);
  const double scaled_flat = flat_threshold * md;
  if (detail::scaled_var_left(s, md) <= scaled_flat || detail::scaled_var_right(s, md) <= scaled_flat)
    throw Error(ErrorCode::Degenerate, "f_score is undefined for a flat window (flat-window convention applies)");
  return detail::f_value(s, md, scaled_flat);
}

double dist_euclidean(const TimeSeries& ts, std::size_t i, std::size_t j, std::size_t m) {
  require_window(ts, i, m, "left");
  require_window(ts, j, m, "right");
  double acc = 0.0;
  for (std::size_t l = 0; l < m; ++l) {
    const double d = ts[i + l] - ts[j + l];
    acc += d * d;
  }
  return std::sqrt(acc);
}

double dist_pnorm(const TimeSeries& ts, std::size_t i, std::size_t j, std::size_t m, double p) {
  require_window(ts, i, m, "left");
  require_window(ts, j, m, "right");
  if (!(p >= 1.0)) throw Error(ErrorCode::BadP, "p-norm exponent must be >= 1, got " + std::to_string(p));
  double acc = 0.0;
  for (std::size_t l = 0; l < m; ++l) acc += detail::abs_pow(ts[i + l] - ts[j + l], p);
  return std::pow(acc, 1.0 / p);
}

double dist_znorm(const TimeSeries& ts, std::size_t i, std::size_t j, std::size_t m,
                  double flat_threshold) {
  require_window(ts, i, m, "left");
  require_window(ts, j, m, "right");
  double mi, vi, mj, vj;
  window_moments(ts, i, m, &mi, &vi);
  window_moments(ts, j, m, &mj, &vj);
  const bool fi = vi <= flat_threshold, fj = vj <= flat_threshold;
  if (fi || fj) return (fi && fj) ? 0.0 : std::sqrt(2.0 * static_cast<double>(m));
  const double si = 1.0 / std::sqrt(vi), sj = 1.0 / std::sqrt(vj);
  double acc = 0.0;
  for (std::size_t l = 0; l < m; ++l) {
    const double d = (ts[i + l] - mi) * si - (ts[j + l] - mj) * sj;
    acc += d * d;
  }
  return std::sqrt(acc);
}

MatrixProfile brute_profile(const TimeSeries& ts, const ProfileConfig& cfg) {
  return run(ts, cfg, {}, [&](const mprof_config* c, double* P, int64_t* I, mprof_run_info*) {
    return mprof_brute_profile(nullptr, ts.data(), ts.size(), c, P, I);
  });
}

MatrixProfile profile_on_devices(const TimeSeries& ts, const ProfileConfig& cfg,
                                 std::span<const int> devices, Engine engine) {
  std::vector<int32_t> dev(devices.begin(), devices.end());
  return run(ts, cfg, {}, [&](const mprof_config* c, double* P, int64_t* I, mprof_run_info* info) {
    return mprof_profile_multi(dev.data(), static_cast<uint32_t>(dev.size()),
                               static_cast<int32_t>(engine), ts.data(), ts.size(), c, P, I, info);
  });
}

// ---- EngineState -----------------------------------------------------------------------------

namespace {

EngineState snapshot(std::shared_ptr<mprof_state> dev, const ProfileConfig& cfg) {
  const uint64_t n = mprof_state_series_length(dev.get());
  const uint64_t L = n - cfg.m + 1;
  std::vector<double> t(n), P(L), cmp(L);
  std::vector<Index> I(L);
  int32_t st = mprof_state_series(dev.get(), t.data());
  if (st == MPROF_OK) st = mprof_state_profile(dev.get(), P.data(), I.data(), cmp.data());
  if (st != MPROF_OK) rethrow(st);
  MatrixProfile mp;
  mp.distances = std::move(P);
  mp.nn_index = std::move(I);
  mp.m = cfg.m;
  mp.kind = cfg.kind;
  // completed diagonals (ascending from the exclusion) and their tail cursors
  const uint64_t done = mprof_state_completed_diagonals(dev.get());
  const bool zn = cfg.kind.family == DistanceFamily::ZNormalized;
  std::vector<double> tail(done * (zn ? 5 : 1));
  if (done) {
    st = mprof_state_tail(dev.get(), tail.data());
    if (st != MPROF_OK) rethrow(st);
  }
  std::vector<std::size_t> diags(done);
  std::vector<DiagonalCursor> pc;
  std::vector<ZnormCursor> zc;
  (zn ? zc.reserve(done) : pc.reserve(done));
  for (uint64_t r = 0; r < done; ++r) {
    const std::size_t k = cfg.exclusion + r;
    diags[r] = k;
    const std::size_t pos = n - cfg.m - k;  // the diagonal's last cell
    if (zn) {
      ZnormCursor z;
      z.stats = DiagStats{tail[5 * r], tail[5 * r + 1], tail[5 * r + 2], tail[5 * r + 3],
                          tail[5 * r + 4], k, pos};
      zc.push_back(z);
    } else {
      pc.push_back(DiagonalCursor{k, pos, tail[r], 0});
    }
  }
  return EngineState{make_time_series(std::move(t)), cfg,        std::move(mp), std::move(cmp),
                     std::move(diags),                std::move(pc), std::move(zc), std::move(dev)};
}

}  // namespace

EngineState build_engine_state(const TimeSeries& ts, const ProfileConfig& cfg, ProgressFn progress,
                               unsigned) {
  const mprof_config c = to_c(cfg);
  mprof_state* raw = nullptr;
  int32_t st;
  {
    ProgressScope scope(progress);  // the observer may cancel: the state is then incomplete
    st = mprof_state_build(nullptr, ts.data(), ts.size(), &c, &raw, nullptr);
  }
  if (st != MPROF_OK) rethrow(st);
  return snapshot(std::shared_ptr<mprof_state>(raw, mprof_state_destroy), cfg);
}

EngineState extend_profile(const EngineState& state, std::span<const double> new_samples) {
  // engine_state.cpp:56-66 order: IncompleteState, then the empty span, then NonFinite
  if (!state.complete())
    throw Error(ErrorCode::IncompleteState,
                "cannot extend a partially computed profile (" +
                    std::to_string(state.completed_diagonals.size()) + " diagonals done)");
  if (new_samples.empty()) return state;
  for (std::size_t i = 0; i < new_samples.size(); ++i)
    if (!std::isfinite(new_samples[i]))
      throw Error(ErrorCode::NonFinite, "appended sample " + std::to_string(i) + " is not finite");
  mprof_state* raw = nullptr;
  int32_t st = mprof_state_clone(state.device.get(), &raw);
  if (st != MPROF_OK) rethrow(st);
  std::shared_ptr<mprof_state> dev(raw, mprof_state_destroy);
  st = mprof_state_extend(dev.get(), new_samples.data(), new_samples.size(), nullptr);
  if (st != MPROF_OK) rethrow(st);
  return snapshot(std::move(dev), state.cfg);
}

}  // namespace mprof
