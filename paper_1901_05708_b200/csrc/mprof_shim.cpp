// mprof_shim.cpp — the C++ drop-in API (include/mprof/*.hpp) over the C ABI.
// Replaces the reference's src/aamp.cpp, src/acamp.cpp and src/core.cpp for a GPU build:
// same validation order and error codes, MatrixProfile returned by value.
#include <cmath>
#include <string>

#include "mprof/aamp.hpp"
#include "mprof/acamp.hpp"
#include "mprof/core.hpp"
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
  const int32_t st = call(&c, out.distances.data(), out.nn_index.data(), &info);
  if (st != MPROF_OK) rethrow(st);
  if (progress) progress(info.diagonals, info.diagonals);
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

}  // namespace mprof
