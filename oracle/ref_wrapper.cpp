// ref_wrapper.cpp — TEST INFRASTRUCTURE ONLY. Compiled together with the reference library's
// own sources (/root/reference/proj/src/*.cpp, never copied) into oracle/_ref/libmprof_ref.so,
// with -Dmprof=mprof_ref so it can never collide with the drop-in's mprof:: symbols.
// Exposes the reference's public entry points (aamp / aamp_pnorm / acamp / brute_profile and
// run_engine's comparison values) behind plain C functions for ctypes.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "detail/diag_scan.hpp"
#include "mprof/aamp.hpp"
#include "mprof/acamp.hpp"
#include "mprof/oracle.hpp"

using namespace mprof;

namespace {
// sentinel for "keep ProfileConfig's default flat_threshold" (any other value is passed through,
// including invalid ones, so validation parity can be tested)
constexpr double kDefaultFlat = -7.0e300;
int code_of(const Error& e) { return static_cast<int>(e.code()) + 1; }

ProfileConfig make_cfg(uint64_t m, int family, double p, uint64_t excl, uint64_t refresh, double flat) {
  DistanceKind kind = family == 0 ? DistanceKind::euclidean()
                      : family == 1 ? DistanceKind::pnorm(p)
                                    : DistanceKind::znormalized();
  ProfileConfig cfg(m, kind);
  cfg.exclusion = excl;
  cfg.refresh_interval = refresh;
  if (flat != kDefaultFlat) cfg.flat_threshold = flat;
  return cfg;
}

void copy_out(const MatrixProfile& mp, double* P, int64_t* I) {
  std::memcpy(P, mp.distances.data(), sizeof(double) * mp.distances.size());
  std::memcpy(I, mp.nn_index.data(), sizeof(int64_t) * mp.nn_index.size());
}
}  // namespace

extern "C" {

// family 0 aamp, 1 aamp_pnorm, 2 acamp(variant: 1 FScore, 0 SquaredDistance).
// flat == -7e300: ProfileConfig's default.
// Returns 0 or ErrorCode+1; -1 for any other exception.
int ref_profile(const double* t, uint64_t n, uint64_t m, int family, double p, uint64_t excl,
                uint64_t refresh, double flat, int variant, unsigned threads, double* P, int64_t* I) {
  try {
    const TimeSeries ts = make_time_series(std::vector<double>(t, t + n));
    const ProfileConfig cfg = make_cfg(m, family, p, excl, refresh, flat);
    MatrixProfile mp;
    if (family == 0) mp = aamp(ts, cfg, {}, threads);
    else if (family == 1) mp = aamp_pnorm(ts, cfg, {}, threads);
    else mp = acamp(ts, cfg, variant ? AcampVariant::FScore : AcampVariant::SquaredDistance, {}, threads);
    copy_out(mp, P, I);
    return 0;
  } catch (const Error& e) {
    return code_of(e);
  } catch (...) {
    return -1;
  }
}

// Like ref_profile for an explicit (validated) family, also returning the comparison values.
int ref_engine(const double* t, uint64_t n, uint64_t m, int family, double p, uint64_t excl,
               uint64_t refresh, double flat, int variant, unsigned threads, double* cmp, double* P,
               int64_t* I) {
  try {
    const TimeSeries ts = make_time_series(std::vector<double>(t, t + n));
    const ProfileConfig cfg = validate_config(ts, make_cfg(m, family, p, excl, refresh, flat));
    const detail::EngineRun run = detail::run_engine(
        ts, cfg, variant ? AcampVariant::FScore : AcampVariant::SquaredDistance, {}, threads,
        nullptr, nullptr);
    std::memcpy(cmp, run.comparison.data(), sizeof(double) * run.comparison.size());
    copy_out(run.profile, P, I);
    return 0;
  } catch (const Error& e) {
    return code_of(e);
  } catch (...) {
    return -1;
  }
}

int ref_brute(const double* t, uint64_t n, uint64_t m, int family, double p, uint64_t excl,
              double flat, double* P, int64_t* I) {
  try {
    const TimeSeries ts = make_time_series(std::vector<double>(t, t + n));
    copy_out(brute_profile(ts, make_cfg(m, family, p, excl, 0, flat)), P, I);
    return 0;
  } catch (const Error& e) {
    return code_of(e);
  } catch (...) {
    return -1;
  }
}

// Full validation path of the entry points (make_time_series + validate_config + family check),
// for error-code parity tests. Calls the engine only on a valid tiny config.
int ref_validate(const double* t, uint64_t n, uint64_t m, int family, double p, uint64_t excl,
                 double flat, int entry) {
  try {
    const TimeSeries ts = make_time_series(std::vector<double>(t, t + n));
    const ProfileConfig cfg = make_cfg(m, family, p, excl, 0, flat);
    if (entry == 0) aamp(ts, cfg, {}, 1);
    else if (entry == 1) aamp_pnorm(ts, cfg, {}, 1);
    else acamp(ts, cfg, AcampVariant::FScore, {}, 1);
    return 0;
  } catch (const Error& e) {
    return code_of(e);
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
