// Drop-in check: code written against the reference's C++ API (mprof::aamp / aamp_pnorm / acamp,
// ProfileConfig, MatrixProfile, Error, ProgressFn, build_engine_state / extend_profile,
// brute_profile) compiled against include/mprof/*.hpp + libmprof_gpu.so, plus the multi-device
// entry point. Exit codes: 0 = every check passed, 1 = mismatch, 3 = no CUDA device (Error::Cuda).
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "mprof/aamp.hpp"
#include "mprof/acamp.hpp"
#include "mprof/engine_state.hpp"
#include "mprof/multi_gpu.hpp"
#include "mprof/oracle.hpp"

using namespace mprof;

static bool near(double a, double b, double tol = 1e-12) {
  return std::fabs(a - b) <= tol * std::fmax(1.0, std::fabs(b));
}

static bool same(const MatrixProfile& a, const MatrixProfile& b, double tol) {
  if (a.size() != b.size()) return false;
  for (std::size_t i = 0; i < a.size(); ++i)
    if (!near(a.distances[i], b.distances[i], tol)) return false;
  return true;
}

static int check(const char* what, bool ok) {
  std::printf("%-40s %s\n", what, ok ? "ok" : "MISMATCH");
  return ok ? 0 : 1;
}

int main() {
  try {
    int fails = 0;
    // known answers (tests/test_aamp.cpp:63-72, tests/test_acamp.cpp:181-191, acceptance.cpp:193-201)
    const TimeSeries zig = make_time_series({0, 1, 2, 1, 0, 1, 2});
    const MatrixProfile e = aamp(zig, ProfileConfig(3, DistanceKind::euclidean()));
    const MatrixProfile z = acamp(zig, ProfileConfig(3, DistanceKind::znormalized()));
    const MatrixProfile p = aamp_pnorm(zig, ProfileConfig(3, DistanceKind::pnorm(3.0)));
    const double r3 = std::sqrt(3.0), r6 = std::sqrt(6.0), c3 = std::cbrt(3.0);
    const double we[] = {0, r3, r3, r3, 0}, wz[] = {0, r6, r6, r6, 0}, wp[] = {0, c3, c3, c3, 0};
    const Index ie[] = {4, 0, 1, 0, 0};
    bool ok = e.size() == 5 && z.size() == 5 && p.size() == 5;
    for (int i = 0; ok && i < 5; ++i)
      ok = near(e.distances[i], we[i]) && e.nn_index[i] == ie[i] && near(z.distances[i], wz[i]) &&
           std::fabs(p.distances[i] - wp[i]) <= 1e-9;
    fails += check("zigzag known answers", ok);
    bool bad_kind = false;
    try {
      aamp(zig, ProfileConfig(3, DistanceKind::pnorm(3.0)));
    } catch (const Error& err) {
      bad_kind = err.code() == ErrorCode::BadKind;
    }
    fails += check("BadKind from the entry point", bad_kind);

    // a random walk for the remaining checks
    std::mt19937_64 rng(7);
    std::normal_distribution<double> step(0.0, 1.0);
    std::vector<double> walk(6000);
    double x = 0.0;
    for (auto& v : walk) v = (x += step(rng));
    const TimeSeries ts = make_time_series(walk);
    const ProfileConfig cfg(64, DistanceKind::euclidean());
    const MatrixProfile full = aamp(ts, cfg);

    // ProgressFn: band-granular ticks ending at total; returning false cancels
    std::size_t ticks = 0, last_done = 0, last_total = 0;
    const MatrixProfile observed = aamp(ts, cfg, [&](std::size_t done, std::size_t total) {
      ++ticks;
      last_done = done;
      last_total = total;
      return true;
    });
    fails += check("progress ticks reach total", ticks > 1 && last_done == last_total &&
                                                     same(observed, full, 1e-12));
    std::size_t calls = 0;
    const MatrixProfile cancelled = aamp(ts, cfg, [&](std::size_t, std::size_t) { return ++calls < 3; });
    bool partial_ok = calls == 3 && cancelled.size() == full.size();
    for (std::size_t i = 0; partial_ok && i < full.size(); ++i)  // a minimum over fewer diagonals
      partial_ok = cancelled.distances[i] >= full.distances[i] * (1 - 1e-12);
    fails += check("progress cancellation", partial_ok);

    // EngineState: build on a prefix, extend twice, equals the full profile
    const std::vector<double> head(walk.begin(), walk.begin() + 4000);
    EngineState st = build_engine_state(make_time_series(head), cfg);
    st = extend_profile(st, std::span<const double>(walk.data() + 4000, 1500));
    st = extend_profile(st, std::span<const double>(walk.data() + 5500, 500));
    fails += check("build_engine_state + extend_profile", same(st.profile, full, 1e-9) &&
                                                              st.ts.size() == walk.size());

    // brute_profile (GPU) agrees with the sweep
    const TimeSeries small = make_time_series(std::vector<double>(walk.begin(), walk.begin() + 900));
    fails += check("brute_profile vs aamp", same(brute_profile(small, cfg), aamp(small, cfg), 1e-9));

    // diagonals split across two contexts of device 0
    const int devices[] = {0, 0};
    fails += check("profile_on_devices", same(profile_on_devices(ts, cfg, devices, Engine::Aamp), full, 1e-9));
    return fails ? 1 : 0;
  } catch (const Error& err) {
    if (err.code() == ErrorCode::Cuda) {
      std::printf("no CUDA device: %s\n", err.what());
      return 3;
    }
    std::printf("error %d: %s\n", static_cast<int>(err.code()), err.what());
    return 1;
  }
}
