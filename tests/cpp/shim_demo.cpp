// Drop-in check: code written against the reference's C++ API (mprof::aamp / aamp_pnorm / acamp,
// ProfileConfig, MatrixProfile, Error) compiled against include/mprof/*.hpp + libmprof_gpu.so.
// Exit codes: 0 = all known answers reproduced, 1 = mismatch, 3 = no CUDA device (Error::Cuda).
#include <cmath>
#include <cstdio>

#include "mprof/aamp.hpp"
#include "mprof/acamp.hpp"

using namespace mprof;

static bool near(double a, double b) { return std::fabs(a - b) <= 1e-12 * std::fmax(1.0, std::fabs(b)); }

int main() {
  try {
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
    bool bad_kind = false;
    try {
      aamp(zig, ProfileConfig(3, DistanceKind::pnorm(3.0)));
    } catch (const Error& err) {
      bad_kind = err.code() == ErrorCode::BadKind;
    }
    std::printf("aamp %s, BadKind %s\n", ok ? "ok" : "MISMATCH", bad_kind ? "ok" : "MISSING");
    return ok && bad_kind ? 0 : 1;
  } catch (const Error& err) {
    if (err.code() == ErrorCode::Cuda) {
      std::printf("no CUDA device: %s\n", err.what());
      return 3;
    }
    std::printf("error %d: %s\n", static_cast<int>(err.code()), err.what());
    return 1;
  }
}
