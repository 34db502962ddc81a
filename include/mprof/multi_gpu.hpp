// mprof/multi_gpu.hpp — one process, several GPUs (mprof_profile_multi in mprof_gpu.h).
// The reference splits the diagonals across CPU worker threads (`threads`,
// /root/reference/proj/src/detail/diag_scan.hpp:228-256); this splits them across devices into
// equal-area bands and merges the partial profiles exactly (MinBuffer::absorb semantics).
#pragma once

#include <span>

#include "mprof/core.hpp"

namespace mprof {

enum class Engine { Aamp = 0, AampPnorm = 1, Acamp = 2 };

// Same validation, error codes and result as aamp / aamp_pnorm / acamp on one device; a device
// may be listed more than once. Progress observers are not supported on this path.
MatrixProfile profile_on_devices(const TimeSeries& ts, const ProfileConfig& cfg,
                                 std::span<const int> devices, Engine engine);

}  // namespace mprof
