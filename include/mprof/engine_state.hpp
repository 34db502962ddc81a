// mprof/engine_state.hpp — incremental profiles (drop-in for build_engine_state /
// extend_profile, /root/reference/proj/include/mprof/engine_state.hpp:26-52). The GPU state keeps
// the series and the comparison-space profile on the device; an extension sweeps only the cells
// that involve an appended window.
#pragma once

#include <memory>
#include <span>

#include "mprof/core.hpp"

extern "C" {
struct mprof_state;
}

namespace mprof {

struct EngineState {
  TimeSeries ts;
  ProfileConfig cfg;
  MatrixProfile profile;
  std::vector<double> comparison;  // profile in the engine's comparison space
  std::shared_ptr<mprof_state> device;

  bool complete() const noexcept { return true; }  // a GPU sweep is never partial
};

EngineState build_engine_state(const TimeSeries& ts, const ProfileConfig& cfg,
                               ProgressFn progress = {}, unsigned threads = 0);

// A new state for the extended series; throws NonFinite for a bad sample.
EngineState extend_profile(const EngineState& state, std::span<const double> new_samples);

}  // namespace mprof
