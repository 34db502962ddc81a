// mprof/engine_state.hpp — incremental profiles (drop-in for build_engine_state /
// extend_profile, /root/reference/proj/include/mprof/engine_state.hpp:13-52).
//
// The GPU state keeps the series and the comparison-space profile on the device; an extension
// sweeps only the cells that involve an appended window (the reflected sweep). The
// reference's fields are all present: `completed_diagonals` records which diagonals the build
// finished (a progress observer may cancel it), and the tail cursors hold each completed
// diagonal's state at its last cell, evaluated directly on the GPU (the extension itself does not
// need them: it re-derives new cells from the series).
#pragma once

#include <memory>
#include <span>
#include <vector>

#include "mprof/aamp.hpp"
#include "mprof/acamp.hpp"
#include "mprof/core.hpp"

extern "C" {
struct mprof_state;
}

namespace mprof {

// Tail of one z-normalized diagonal (engine_state.hpp:13-16).
struct ZnormCursor {
  DiagStats stats;
  std::size_t steps_since_refresh = 0;
};

struct EngineState {
  TimeSeries ts;
  ProfileConfig cfg;
  MatrixProfile profile;
  std::vector<double> comparison;                // profile in the engine's comparison space
  std::vector<std::size_t> completed_diagonals;  // ascending offsets k
  std::vector<DiagonalCursor> tail_cursors;      // Euclidean / PNorm, parallel to completed_diagonals
  std::vector<ZnormCursor> znorm_cursors;        // ZNormalized, parallel to completed_diagonals
  std::shared_ptr<mprof_state> device;           // GPU-resident series + profile

  // True when every diagonal of the configured scan completed (engine_state.hpp:37-39).
  bool complete() const noexcept {
    return completed_diagonals.size() == ts.size() - cfg.m - cfg.exclusion + 1;
  }
};

// Runs the engine of cfg.kind and keeps the state; a build cancelled by `progress` is an
// incomplete state (a valid upper-bound profile) that extend_profile refuses.
EngineState build_engine_state(const TimeSeries& ts, const ProfileConfig& cfg,
                               ProgressFn progress = {}, unsigned threads = 0);

// A new state for the extended series. Throws IncompleteState unless state.complete(), then
// NonFinite for a bad sample; an empty span returns an equal state.
EngineState extend_profile(const EngineState& state, std::span<const double> new_samples);

}  // namespace mprof
