// moshpit_b200/harness_bridge.hpp -- run the reference harness's Moshpit
// trials on the B200 engine while every other protocol stays on the
// reference's CPU code.
//
// The reference harness (proj/include/moshpit/harness.hpp:20-23) includes
// protocols.hpp / theory.hpp itself and dispatches on ProtocolKind
// (harness.hpp:175-188), so it cannot be compiled against the drop-in header
// alone (the drop-in covers the Moshpit hot path, not run_gossip & co.).
// This header puts the drop-in in its own namespace (MOSHPIT_B200_NS =
// moshpit_b200) next to the reference's `moshpit`, and offers
// moshpit::b200_bridge::run_moshpit with the reference's exact signature
// (protocols.hpp:108-111) and return type.  The maintainer's change is one
// line in harness::run_trial's Moshpit case:
//     return protocols::run_moshpit(cfg.grid, initial, failure, rng, cfg.round_cap);
//  -> return b200_bridge::run_moshpit(cfg.grid, initial, failure, rng, cfg.round_cap);
// The report is bit-identical (fp64, reference summation order):
// tests/cpp/test_harness_bridge.cpp checks it against the unmodified
// harness::run_trial on Table-3 cells.
//
// Include order: the reference headers first, then this header; do not also
// include moshpit_b200/moshpit.hpp under its default namespace in the same TU.
#pragma once

#include "moshpit/protocols.hpp"

#ifndef MOSHPIT_B200_NS
#define MOSHPIT_B200_NS moshpit_b200
#endif
#include "moshpit_b200/moshpit.hpp"

namespace moshpit::b200_bridge {

inline protocols::TrialReport run_moshpit(const GridConfig& grid,
                                          const std::vector<ParamVector>& initial,
                                          const FailureModel& failure, const Rng& rng,
                                          std::uint32_t rounds) {
  namespace nb = ::MOSHPIT_B200_NS;
  const auto r = nb::protocols::run_moshpit(
      nb::GridConfig{grid.peers_per_axis, grid.dims, grid.rounds}, initial,
      nb::FailureModel{failure.p_round, failure.churn}, nb::Rng(rng.seed()), rounds);
  protocols::TrialReport out;
  out.initial_distortion = r.initial_distortion;
  out.distortion = r.distortion;
  out.mean_drift = r.mean_drift;
  out.active_counts = r.active_counts;
  out.cost_units = r.cost_units;
  return out;
}

}  // namespace moshpit::b200_bridge
