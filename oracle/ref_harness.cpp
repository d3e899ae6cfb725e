// ref_harness.cpp -- extern "C" hooks over the UNMODIFIED reference harness
// (harness.hpp: trial_rng, run_trial).  TEST INFRASTRUCTURE ONLY; compiled
// into oracle/_ref/libmoshpit_ref_harness.so when the nlohmann json header the
// harness includes is available (oracle/Makefile).
#include <cstring>

#include "moshpit/harness.hpp"

using namespace moshpit;

extern "C" {

std::uint64_t refh_trial_seed(std::uint64_t seed_base, std::uint32_t n, double p,
                              std::uint32_t seed_index) {
  return harness::trial_rng(seed_base, protocols::ProtocolKind::Moshpit, n, p, seed_index).seed();
}

// harness::run_trial for the Moshpit protocol (harness.hpp:157-189).
int refh_run_trial(std::uint64_t seed_base, std::uint32_t n, double p, std::uint32_t seed_index,
                   std::uint32_t M, std::uint32_t d, std::uint32_t dim, int init_normal,
                   std::uint32_t round_cap, double* init_d, double* dist, double* drift,
                   std::uint32_t* active) {
  try {
    harness::ExperimentConfig cfg;
    cfg.grid = GridConfig{M, d, 1};
    cfg.dim = dim;
    cfg.init = init_normal ? "normal" : "uniform";
    cfg.seed_base = seed_base;
    cfg.round_cap = round_cap;
    const auto r = harness::run_trial(cfg, protocols::ProtocolKind::Moshpit, n, p, seed_index);
    *init_d = r.initial_distortion;
    for (std::size_t t = 0; t < r.distortion.size(); ++t) {
      dist[t] = r.distortion[t];
      drift[t] = r.mean_drift[t];
      active[t] = r.active_counts[t];
    }
    return 0;
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
