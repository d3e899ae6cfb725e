// The unmodified reference harness (harness.hpp) and the B200 bridge in one
// translation unit: harness::run_trial (reference, CPU) against the same
// dispatch with its Moshpit case switched to b200_bridge::run_moshpit (the
// one-line change INTEGRATION.md describes), compared bit for bit on
// Table-3-style cells (harness.hpp:145-189).  TEST ONLY: built where the
// reference tree exists (tests/test_cpp_dropin.py), run on a GPU box.
#include <cstdio>
#include <cstring>

#include "moshpit/harness.hpp"
#include "moshpit_b200/harness_bridge.hpp"

using namespace moshpit;

// harness::run_trial (harness.hpp:157-189) with the Moshpit case patched.
static protocols::TrialReport run_trial_patched(const harness::ExperimentConfig& cfg,
                                                std::uint32_t n, double p,
                                                std::uint32_t seed_index) {
  const Rng rng = harness::trial_rng(cfg.seed_base, protocols::ProtocolKind::Moshpit, n, p,
                                     seed_index);
  auto init_stream = rng.stream("init");
  std::vector<ParamVector> initial(n);
  for (auto& theta : initial) {
    if (cfg.init == "normal") {
      theta = init_stream.normals(cfg.dim);
    } else {
      theta.resize(cfg.dim);
      for (auto& x : theta) x = init_stream.uniform();
    }
  }
  const FailureModel failure{p, {}};
  return b200_bridge::run_moshpit(cfg.grid, initial, failure, rng, cfg.round_cap);
}

static bool same(const protocols::TrialReport& a, const protocols::TrialReport& b) {
  auto eqd = [](const std::vector<double>& x, const std::vector<double>& y) {
    return x.size() == y.size() &&
           (x.empty() || std::memcmp(x.data(), y.data(), x.size() * sizeof(double)) == 0);
  };
  return std::memcmp(&a.initial_distortion, &b.initial_distortion, 8) == 0 &&
         eqd(a.distortion, b.distortion) && eqd(a.mean_drift, b.mean_drift) &&
         a.active_counts == b.active_counts && a.cost_units == b.cost_units;
}

// SURVEY 8f rank 4 in C++: the reference's contested matchmaking (skewed
// arrivals + FailStop, matchmaking.hpp:104-294) forms the groups on the CPU;
// the drop-in's butterfly_round averages all of them in one GPU launch; the
// reference's butterfly_allreduce per sealed group is the expected result.
static bool contested_round_case(std::uint64_t seed) {
  using namespace matchmaking;
  auto stream = Rng(seed).stream("trial");
  const std::size_t n = 4 + stream.below(24), dim = 1 + stream.below(40);
  std::vector<MatchPeer> peers;
  for (std::size_t i = 0; i < n; ++i)
    peers.push_back(MatchPeer{static_cast<PeerId>(i),
                              GroupKey{{static_cast<std::uint32_t>(stream.below(3))}},
                              stream() >> 16, stream.below(3)});
  std::vector<FailStop> failures;
  std::vector<bool> dead(n, false);
  for (std::size_t f = stream.below(n / 2 + 1); f > 0; --f) {
    failures.push_back(FailStop{stream.below(8), static_cast<PeerId>(stream.below(n))});
    dead[failures.back().peer] = true;
  }
  Dht dht(1000);
  const auto result = form_groups(0, peers, dht, failures);
  std::vector<ParamVector> x(n);
  for (auto& v : x) v = stream.normals(dim);
  auto want = x;
  std::vector<::moshpit_b200::matchmaking::SealedGroup> groups;
  std::vector<bool> gfail;
  for (const auto& sg : result.groups) {
    std::vector<ParamVector> in;
    std::vector<bool> failed;
    bool any = false;
    for (PeerId m : sg.members) {
      in.push_back(x[m]);
      failed.push_back(dead[m]);
      any = any || dead[m];
    }
    const auto o = allreduce::butterfly_allreduce(
        in, allreduce::PartitionWeights::uniform(in.size()), failed);
    for (std::size_t q = 0; q < sg.members.size(); ++q) want[sg.members[q]] = o.vectors[q];
    groups.push_back({sg.leader, sg.members});
    gfail.push_back(any);
  }
  auto got = x;
  ::moshpit_b200::allreduce::butterfly_round(got, groups, gfail);
  for (std::size_t i = 0; i < n; ++i)
    if (std::memcmp(got[i].data(), want[i].data(), dim * sizeof(double)) != 0) return false;
  return true;
}

int main() {
  int pass = 0, fail = 0;
  for (std::uint64_t s = 0; s < 40; ++s) {
    const bool ok = contested_round_case(900 + s);
    ok ? ++pass : ++fail;
    if (!ok) std::printf("MISMATCH contested round seed=%llu\n", (unsigned long long)(900 + s));
  }
  harness::ExperimentConfig cfg;
  cfg.grid = GridConfig{32, 2, 1};
  cfg.round_cap = 50;
  cfg.seed_base = 0;
  struct Cell {
    std::uint32_t n, dim;
    double p;
    const char* init;
  };
  const Cell cells[] = {{1024, 1, 0.0, "uniform"},  {1024, 1, 0.01, "uniform"},
                        {512, 1, 0.005, "uniform"}, {900, 1, 0.01, "uniform"},
                        {768, 8, 0.0, "normal"},    {1024, 64, 0.01, "normal"}};
  for (const Cell& c : cells) {
    cfg.dim = c.dim;
    cfg.init = c.init;
    for (std::uint32_t s = 0; s < 3; ++s) {
      const auto want = harness::run_trial(cfg, protocols::ProtocolKind::Moshpit, c.n, c.p, s);
      const auto got = run_trial_patched(cfg, c.n, c.p, s);
      const bool ok = same(want, got);
      ok ? ++pass : ++fail;
      if (!ok)
        std::printf("MISMATCH n=%u dim=%u p=%g seed=%u rounds_to(1e-9): ref %u b200 %u\n", c.n,
                    c.dim, c.p, s, want.rounds_to(1e-9, 50), got.rounds_to(1e-9, 50));
    }
  }
  std::printf("PASS=%d FAIL=%d\n", pass, fail);
  return fail ? 1 : 0;
}
