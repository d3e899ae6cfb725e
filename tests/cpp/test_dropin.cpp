// test_dropin.cpp -- the reference's own hot-path test cases, compiled
// against the DROP-IN header (include/moshpit_b200/moshpit.hpp) instead of
// the reference headers, so they exercise the GPU path through the C ABI.
// Cases follow proj/tests/test_core.cpp, test_allreduce.cpp,
// test_matchmaking.cpp and test_protocols.cpp (cited per case).  Catch2 is
// absent in this image, so a minimal CHECK macro stands in.
// Final line: a TrialReport for the golden C2-shaped case, as hex, which
// tests/test_cpp_dropin.py compares bit-for-bit with tests/golden/golden.json.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <set>

#include "moshpit_b200/moshpit.hpp"

using namespace moshpit;

static int g_fail = 0, g_pass = 0;
#define CHECK(...)                                                           \
  do {                                                                       \
    if (__VA_ARGS__) {                                                       \
      ++g_pass;                                                              \
    } else {                                                                 \
      ++g_fail;                                                              \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, T)        \
  do {                                  \
    bool ok_ = false;                   \
    try {                               \
      (void)(expr);                     \
    } catch (const T&) {                \
      ok_ = true;                       \
    } catch (...) {                     \
    }                                   \
    CHECK(ok_ && #expr);                \
  } while (0)

static std::vector<ParamVector> random_peers(std::size_t n, std::size_t dim, RngStream& s) {
  std::vector<ParamVector> peers(n);
  for (auto& v : peers) {
    v.resize(dim);
    for (auto& x : v) x = s.uniform();
  }
  return peers;
}

static void hex(const char* tag, double x) {
  unsigned char b[8];
  std::memcpy(b, &x, 8);
  std::printf("%s=", tag);
  for (int i = 0; i < 8; ++i) std::printf("%02x", b[i]);
  std::printf("\n");
}

int main() {
  // test_core.cpp:32-48
  {
    ParamVector a{1.0, 2.0}, b{3.0, 6.0};
    CHECK((group_mean({&a, &b}) == ParamVector{2.0, 4.0}));
    std::vector<ParamVector> peers{{1.0}, {3.0}};
    CHECK(distortion(peers, ParamVector{2.0}) == 1.0);
    std::vector<ParamVector> same{{5.0, 5.0}, {5.0, 5.0}};
    CHECK(distortion(same, ParamVector{5.0, 5.0}) == 0.0);
    std::vector<ParamVector> bad{{1.0}, {1.0, 2.0}};
    CHECK_THROWS_AS(distortion(bad, ParamVector{2.0}), std::invalid_argument);
    CHECK(GridConfig{3, 2, 1}.capacity() == 9);
    CHECK_THROWS_AS((GridConfig{0, 2, 1}.validate()), std::invalid_argument);
  }
  // test_core.cpp:66-86
  {
    Rng a(7), b(7);
    auto s1 = a.stream("x"), s2 = b.stream("x"), s3 = a.stream("y");
    bool eq = true, neq = true;
    for (int i = 0; i < 64; ++i) {
      const auto v = s1();
      eq = eq && v == s2();
      neq = neq && v == s3();
    }
    CHECK(eq);
    CHECK(!neq);
  }
  // test_matchmaking.cpp:39-68
  {
    const GridConfig grid{3, 3, 1};
    CHECK((matchmaking::initial_index(0, grid).indices == std::vector<std::uint32_t>{0, 0}));
    CHECK((matchmaking::initial_index(5, grid).indices == std::vector<std::uint32_t>{1, 0}));
    CHECK((matchmaking::initial_index(26, grid).indices == std::vector<std::uint32_t>{2, 2}));
    CHECK_THROWS_AS(matchmaking::initial_index(27, grid), std::out_of_range);
    CHECK(matchmaking::initial_index(2, GridConfig{5, 1, 1}).indices.empty());
    const GridConfig g4{4, 3, 1};
    CHECK((matchmaking::next_group_key(GroupKey{{1, 2}}, 3, g4).indices ==
           std::vector<std::uint32_t>{2, 3}));
    CHECK_THROWS_AS(matchmaking::next_group_key(GroupKey{{1, 2}}, 4, g4), std::out_of_range);
    std::map<GroupKey, int> counts;
    for (std::uint64_t c = 0; c < g4.capacity(); ++c) counts[matchmaking::initial_index(c, g4)]++;
    CHECK(counts.size() == 16);
    for (auto& [k, c] : counts) CHECK(c == 4);
  }
  // test_matchmaking.cpp:70-106 (closed form)
  {
    Rng rng(2);
    auto stream = rng.stream("priorities");
    std::vector<matchmaking::MatchPeer> peers;
    for (std::uint32_t k = 0; k < 4; ++k)
      for (std::uint32_t i = 0; i < 5; ++i)
        peers.push_back(matchmaking::MatchPeer{k * 5 + i, GroupKey{{k}}, stream() >> 16, 0});
    const auto groups = matchmaking::form_groups_uncontested(peers);
    CHECK(groups.size() == 4);
    for (const auto& g : groups) {
      std::set<std::uint32_t> keys;
      for (PeerId m : g.members) keys.insert(peers[m].key.indices[0]);
      CHECK(keys.size() == 1);
      CHECK(g.members.size() == 5);
      CHECK(g.leader == g.members.front());
      for (std::size_t i = 1; i < g.members.size(); ++i)
        CHECK((matchmaking::Priority{peers[g.members[i - 1]].timestamp, g.members[i - 1]} <
               matchmaking::Priority{peers[g.members[i]].timestamp, g.members[i]}));
    }
  }
  // test_allreduce.cpp:46-88
  {
    Rng rng(2);
    auto stream = rng.stream("v");
    for (std::size_t n : {1u, 2u, 5u, 8u}) {
      std::vector<ParamVector> inputs(n);
      ParamVector mean(6, 0.0);
      for (auto& v : inputs) {
        v = stream.normals(6);
        for (std::size_t j = 0; j < 6; ++j) mean[j] += v[j] / n;
      }
      const auto out =
          allreduce::butterfly_allreduce(inputs, allreduce::PartitionWeights::uniform(n));
      CHECK(out.completed);
      CHECK(out.chunks.size() == n);
      for (const auto& v : out.vectors)
        for (std::size_t j = 0; j < 6; ++j) CHECK(std::abs(v[j] - mean[j]) <= 1e-12);
    }
    std::vector<ParamVector> in2{{1.0, 2.0, 3.0, 10.0}, {3.0, 4.0, 5.0, 20.0}};
    CHECK(allreduce::butterfly_allreduce(in2, allreduce::PartitionWeights::uniform(2)).vectors ==
          allreduce::butterfly_allreduce(in2, allreduce::PartitionWeights{{0.9, 0.1}}).vectors);
    std::vector<ParamVector> in3{{1.0}, {2.0}, {3.0}};
    const auto v = allreduce::butterfly_allreduce(in3, allreduce::PartitionWeights::uniform(3),
                                                  {false, true, false});
    CHECK(!v.completed);
    CHECK(v.vectors == in3);
    CHECK((v.chunks == std::vector<std::uint32_t>{0, 1, 2}));
    std::vector<ParamVector> bad{{1.0}, {2.0, 3.0}};
    CHECK_THROWS_AS(allreduce::butterfly_allreduce(bad, allreduce::PartitionWeights::uniform(2)),
                    std::invalid_argument);
    CHECK((allreduce::chunk_sizes(8, allreduce::PartitionWeights{{0.5, 0.25, 0.125, 0.125}}) ==
           std::vector<std::size_t>{4, 2, 1, 1}));
  }
  // test_protocols.cpp:34-122, 190-200
  {
    Rng seed_rng(10);
    auto stream = seed_rng.stream("init");
    const auto initial = random_peers(9, 2, stream);
    const auto report =
        protocols::run_moshpit(GridConfig{3, 2, 1}, initial, FailureModel{}, Rng(99), 4);
    CHECK(report.distortion[0] > 1e-24);
    CHECK(report.distortion[1] <= 1e-24);
    CHECK(report.distortion[3] <= 1e-24);
    const std::vector<ParamVector> one{{3.0, 4.0}};
    const auto r1 = protocols::run_moshpit(GridConfig{4, 2, 1}, one, FailureModel{}, Rng(1), 3);
    CHECK(r1.initial_distortion == 0.0);
    CHECK(r1.rounds_to(1e-9, 50) == 0);
    CHECK_THROWS_AS(protocols::run_moshpit(GridConfig{2, 2, 1},
                                           std::vector<ParamVector>(5, ParamVector{1.0}),
                                           FailureModel{}, Rng(1), 1),
                    std::invalid_argument);
    Rng s11(11);
    for (int trial = 0; trial < 5; ++trial) {
      auto st = s11.stream("init", trial);
      const auto init = random_peers(24, 3, st);
      const auto r = protocols::run_moshpit(GridConfig{5, 2, 1}, init,
                                            FailureModel{trial * 0.05, {}}, Rng(1000 + trial), 10);
      for (double drift : r.mean_drift) CHECK(drift <= 1e-12);
    }
    Rng s19(19);
    auto st19 = s19.stream("init");
    const auto init30 = random_peers(30, 2, st19);
    const auto a = protocols::run_moshpit(GridConfig{6, 2, 1}, init30, FailureModel{0.05, {}},
                                          Rng(12), 20);
    const auto b = protocols::run_moshpit(GridConfig{6, 2, 1}, init30, FailureModel{0.05, {}},
                                          Rng(12), 20);
    CHECK(a.distortion == b.distortion);
    CHECK(a.active_counts == b.active_counts);
    CHECK(protocols::TrialReport{1.0, {0.5, 1e-5, 1e-10}, {}, {}, 0}.rounds_to(1e-4, 50) == 2);
  }
  // optimizer.hpp:249-284 through the drop-in: full grid averages exactly
  {
    Rng r(5);
    auto st = r.stream("init");
    auto thetas = random_peers(16, 3, st);
    const auto m0 = mean_of(thetas);
    auto avg = r.stream("averaging");
    optimizer::detail::moshpit_average(thetas, GridConfig{4, 2, 1}, 2, avg);
    for (const auto& t : thetas)
      for (std::size_t j = 0; j < 3; ++j) CHECK(std::abs(t[j] - m0[j]) <= 1e-15);
  }
  // test_optimizer.cpp:60-98, 160-193 through the drop-in (GPU)
  {
    const optimizer::Quadratic quad(2, 2.0, 2.0, ParamVector{1.0, 1.0});
    ParamVector theta{0.0, 0.0};
    Rng rng(23);
    auto noise = rng.stream("n");
    optimizer::local_step(theta, quad, 0.25, 0.0, noise);
    CHECK(std::abs(theta[0] - 0.5) < 1e-12);
    CHECK(std::abs(theta[1] - 0.5) < 1e-12);

    Rng r24(24);
    auto st = r24.stream("target");
    const optimizer::Quadratic q4(4, 5.0, 0.5, st.normals(4));
    optimizer::OptimizerConfig cfg;
    cfg.gamma = 0.05;
    cfg.tau = 1;
    cfg.steps = 60;
    cfg.grid = GridConfig{4, 2, 1};
    cfg.n_peers = 9;
    const ParamVector theta0(4, 2.0);
    const auto res = optimizer::run_moshpit_sgd(cfg, q4, theta0, {}, Rng(500));
    ParamVector th = theta0;
    for (std::uint32_t k = 0; k < cfg.steps; ++k) {
      const auto g = q4.gradient(th);
      for (std::size_t j = 0; j < th.size(); ++j) th[j] -= cfg.gamma * g[j];
      CHECK(std::abs(res.f_gap[k] - q4.value(th)) <= 1e-12);
      CHECK(res.diagnostics.dispersion[k] <= 1e-24);
    }
    const optimizer::Quadratic q2(2, 2.0, 1.0, ParamVector(2, 1.0));
    optimizer::OptimizerConfig c2;
    c2.gamma = 0.1;
    c2.tau = 2;
    c2.steps = 20;
    c2.sigma = 0.5;
    c2.grid = GridConfig{4, 2, 1};
    c2.n_peers = 8;
    const auto rm = optimizer::run_moshpit_sgd(c2, q2, ParamVector(2, 0.0), {{5, -3}, {12, +2}},
                                               Rng(777));
    CHECK(rm.diagnostics.n_min == 5);
    CHECK(rm.f_gap.size() == c2.steps);
    CHECK_THROWS_AS(optimizer::run_moshpit_sgd(c2, q2, ParamVector(2, 0.0), {{3, -8}}, Rng(1)),
                    std::invalid_argument);
    optimizer::OptimizerConfig bad;
    bad.grid = GridConfig{2, 2, 1};
    bad.n_peers = 5;
    CHECK_THROWS_AS(bad.validate(), std::invalid_argument);
  }
  // test_optimizer.cpp:30-58 (LogisticRegression through the drop-in: GPU
  // value/gradient vs central finite differences, objective constants) and a
  // GPU run_moshpit_sgd on the logistic objective.
  {
    Rng rng(21);
    auto stream = rng.stream("theta");
    (void)stream.normals(6);  // the Quadratic's target in the reference test
    const auto logit = optimizer::LogisticRegression::synthetic(5, 80, 0.05, stream);
    for (int trial = 0; trial < 10; ++trial) {
      const ParamVector theta = stream.normals(5);
      const ParamVector g = logit.gradient(theta);
      for (std::size_t j = 0; j < theta.size(); ++j) {
        const double h = 1e-6 * std::max(1.0, std::abs(theta[j]));
        ParamVector lo = theta, hi = theta;
        lo[j] -= h;
        hi[j] += h;
        const double fd = (logit.value(hi) - logit.value(lo)) / (2.0 * h);
        const double scale = std::max({std::abs(g[j]), std::abs(fd), 1e-8});
        CHECK(std::abs(g[j] - fd) / scale <= 1e-6);
      }
    }
    Rng r22(22);
    auto st22 = r22.stream("t");
    const auto l4 = optimizer::LogisticRegression::synthetic(4, 50, 0.1, st22);
    CHECK(l4.smoothness() >= l4.strong_convexity());
    CHECK_THROWS_AS(optimizer::LogisticRegression({}, {}, 0.1), std::invalid_argument);
    optimizer::OptimizerConfig cfg;
    cfg.gamma = 0.3;
    cfg.tau = 2;
    cfg.steps = 30;
    cfg.sigma = 0.2;
    cfg.grid = GridConfig{4, 2, 1};
    cfg.n_peers = 16;
    const auto res = optimizer::run_moshpit_sgd(cfg, l4, ParamVector(4, 0.0), {}, Rng(3));
    CHECK(res.f_gap.size() == cfg.steps);
    CHECK(res.f_gap.back() < l4.value(ParamVector(4, 0.0)));
    ParamVector th(4, 0.0);
    auto nz = Rng(5).stream("noise");
    optimizer::local_step(th, l4, 0.5, 0.0, nz);
    const auto g0 = l4.gradient(ParamVector(4, 0.0));
    for (std::size_t j = 0; j < 4; ++j) CHECK(std::abs(th[j] + 0.5 * g0[j]) <= 1e-15);
  }
  // golden case: counter init, C2-shaped (32x32, p=0.01, 10 rounds), dim 4
  {
    const std::size_t n = 1024, dim = 4;
    std::vector<ParamVector> init(n, ParamVector(dim));
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = 0; j < dim; ++j) {
        std::uint64_t s = 0x5EEDull ^ (static_cast<std::uint64_t>(i) << 32) ^ j;
        std::uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        init[i][j] = static_cast<double>(z >> 40) * 0x1.0p-24;
      }
    const auto r = protocols::run_moshpit(GridConfig{32, 2, 1}, init, FailureModel{0.01, {}},
                                          Rng(7), 10);
    hex("initial_distortion", r.initial_distortion);
    for (std::size_t t = 0; t < r.distortion.size(); ++t) {
      hex("distortion", r.distortion[t]);
      hex("mean_drift", r.mean_drift[t]);
      std::printf("active=%u\n", r.active_counts[t]);
    }
    hex("cost_units", r.cost_units);
  }
  std::printf("PASS=%d FAIL=%d\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
