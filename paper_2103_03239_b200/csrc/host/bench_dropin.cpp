// bench_dropin.cpp -- times the reference-facing C++ call a reference user
// makes after swapping headers: moshpit::protocols::run_moshpit (the drop-in,
// include/moshpit_b200/moshpit.hpp) on a std::vector<ParamVector> (pageable
// host memory, fp64, EXACT diagnostics: the TrialReport is bit-identical to
// the reference's).  The vectors are filled with the bench's counter-based
// init (outside the timed region, on all cores).  Prints one JSON line.
//
//   bench_dropin M d n dim p rounds reps
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "moshpit_b200/moshpit.hpp"

static std::uint64_t splitmix64(std::uint64_t s) {
  std::uint64_t z = s + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s M d n dim p rounds reps\n", argv[0]);
    return 2;
  }
  const std::uint32_t M = std::atoi(argv[1]), d = std::atoi(argv[2]);
  const std::size_t n = std::strtoull(argv[3], nullptr, 10);
  const std::size_t dim = std::strtoull(argv[4], nullptr, 10);
  const double p = std::atof(argv[5]);
  const std::uint32_t rounds = std::atoi(argv[6]), reps = std::atoi(argv[7]);
  const std::uint64_t seed = 0x5EED;
  std::vector<moshpit::ParamVector> initial(n);
  {
    const unsigned T = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (std::size_t i = n * t / T; i < n * (t + 1) / T; ++i) {
          initial[i].resize(dim);
          for (std::size_t j = 0; j < dim; ++j)
            initial[i][j] = (double)(splitmix64(seed ^ (i << 32) ^ j) >> 40) * 0x1.0p-24;
        }
      });
    for (auto& x : th) x.join();
  }
  const moshpit::GridConfig grid{M, d, rounds};
  const moshpit::FailureModel failure{p, {}};
  std::vector<double> secs;
  moshpit::protocols::TrialReport rep;
  for (std::uint32_t k = 0; k < reps + 1; ++k) {  // first call = warm-up (module load)
    const auto t0 = std::chrono::steady_clock::now();
    rep = moshpit::protocols::run_moshpit(grid, initial, failure, moshpit::Rng(7), rounds);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (k) secs.push_back(s);
  }
  std::vector<double> sorted = secs;
  std::sort(sorted.begin(), sorted.end());
  const double med = sorted[sorted.size() / 2];
  std::printf("{\"call\": \"moshpit::protocols::run_moshpit (drop-in header, fp64, EXACT "
              "diagnostics, std::vector<ParamVector> pageable rows)\", \"n\": %zu, \"dim\": %zu, "
              "\"rounds\": %u, \"p\": %g, \"seconds_median\": %.6f, \"seconds\": [",
              n, dim, rounds, p, med);
  for (std::size_t i = 0; i < secs.size(); ++i) std::printf("%s%.6f", i ? ", " : "", secs[i]);
  std::printf("], \"initial_distortion\": %.17g, \"final_distortion\": %.17g, "
              "\"final_active\": %u, \"rounds_to_1e-9\": %u}\n",
              rep.initial_distortion, rep.distortion.back(), rep.active_counts.back(),
              rep.rounds_to(1e-9, rounds));
  return 0;
}
