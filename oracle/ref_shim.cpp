// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// headers (compiled from /root/reference/proj/include where they lie; no
// reference source is copied into this repo).  TEST INFRASTRUCTURE ONLY:
// built by oracle/Makefile into oracle/_ref/libmoshpit_ref.so and used by
// tests/ (to pin the oracle), tests/golden/gen_golden.py (to make the golden
// vectors) and bench.py's CPU reference arm.
#include <atomic>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "moshpit/allreduce.hpp"
#include "moshpit/core.hpp"
#include "moshpit/matchmaking.hpp"
#include "moshpit/optimizer.hpp"
#include "moshpit/protocols.hpp"
#include "moshpit/rng.hpp"

using namespace moshpit;

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (const std::out_of_range&) {
    return -2;
  } catch (const std::runtime_error&) {
    return -3;
  } catch (...) {
    return -4;
  }
}

std::vector<ParamVector> rows_of(const double* x, std::uint64_t n,
                                 std::uint64_t dim) {
  std::vector<ParamVector> v(n, ParamVector(dim));
  for (std::uint64_t i = 0; i < n; ++i)
    std::memcpy(v[i].data(), x + i * dim, dim * sizeof(double));
  return v;
}

void fill_report(const protocols::TrialReport& r, double* init_d, double* dist,
                 double* drift, std::uint32_t* active, double* cost) {
  *init_d = r.initial_distortion;
  for (std::size_t t = 0; t < r.distortion.size(); ++t) {
    dist[t] = r.distortion[t];
    drift[t] = r.mean_drift[t];
    active[t] = r.active_counts[t];
  }
  *cost = r.cost_units;
}

double init_value(std::uint64_t seed, std::uint64_t i, std::uint64_t j) {
  std::uint64_t s = seed ^ (i << 32) ^ j;
  return static_cast<double>(detail::splitmix64(s) >> 40) * 0x1.0p-24;
}

}  // namespace

extern "C" {

void ref_stream_draws(std::uint64_t root, const char* name, std::int64_t index,
                      int kind, std::uint64_t arg, double arg_f, std::uint64_t n,
                      void* out) {
  Rng rng(root);
  RngStream s = index < 0 ? rng.stream(name)
                          : rng.stream(name, static_cast<std::uint64_t>(index));
  for (std::uint64_t i = 0; i < n; ++i) {
    switch (kind) {
      case 0: static_cast<std::uint64_t*>(out)[i] = s(); break;
      case 1: static_cast<double*>(out)[i] = s.uniform(); break;
      case 2: static_cast<std::uint64_t*>(out)[i] = s.below(arg); break;
      case 3: static_cast<double*>(out)[i] = s.normal(); break;
      default: static_cast<std::uint8_t*>(out)[i] = s.bernoulli(arg_f); break;
    }
  }
}

int ref_initial_index(std::uint64_t cell, std::uint32_t M, std::uint32_t d,
                      std::uint32_t* key) {
  return guarded([&] {
    const auto k = matchmaking::initial_index(cell, GridConfig{M, d, 1});
    for (std::size_t i = 0; i < k.indices.size(); ++i) key[i] = k.indices[i];
  });
}

int ref_next_group_key(const std::uint32_t* key, std::uint32_t klen,
                       std::uint32_t chunk, std::uint32_t M, std::uint32_t* out) {
  return guarded([&] {
    GroupKey k;
    k.indices.assign(key, key + klen);
    const auto nk = matchmaking::next_group_key(k, chunk, GridConfig{M, klen + 1, 1});
    for (std::size_t i = 0; i < nk.indices.size(); ++i) out[i] = nk.indices[i];
  });
}

std::int64_t ref_form_groups_uncontested(std::uint64_t n, const std::uint32_t* ids,
                                         const std::uint32_t* keys,
                                         std::uint32_t klen,
                                         const std::uint64_t* ts, std::uint32_t cap,
                                         std::uint32_t* members,
                                         std::uint32_t* group_off) {
  std::vector<matchmaking::MatchPeer> peers(n);
  for (std::uint64_t i = 0; i < n; ++i) {
    peers[i].id = ids[i];
    peers[i].key.indices.assign(keys + i * klen, keys + (i + 1) * klen);
    peers[i].timestamp = ts[i];
  }
  const auto groups = matchmaking::form_groups_uncontested(peers, cap);
  std::uint32_t p = 0;
  for (std::size_t g = 0; g < groups.size(); ++g) {
    group_off[g] = p;
    for (auto id : groups[g].members) members[p++] = id;
  }
  group_off[groups.size()] = p;
  return static_cast<std::int64_t>(groups.size());
}

int ref_chunk_sizes(std::uint64_t dim, const double* w, std::uint64_t n,
                    std::uint64_t* sizes) {
  return guarded([&] {
    const auto s = allreduce::chunk_sizes(
        dim, allreduce::PartitionWeights{std::vector<double>(w, w + n)});
    for (std::size_t i = 0; i < s.size(); ++i) sizes[i] = s[i];
  });
}

double ref_pairwise_sum(const double* xs, std::uint64_t n) {
  return pairwise_sum(std::vector<double>(xs, xs + n));
}

int ref_group_mean(const double* rows, std::uint64_t n, std::uint64_t dim,
                   const std::uint32_t* members, double* out) {
  return guarded([&] {
    const auto v = rows_of(rows, n, dim);
    std::vector<const ParamVector*> ptrs;
    for (std::uint64_t i = 0; i < n; ++i) ptrs.push_back(&v[members ? members[i] : i]);
    const auto m = group_mean(ptrs);
    std::memcpy(out, m.data(), dim * sizeof(double));
  });
}

int ref_butterfly(const double* inputs, std::uint64_t n, std::uint64_t dim,
                  const std::uint8_t* failed, double* out, int* completed,
                  std::uint32_t* chunks) {
  return guarded([&] {
    const auto v = rows_of(inputs, n, dim);
    std::vector<bool> f;
    if (failed)
      for (std::uint64_t i = 0; i < n; ++i) f.push_back(failed[i] != 0);
    const auto o = allreduce::butterfly_allreduce(
        v, allreduce::PartitionWeights::uniform(n), f);
    *completed = o.completed;
    for (std::uint64_t i = 0; i < n; ++i) {
      std::memcpy(out + i * dim, o.vectors[i].data(), dim * sizeof(double));
      chunks[i] = o.chunks[i];
    }
  });
}

// One CONTESTED matchmaking round (matchmaking.hpp:104-294, form_groups
// :325-333) with skewed arrivals and FailStop injections, drawn as in
// test_matchmaking.cpp:153-181, followed by butterfly_allreduce of every
// sealed group (allreduce.hpp:79-121) with failed = "the member fail-stopped
// this round" (a group with any such member is void, protocols.hpp:162-170).
// Outputs the group table (members in sealed priority order, offsets, void
// flags) and the vectors after the round (peers in no group keep theirs).
int ref_contested_round(std::uint64_t trial_seed, std::uint32_t n, std::uint32_t nkeys,
                        std::uint32_t cap, const double* x, std::uint64_t dim,
                        std::uint32_t* members, std::uint32_t* goff, std::uint32_t* n_groups,
                        std::uint8_t* void_flags, double* out) {
  using namespace matchmaking;
  return guarded([&] {
    auto stream = Rng(trial_seed).stream("trial");
    std::vector<MatchPeer> peers;
    for (std::uint32_t i = 0; i < n; ++i)
      peers.push_back(MatchPeer{static_cast<PeerId>(i),
                                GroupKey{{static_cast<std::uint32_t>(stream.below(nkeys))}},
                                stream() >> 16, stream.below(3)});
    std::vector<FailStop> failures;
    const std::size_t n_failures = stream.below(n / 2 + 1);
    std::vector<bool> dead(n, false);
    for (std::size_t f = 0; f < n_failures; ++f) {
      failures.push_back(FailStop{stream.below(8), static_cast<PeerId>(stream.below(n))});
      dead[failures.back().peer] = true;
    }
    Dht dht(1000);
    const auto result = form_groups(0, peers, dht, failures, cap ? 3 + 2 * (LogicalTime)n : 3,
                                    cap ? cap : std::numeric_limits<std::uint32_t>::max());
    auto v = rows_of(x, n, dim);
    std::uint32_t k = 0, g = 0;
    goff[0] = 0;
    for (const auto& sg : result.groups) {
      std::vector<ParamVector> in;
      std::vector<bool> failed;
      bool any = false;
      for (PeerId m : sg.members) {
        members[k++] = m;
        in.push_back(v[m]);
        failed.push_back(dead[m]);
        any = any || dead[m];
      }
      const auto o = allreduce::butterfly_allreduce(
          in, allreduce::PartitionWeights::uniform(in.size()), failed);
      for (std::size_t q = 0; q < sg.members.size(); ++q) v[sg.members[q]] = o.vectors[q];
      void_flags[g] = any ? 1 : 0;
      goff[++g] = k;
    }
    *n_groups = g;
    for (std::uint32_t i = 0; i < n; ++i) std::memcpy(out + i * dim, v[i].data(), dim * 8);
  });
}

double ref_distortion(const double* peers, std::uint64_t n, std::uint64_t dim,
                      const double* ref) {
  return distortion(rows_of(peers, n, dim), ParamVector(ref, ref + dim));
}

int ref_mean_of(const double* peers, std::uint64_t n, std::uint64_t dim,
                double* out) {
  return guarded([&] {
    const auto m = mean_of(rows_of(peers, n, dim));
    std::memcpy(out, m.data(), dim * sizeof(double));
  });
}

double ref_complexity_estimate(std::uint32_t t, std::uint32_t n, std::uint32_t m,
                               std::uint32_t dim) {
  return theory::complexity_estimate(t, n, m, dim);
}

// The unmodified protocols::run_moshpit (protocols.hpp:108-179).
int ref_run_moshpit(std::uint32_t M, std::uint32_t d, std::uint32_t T,
                    const double* initial, std::uint64_t n, std::uint64_t dim,
                    double p, std::uint64_t seed, std::uint32_t rounds,
                    double* init_d, double* dist, double* drift,
                    std::uint32_t* active, double* cost) {
  return guarded([&] {
    const auto r = protocols::run_moshpit(GridConfig{M, d, T}, rows_of(initial, n, dim),
                                          FailureModel{p, {}}, Rng(seed), rounds);
    fill_report(r, init_d, dist, drift, active, cost);
  });
}

// run_moshpit's loop restated from the reference's own public functions so
// that the final vectors (which run_moshpit never returns) are observable.
// tests/test_oracle_vs_ref.py checks its report equals ref_run_moshpit's.
int ref_run_moshpit_vectors(std::uint32_t M, std::uint32_t d, std::uint32_t T,
                            const double* initial, std::uint64_t n,
                            std::uint64_t dim, double p, std::uint64_t seed,
                            std::uint32_t rounds, double* init_d, double* dist,
                            double* drift, std::uint32_t* active, double* cost,
                            double* final_vectors) {
  return guarded([&] {
    const GridConfig grid{M, d, T};
    grid.validate();
    const FailureModel failure{p, {}};
    failure.validate();
    const Rng rng(seed);
    const auto init = rows_of(initial, n, dim);
    if (n == 0 || n > grid.capacity()) throw std::invalid_argument("n");
    const ParamVector reference = mean_of(init);
    protocols::TrialReport report;
    report.initial_distortion = distortion(init, reference);
    auto cell_stream = rng.stream("cells");
    std::vector<std::uint64_t> cells(grid.capacity());
    for (std::uint64_t i = 0; i < cells.size(); ++i) cells[i] = i;
    for (std::size_t i = 0; i < n; ++i) {
      const std::size_t j = i + cell_stream.below(cells.size() - i);
      std::swap(cells[i], cells[j]);
    }
    auto vectors = init;
    std::vector<GroupKey> keys(n);
    for (std::size_t i = 0; i < n; ++i) keys[i] = matchmaking::initial_index(cells[i], grid);
    auto fail_stream = rng.stream("failures");
    auto clock_stream = rng.stream("priorities");
    for (std::uint32_t round = 1; round <= rounds; ++round) {
      const auto failed = protocols::detail::draw_failures(fail_stream, n, p);
      std::vector<matchmaking::MatchPeer> declared(n);
      for (std::size_t i = 0; i < n; ++i)
        declared[i] = matchmaking::MatchPeer{static_cast<PeerId>(i), keys[i],
                                             clock_stream() >> 16, 0};
      const auto groups = matchmaking::form_groups_uncontested(declared, M);
      std::uint32_t act = 0;
      for (const auto& group : groups) {
        std::vector<ParamVector> inputs;
        std::vector<bool> gf;
        for (PeerId id : group.members) {
          inputs.push_back(vectors[id]);
          gf.push_back(failed[id]);
        }
        const auto out = allreduce::butterfly_allreduce(
            inputs, allreduce::PartitionWeights::uniform(inputs.size()), gf);
        for (std::size_t k = 0; k < group.members.size(); ++k) {
          const PeerId id = group.members[k];
          if (out.completed) vectors[id] = out.vectors[k];
          keys[id] = matchmaking::next_group_key(keys[id], out.chunks[k], grid);
          act += !failed[id];
        }
      }
      protocols::detail::record_round(report, vectors, reference, act);
    }
    report.cost_units = theory::complexity_estimate(rounds, static_cast<std::uint32_t>(n),
                                                    M, static_cast<std::uint32_t>(dim));
    fill_report(report, init_d, dist, drift, active, cost);
    for (std::uint64_t i = 0; i < n; ++i)
      std::memcpy(final_vectors + i * dim, vectors[i].data(), dim * sizeof(double));
  });
}

// optimizer::detail::moshpit_average over Rng(seed).stream(name).
int ref_moshpit_average(double* thetas, std::uint64_t n, std::uint64_t dim,
                        std::uint32_t M, std::uint32_t d, std::uint32_t rounds,
                        std::uint64_t seed, const char* name) {
  return guarded([&] {
    auto v = rows_of(thetas, n, dim);
    auto s = Rng(seed).stream(name);
    optimizer::detail::moshpit_average(v, GridConfig{M, d, 1}, rounds, s);
    for (std::uint64_t i = 0; i < n; ++i)
      std::memcpy(thetas + i * dim, v[i].data(), dim * sizeof(double));
  });
}

// optimizer::run_moshpit_sgd with the Quadratic objective (optimizer.hpp:297).
int ref_sgd_quadratic(std::uint32_t M, std::uint32_t d, std::uint32_t T, std::uint32_t n_peers,
                      std::uint64_t dim, double L, double mu, const double* target,
                      const double* theta0, double gamma, std::uint32_t tau,
                      std::uint32_t steps, double sigma, std::uint32_t inner_rounds,
                      std::uint64_t seed, const std::uint32_t* ev_step,
                      const std::int32_t* ev_delta, std::uint64_t n_events, double* f_gap,
                      double* grad_norm_sq, double* f_gap_weighted, double* dispersion,
                      double* final_mean, double* diag6) {
  return guarded([&] {
    const optimizer::Quadratic quad(dim, L, mu, ParamVector(target, target + dim));
    optimizer::OptimizerConfig cfg;
    cfg.gamma = gamma;
    cfg.tau = tau;
    cfg.steps = steps;
    cfg.grid = GridConfig{M, d, T};
    cfg.sigma = sigma;
    cfg.n_peers = n_peers;
    cfg.inner_rounds = inner_rounds;
    std::vector<optimizer::MembershipEvent> sched;
    for (std::uint64_t e = 0; e < n_events; ++e) sched.push_back({ev_step[e], ev_delta[e]});
    const auto r = optimizer::run_moshpit_sgd(cfg, quad, ParamVector(theta0, theta0 + dim), sched,
                                              Rng(seed));
    for (std::size_t k = 0; k < r.f_gap.size(); ++k) {
      f_gap[k] = r.f_gap[k];
      grad_norm_sq[k] = r.grad_norm_sq[k];
      f_gap_weighted[k] = r.f_gap_weighted[k];
      dispersion[k] = r.diagnostics.dispersion[k];
    }
    for (std::size_t j = 0; j < r.final_mean.size(); ++j) final_mean[j] = r.final_mean[j];
    diag6[0] = r.diagnostics.delta_aq_hat;
    diag6[1] = r.diagnostics.sigma_hat;
    diag6[2] = r.diagnostics.delta_pv1_hat;
    diag6[3] = r.diagnostics.delta_pv2_hat;
    diag6[4] = r.diagnostics.n_min;
    diag6[5] = 0;
  });
}

// optimizer::local_step with the Quadratic objective over Rng(seed).stream(name).
int ref_local_step_quadratic(double* theta, std::uint64_t dim, double L, double mu,
                             const double* target, double gamma, double sigma,
                             std::uint64_t seed, const char* name) {
  return guarded([&] {
    const optimizer::Quadratic quad(dim, L, mu, ParamVector(target, target + dim));
    ParamVector th(theta, theta + dim);
    auto s = Rng(seed).stream(name);
    optimizer::local_step(th, quad, gamma, sigma, s);
    std::memcpy(theta, th.data(), dim * sizeof(double));
  });
}

// LogisticRegression(xs, ys, l2) value / gradient / smoothness (optimizer.hpp:75-146).
int ref_logistic_eval(const double* xs, const double* ys, std::uint64_t samples, std::uint64_t dim,
                      double l2, const double* theta, double* value, double* grad,
                      double* smooth) {
  return guarded([&] {
    const optimizer::LogisticRegression lr(rows_of(xs, samples, dim),
                                           std::vector<double>(ys, ys + samples), l2);
    const ParamVector th(theta, theta + dim);
    *value = lr.value(th);
    const auto g = lr.gradient(th);
    std::memcpy(grad, g.data(), dim * sizeof(double));
    *smooth = lr.smoothness();
  });
}

// LogisticRegression::synthetic over Rng(data_seed).stream(name), evaluated at
// theta: pins the oracle's dataset generation without exposing private data.
int ref_logistic_synthetic_eval(std::uint64_t dim, std::uint64_t samples, double l2,
                                std::uint64_t data_seed, const char* name, const double* theta,
                                double* value, double* grad, double* smooth) {
  return guarded([&] {
    auto st = Rng(data_seed).stream(name);
    const auto lr = optimizer::LogisticRegression::synthetic(dim, samples, l2, st);
    const ParamVector th(theta, theta + dim);
    *value = lr.value(th);
    const auto g = lr.gradient(th);
    std::memcpy(grad, g.data(), dim * sizeof(double));
    *smooth = lr.smoothness();
  });
}

// run_moshpit_sgd with LogisticRegression::synthetic(dim, samples, l2,
// Rng(data_seed).stream(name)).
int ref_sgd_logistic(std::uint32_t M, std::uint32_t d, std::uint32_t T, std::uint32_t n_peers,
                     std::uint64_t dim, std::uint64_t samples, double l2,
                     std::uint64_t data_seed, const char* name, const double* theta0,
                     double gamma, std::uint32_t tau, std::uint32_t steps, double sigma,
                     std::uint32_t inner_rounds, std::uint64_t seed, double* f_gap,
                     double* grad_norm_sq, double* f_gap_weighted, double* dispersion,
                     double* final_mean, double* diag6) {
  return guarded([&] {
    auto st = Rng(data_seed).stream(name);
    const auto lr = optimizer::LogisticRegression::synthetic(dim, samples, l2, st);
    optimizer::OptimizerConfig cfg;
    cfg.gamma = gamma;
    cfg.tau = tau;
    cfg.steps = steps;
    cfg.grid = GridConfig{M, d, T};
    cfg.sigma = sigma;
    cfg.n_peers = n_peers;
    cfg.inner_rounds = inner_rounds;
    const auto r = optimizer::run_moshpit_sgd(cfg, lr, ParamVector(theta0, theta0 + dim), {},
                                              Rng(seed));
    for (std::size_t k = 0; k < r.f_gap.size(); ++k) {
      f_gap[k] = r.f_gap[k];
      grad_norm_sq[k] = r.grad_norm_sq[k];
      f_gap_weighted[k] = r.f_gap_weighted[k];
      dispersion[k] = r.diagnostics.dispersion[k];
    }
    for (std::size_t j = 0; j < r.final_mean.size(); ++j) final_mean[j] = r.final_mean[j];
    diag6[0] = r.diagnostics.delta_aq_hat;
    diag6[1] = r.diagnostics.sigma_hat;
    diag6[2] = r.diagnostics.delta_pv1_hat;
    diag6[3] = r.diagnostics.delta_pv2_hat;
    diag6[4] = r.diagnostics.n_min;
    diag6[5] = 0;
  });
}

// CPU baseline: the unmodified run_moshpit on `slices` column slices of
// width `width` of the counter-initialised state, spread over
// `threads` host threads.  Coordinates are independent, so each slice is
// bit-identical to those coordinates of a full-D run.  Init is excluded
// from *run_s; *init_s reports it.
int ref_slice_bench(std::uint32_t M, std::uint32_t d, std::uint64_t n,
                    std::uint64_t width, std::uint64_t slices, std::uint64_t col0,
                    std::uint64_t init_seed, std::uint64_t seed, double p,
                    std::uint32_t rounds, std::uint32_t threads, double* run_s,
                    double* init_s, double* checksum) {
  return guarded([&] {
    if (threads == 0) threads = 1;
    std::vector<std::vector<ParamVector>> inits(slices);
    const auto t0 = std::chrono::steady_clock::now();
    {
      std::vector<std::thread> pool;
      for (std::uint32_t t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
          for (std::uint64_t s = t; s < slices; s += threads) {
            auto& v = inits[s];
            v.assign(n, ParamVector(width));
            for (std::uint64_t i = 0; i < n; ++i)
              for (std::uint64_t j = 0; j < width; ++j)
                v[i][j] = init_value(init_seed, i, col0 + s * width + j);
          }
        });
      for (auto& th : pool) th.join();
    }
    const auto t1 = std::chrono::steady_clock::now();
    std::vector<double> sums(slices, 0.0);
    std::atomic<int> err{0};
    {
      std::vector<std::thread> pool;
      for (std::uint32_t t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
          for (std::uint64_t s = t; s < slices; s += threads) {
            try {
              const auto r = protocols::run_moshpit(GridConfig{M, d, 1}, inits[s],
                                                    FailureModel{p, {}}, Rng(seed), rounds);
              sums[s] = r.distortion.empty() ? r.initial_distortion : r.distortion.back();
            } catch (...) {
              err = 1;
            }
          }
        });
      for (auto& th : pool) th.join();
    }
    const auto t2 = std::chrono::steady_clock::now();
    if (err) throw std::invalid_argument("run_moshpit failed");
    *init_s = std::chrono::duration<double>(t1 - t0).count();
    *run_s = std::chrono::duration<double>(t2 - t1).count();
    double c = 0.0;
    for (double x : sums) c += x;
    *checksum = c;
  });
}

}  // extern "C"
