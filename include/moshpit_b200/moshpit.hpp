// moshpit_b200/moshpit.hpp -- drop-in C++ face of the B200 Moshpit engine.
//
// Re-exposes the reference's public hot-path API (proj/include/moshpit/*.hpp)
// under the SAME namespaces, type names, signatures, defaults and exception
// types, implemented over the C ABI (include/moshpit_b200.h) so that the data
// plane runs on sm_100a kernels.  A reference user swaps
//     #include "moshpit/moshpit.hpp"      ->   #include "moshpit_b200/moshpit.hpp"
// and links -lmoshpit_b200.  See INTEGRATION.md.
//
// Covered (reference file:line):
//   core.hpp:14-144        ParamVector, GridConfig, GroupKey, FailureModel,
//                          pairwise_sum, group_mean, distortion, mean_of
//   rng.hpp:31-127         RngStream, Rng (bit-identical sequences)
//   matchmaking.hpp:20-90  Priority, MatchPeer, SealedGroup, initial_index,
//                          next_group_key; :300-323 form_groups_uncontested
//   allreduce.hpp:15-121   PartitionWeights, chunk_sizes, AllReduceOutcome,
//                          butterfly_allreduce
//   theory.hpp:149-155     complexity_estimate
//   protocols.hpp:49-179   TrialReport, run_moshpit
//   optimizer.hpp:19-242   Objective, Quadratic, OptimizerConfig, MembershipEvent,
//                          AssumptionDiagnostics, SgdResult, local_step
//   optimizer.hpp:249-284  detail::moshpit_average
//   optimizer.hpp:297-439  run_moshpit_sgd (Quadratic objective)
#pragma once

#include <cmath>
#include <compare>
#include <cstdint>
#include <cstring>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../moshpit_b200.h"

// The top-level namespace is `moshpit`, as in the reference.  A translation
// unit that also includes the reference headers (e.g. a harness that keeps the
// comparison protocols on the CPU) defines MOSHPIT_B200_NS to another name
// before including this header; see INTEGRATION.md.
#ifndef MOSHPIT_B200_NS
#define MOSHPIT_B200_NS moshpit
#endif

namespace MOSHPIT_B200_NS {

using ParamVector = std::vector<double>;
using PeerId = std::uint32_t;
using LogicalTime = std::uint64_t;

namespace b200 {
// Status -> the reference's exception type.
inline void check(int rc) {
  if (rc == MOSHPIT_OK) return;
  const std::string msg = moshpit_last_error();
  switch (rc) {
    case MOSHPIT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case MOSHPIT_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

inline std::vector<double> flatten(const std::vector<ParamVector>& rows, std::size_t dim,
                                   const char* who) {
  std::vector<double> flat(rows.size() * dim);
  for (std::size_t i = 0; i < rows.size(); ++i) {
    if (rows[i].size() != dim)
      throw std::invalid_argument(std::string(who) + ": dimension mismatch");
    if (dim) std::memcpy(flat.data() + i * dim, rows[i].data(), dim * sizeof(double));
  }
  return flat;
}

inline std::vector<ParamVector> unflatten(const std::vector<double>& flat, std::size_t n,
                                          std::size_t dim) {
  std::vector<ParamVector> rows(n, ParamVector(dim));
  for (std::size_t i = 0; i < n; ++i)
    if (dim) std::memcpy(rows[i].data(), flat.data() + i * dim, dim * sizeof(double));
  return rows;
}
}  // namespace b200

// ---- core.hpp:19-66 --------------------------------------------------------
struct GridConfig {
  std::uint32_t peers_per_axis = 1;  // M
  std::uint32_t dims = 1;            // d
  std::uint32_t rounds = 1;          // T

  void validate() const { b200::check(moshpit_grid_validate(peers_per_axis, dims, rounds)); }
  std::uint64_t capacity() const { return moshpit_grid_capacity(peers_per_axis, dims); }
};

struct GroupKey {
  std::vector<std::uint32_t> indices;
  friend bool operator==(const GroupKey&, const GroupKey&) = default;
  friend auto operator<=>(const GroupKey&, const GroupKey&) = default;
};

struct FailureModel {
  double p_round = 0.0;
  std::vector<std::pair<std::uint32_t, std::int32_t>> churn;

  void validate() const {
    if (p_round < 0.0 || p_round > 1.0)
      throw std::invalid_argument("FailureModel: p_round must be in [0,1]");
  }
};

// ---- rng.hpp:31-127 ----------------------------------------------------------
class RngStream {
 public:
  using result_type = std::uint64_t;
  // rng.hpp:35-38: the stream seeded directly (splitmix64 words of `seed`)
  explicit RngStream(std::uint64_t seed) : st_{} {
    b200::check(moshpit_rng_seeded(seed, &st_));
  }
  explicit RngStream(const moshpit_rng_state& st) : st_(st) {}
  static constexpr result_type min() { return 0; }
  static constexpr result_type max() { return ~std::uint64_t{0}; }

  result_type operator()() { return draw<std::uint64_t>(0); }
  double uniform() { return draw<double>(1); }
  std::uint64_t below(std::uint64_t n) { return draw<std::uint64_t>(2, n); }
  double normal() { return draw<double>(3); }
  std::vector<double> normals(std::size_t n) {
    std::vector<double> out(n);
    if (n) b200::check(moshpit_rng_draws(&st_, 3, 0, 0.0, n, out.data()));
    return out;
  }
  bool bernoulli(double p) { return draw<std::uint8_t>(4, 0, p) != 0; }
  template <typename T>
  void shuffle(std::vector<T>& v) {
    for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[below(i)]);
  }
  moshpit_rng_state& state() { return st_; }

 private:
  template <typename T>
  T draw(int kind, std::uint64_t arg = 0, double p = 0.0) {
    T out{};
    b200::check(moshpit_rng_draws(&st_, kind, arg, p, 1, &out));
    return out;
  }
  moshpit_rng_state st_;
};

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : seed_(seed) {}
  std::uint64_t seed() const { return seed_; }
  RngStream stream(std::string_view name) const { return make(name, -1); }
  RngStream stream(std::string_view name, std::uint64_t index) const {
    return make(name, static_cast<std::int64_t>(index));
  }

 private:
  RngStream make(std::string_view name, std::int64_t index) const {
    moshpit_rng_state st{};
    const std::string n(name);
    b200::check(moshpit_rng_stream(seed_, n.c_str(), index, &st));
    return RngStream(st);
  }
  std::uint64_t seed_;
};

// ---- core.hpp:68-144 ---------------------------------------------------------
namespace detail {
// Host utility (core.hpp:72-81); the GPU kernels evaluate the same tree.
inline double pairwise_sum(std::span<const double> xs) {
  const std::size_t n = xs.size();
  if (n <= 8) {
    double s = 0.0;
    for (double x : xs) s += x;
    return s;
  }
  const std::size_t half = n / 2;
  return pairwise_sum(xs.first(half)) + pairwise_sum(xs.subspan(half));
}
}  // namespace detail

inline double pairwise_sum(const std::vector<double>& xs) {
  return detail::pairwise_sum(std::span<const double>(xs));
}

// GPU: pairwise tree over members in order, / n (core.hpp:91-106).
inline ParamVector group_mean(const std::vector<const ParamVector*>& members) {
  if (members.empty()) throw std::invalid_argument("group_mean: empty group");
  const std::size_t dim = members.front()->size();
  std::vector<double> flat(members.size() * dim);
  for (std::size_t i = 0; i < members.size(); ++i) {
    if (members[i]->size() != dim) throw std::invalid_argument("group_mean: dimension mismatch");
    if (dim) std::memcpy(flat.data() + i * dim, members[i]->data(), dim * sizeof(double));
  }
  ParamVector mean(dim);
  b200::check(moshpit_group_mean(MOSHPIT_F64, flat.data(), members.size(), dim, nullptr,
                                 members.size(), mean.data()));
  return mean;
}

// GPU, reference summation order (core.hpp:111-126).
inline double distortion(const std::vector<ParamVector>& peers,
                         const ParamVector& reference_mean) {
  if (peers.empty()) return 0.0;
  const auto flat = b200::flatten(peers, reference_mean.size(), "distortion");
  double out = 0.0;
  b200::check(moshpit_distortion(MOSHPIT_F64, flat.data(), peers.size(), reference_mean.size(),
                                 reference_mean.data(), &out));
  return out;
}

inline ParamVector mean_of(const std::vector<ParamVector>& peers) {
  if (peers.empty()) throw std::invalid_argument("group_mean: empty group");
  const auto flat = b200::flatten(peers, peers.front().size(), "group_mean");
  ParamVector mean(peers.front().size());
  b200::check(moshpit_mean_of(MOSHPIT_F64, flat.data(), peers.size(), mean.size(), mean.data()));
  return mean;
}

inline bool all_finite(const ParamVector& v) {
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

inline std::vector<double> seeded_standard_normal(RngStream& stream, std::size_t n) {
  return stream.normals(n);
}

// ---- matchmaking.hpp ----------------------------------------------------------
namespace matchmaking {

struct Priority {
  LogicalTime timestamp = 0;
  PeerId peer = 0;
  friend auto operator<=>(const Priority&, const Priority&) = default;
};

inline GroupKey initial_index(std::uint64_t peer_cell, const GridConfig& grid) {
  grid.validate();
  GroupKey key;
  key.indices.resize(grid.dims - 1);
  std::uint32_t scratch[1];
  b200::check(moshpit_initial_index(peer_cell, grid.peers_per_axis, grid.dims,
                                    grid.dims > 1 ? key.indices.data() : scratch));
  return key;
}

inline GroupKey next_group_key(const GroupKey& prev, std::uint32_t new_chunk,
                               const GridConfig& grid) {
  GroupKey key;
  key.indices.resize(prev.indices.size());
  b200::check(moshpit_next_group_key(prev.indices.data(),
                                     static_cast<std::uint32_t>(prev.indices.size()), new_chunk,
                                     grid.peers_per_axis, key.indices.data()));
  return key;
}

struct MatchPeer {
  PeerId id = 0;
  GroupKey key;
  LogicalTime timestamp = 0;
  LogicalTime arrival = 0;
};

struct SealedGroup {
  PeerId leader = 0;
  std::vector<PeerId> members;  // ordered by priority; rank = chunk index
};

// GPU kernel 1 (matchmaking.hpp:300-323).
inline std::vector<SealedGroup> form_groups_uncontested(
    const std::vector<MatchPeer>& peers,
    std::uint32_t max_group_size = std::numeric_limits<std::uint32_t>::max()) {
  const std::size_t n = peers.size();
  std::vector<SealedGroup> groups;
  if (n == 0) return groups;
  const std::size_t klen = peers.front().key.indices.size();
  std::vector<std::uint32_t> ids(n), keys(n * klen + 1), members(n), off(n + 1);
  std::vector<std::uint64_t> ts(n);
  for (std::size_t i = 0; i < n; ++i) {
    if (peers[i].key.indices.size() != klen)
      throw std::invalid_argument("form_groups_uncontested: keys of different lengths");
    ids[i] = peers[i].id;
    ts[i] = peers[i].timestamp;
    for (std::size_t k = 0; k < klen; ++k) keys[i * klen + k] = peers[i].key.indices[k];
  }
  std::uint64_t ng = 0;
  b200::check(moshpit_form_groups_uncontested(n, ids.data(), keys.data(),
                                              static_cast<std::uint32_t>(klen), ts.data(),
                                              max_group_size, members.data(), off.data(), &ng));
  groups.resize(ng);
  for (std::uint64_t g = 0; g < ng; ++g) {
    groups[g].members.assign(members.begin() + off[g], members.begin() + off[g + 1]);
    groups[g].leader = groups[g].members.front();
  }
  return groups;
}

}  // namespace matchmaking

// ---- allreduce.hpp:15-121 -----------------------------------------------------
namespace allreduce {

struct PartitionWeights {
  std::vector<double> w;
  void validate() const {
    double total = 0.0;
    for (double wi : w) {
      if (wi < 0.0) throw std::invalid_argument("PartitionWeights: w >= 0");
      total += wi;
    }
    if (std::abs(total - 1.0) > 1e-9)
      throw std::invalid_argument("PartitionWeights: weights must sum to 1");
  }
  static PartitionWeights uniform(std::size_t n) {
    return PartitionWeights{std::vector<double>(n, 1.0 / n)};
  }
};

inline std::vector<std::size_t> chunk_sizes(std::size_t dim, const PartitionWeights& weights) {
  std::vector<std::uint64_t> s(weights.w.size());
  b200::check(moshpit_chunk_sizes(dim, weights.w.data(), weights.w.size(), s.data()));
  return std::vector<std::size_t>(s.begin(), s.end());
}

struct AllReduceOutcome {
  bool completed = false;
  std::vector<ParamVector> vectors;
  std::vector<std::uint32_t> chunks;
};

// GPU kernel 2 on one group (allreduce.hpp:79-121).
inline AllReduceOutcome butterfly_allreduce(const std::vector<ParamVector>& inputs,
                                            const PartitionWeights& weights,
                                            const std::vector<bool>& failed = {}) {
  const std::size_t n = inputs.size();
  if (n == 0) throw std::invalid_argument("butterfly_allreduce: empty group");
  if (weights.w.size() != n)
    throw std::invalid_argument("butterfly_allreduce: one weight per member");
  const std::size_t dim = inputs.front().size();
  const auto flat = b200::flatten(inputs, dim, "butterfly_allreduce");
  std::vector<std::uint8_t> f(failed.begin(), failed.end());
  std::vector<double> out(n * dim);
  AllReduceOutcome o;
  o.chunks.resize(n);
  std::int32_t done = 0;
  b200::check(moshpit_butterfly_allreduce(MOSHPIT_F64, flat.data(), n, dim, weights.w.data(),
                                          weights.w.size(), f.empty() ? nullptr : f.data(),
                                          out.data(), o.chunks.data(), &done));
  o.completed = done != 0;
  o.vectors = b200::unflatten(out, n, dim);
  return o;
}

// Extension: one whole round of butterfly_allreduce over
// an externally formed group table -- e.g. the SealedGroups of the
// reference's contested matchmaking::form_groups, which stays on the CPU --
// in one GPU launch.  vectors[m] for every member m of groups[g] becomes the
// group's mean unless group_failed[g] (then the group keeps its inputs, as
// butterfly_allreduce with a failed member does).  Equal, bit for bit, to
// calling butterfly_allreduce per group with uniform weights.
inline void butterfly_round(std::vector<ParamVector>& vectors,
                            const std::vector<matchmaking::SealedGroup>& groups,
                            const std::vector<bool>& group_failed = {}) {
  if (vectors.empty() || groups.empty()) return;
  const std::size_t n = vectors.size(), dim = vectors.front().size();
  std::vector<std::uint32_t> members, off{0};
  std::vector<std::uint8_t> vf(groups.size(), 0);
  for (std::size_t g = 0; g < groups.size(); ++g) {
    for (PeerId m : groups[g].members) members.push_back(m);
    off.push_back(static_cast<std::uint32_t>(members.size()));
    if (g < group_failed.size()) vf[g] = group_failed[g] ? 1 : 0;
  }
  auto flat = b200::flatten(vectors, dim, "butterfly_allreduce");
  b200::check(moshpit_round_from_groups_host(MOSHPIT_F64, flat.data(), n, dim, members.data(),
                                             off.data(), groups.size(), vf.data()));
  vectors = b200::unflatten(flat, n, dim);
}

}  // namespace allreduce

namespace theory {
inline double complexity_estimate(std::uint32_t t_rounds, std::uint32_t n_peers, std::uint32_t m,
                                  std::uint32_t dim) {
  return moshpit_complexity_estimate(t_rounds, n_peers, m, dim);
}
}  // namespace theory

// ---- protocols.hpp:49-179 -----------------------------------------------------
namespace protocols {

struct TrialReport {
  double initial_distortion = 0.0;
  std::vector<double> distortion;
  std::vector<double> mean_drift;
  std::vector<std::uint32_t> active_counts;
  double cost_units = 0.0;

  std::uint32_t rounds_to(double threshold, std::uint32_t cap) const {
    if (initial_distortion <= threshold) return 0;
    for (std::size_t t = 0; t < distortion.size() && t < cap; ++t)
      if (distortion[t] <= threshold) return static_cast<std::uint32_t>(t + 1);
    return cap;
  }
};

// GPU, fp64, reference summation order for the diagnostics: the TrialReport
// is bit-identical to the reference's (tests/test_cpp_dropin.py).
inline TrialReport run_moshpit(const GridConfig& grid, const std::vector<ParamVector>& initial,
                               const FailureModel& failure, const Rng& rng,
                               std::uint32_t rounds) {
  grid.validate();
  failure.validate();
  if (initial.empty()) throw std::invalid_argument("run_moshpit: no peers");
  const std::size_t n = initial.size(), dim = initial.front().size();
  // row pointers straight into the caller's vectors: the library packs them
  // into pinned staging slab by slab (no flattened copy of the state)
  std::vector<const void*> rows(n);
  for (std::size_t i = 0; i < n; ++i) {
    if (initial[i].size() != dim) throw std::invalid_argument("group_mean: dimension mismatch");
    rows[i] = initial[i].data();
  }
  TrialReport r;
  r.distortion.resize(rounds);
  r.mean_drift.resize(rounds);
  r.active_counts.resize(rounds);
  b200::check(moshpit_run_moshpit_rows(MOSHPIT_F64, grid.peers_per_axis, grid.dims, grid.rounds,
                                       rows.data(), n, dim, failure.p_round, rng.seed(), rounds,
                                       MOSHPIT_DIAG_EXACT, &r.initial_distortion,
                                       r.distortion.data(), r.mean_drift.data(),
                                       r.active_counts.data(), &r.cost_units));
  return r;
}

}  // namespace protocols

// ---- optimizer.hpp:19-242, 297-439 ---------------------------------------------
namespace optimizer {

class Objective {
 public:
  virtual ~Objective() = default;
  virtual double value(const ParamVector& theta) const = 0;
  virtual ParamVector gradient(const ParamVector& theta) const = 0;
  virtual std::size_t dim() const = 0;
  virtual double smoothness() const = 0;
  virtual double strong_convexity() const = 0;
  virtual double optimum_value() const { return 0.0; }
};

// optimizer.hpp:31-72.  value()/gradient() are the objective's own host
// utilities; the optimizer loop (local_step, run_moshpit_sgd) runs on the GPU.
class Quadratic final : public Objective {
 public:
  Quadratic(std::size_t dim, double l, double mu, ParamVector target)
      : target_(std::move(target)), l_(l), mu_(mu) {
    if (l < mu || mu < 0.0) throw std::invalid_argument("Quadratic: need L >= mu >= 0");
    if (target_.size() != dim) throw std::invalid_argument("Quadratic: target dimension mismatch");
    curvature_.resize(dim);
    for (std::size_t j = 0; j < dim; ++j) {
      const double t = dim > 1 ? static_cast<double>(j) / (dim - 1) : 0.0;
      curvature_[j] = mu + (l - mu) * t;
    }
    if (dim == 1) curvature_[0] = l;
  }
  double value(const ParamVector& theta) const override {
    double f = 0.0;
    for (std::size_t j = 0; j < theta.size(); ++j) {
      const double d = theta[j] - target_[j];
      f += 0.5 * curvature_[j] * d * d;
    }
    return f;
  }
  ParamVector gradient(const ParamVector& theta) const override {
    ParamVector g(theta.size());
    for (std::size_t j = 0; j < theta.size(); ++j) g[j] = curvature_[j] * (theta[j] - target_[j]);
    return g;
  }
  std::size_t dim() const override { return target_.size(); }
  double smoothness() const override { return l_; }
  double strong_convexity() const override { return mu_; }
  const ParamVector& optimum() const { return target_; }

 private:
  ParamVector target_;
  std::vector<double> curvature_;
  double l_, mu_;
};

// optimizer.hpp:75-146.  value()/gradient() evaluate on the GPU (the
// reference's summation orders; libdevice exp/log1p), smoothness() is the
// constructor's trace bound, synthetic() draws the reference's dataset.
class LogisticRegression final : public Objective {
 public:
  LogisticRegression(std::vector<ParamVector> xs, std::vector<double> ys, double l2)
      : ys_(std::move(ys)), l2_(l2) {
    if (xs.empty() || xs.size() != ys_.size())
      throw std::invalid_argument("LogisticRegression: bad dataset");
    dim_ = xs.front().size();
    flat_.reserve(xs.size() * dim_);
    for (const auto& x : xs) {
      if (x.size() != dim_) throw std::invalid_argument("LogisticRegression: ragged dataset");
      flat_.insert(flat_.end(), x.begin(), x.end());
    }
    b200::check(moshpit_logistic_eval(flat_.data(), ys_.data(), ys_.size(), dim_, l2_, nullptr,
                                      nullptr, nullptr, &l_));
  }
  static LogisticRegression synthetic(std::size_t dim, std::size_t samples, double l2,
                                      RngStream& stream) {
    std::vector<double> flat(samples * dim), ys(samples);
    b200::check(moshpit_logistic_synthetic(dim, samples, &stream.state(), flat.data(), ys.data()));
    std::vector<ParamVector> xs(samples);
    for (std::size_t i = 0; i < samples; ++i)
      xs[i].assign(flat.begin() + i * dim, flat.begin() + (i + 1) * dim);
    return LogisticRegression(std::move(xs), std::move(ys), l2);
  }
  double value(const ParamVector& theta) const override {
    double v = 0.0;
    b200::check(moshpit_logistic_eval(flat_.data(), ys_.data(), ys_.size(), dim_, l2_,
                                      theta.data(), &v, nullptr, nullptr));
    return v;
  }
  ParamVector gradient(const ParamVector& theta) const override {
    ParamVector g(dim_);
    b200::check(moshpit_logistic_eval(flat_.data(), ys_.data(), ys_.size(), dim_, l2_,
                                      theta.data(), nullptr, g.data(), nullptr));
    return g;
  }
  std::size_t dim() const override { return dim_; }
  double smoothness() const override { return l_; }
  double strong_convexity() const override { return l2_; }
  // B200 extension: the row-major samples x dim dataset and labels.
  const std::vector<double>& flat_xs() const { return flat_; }
  const std::vector<double>& ys() const { return ys_; }
  double l2() const { return l2_; }

 private:
  std::vector<double> flat_;
  std::vector<double> ys_;
  std::size_t dim_ = 0;
  double l2_, l_ = 0.0;
};

struct OptimizerConfig {
  double gamma = 0.1;
  std::uint32_t tau = 1;
  std::uint32_t steps = 100;
  GridConfig grid;
  double sigma = 0.0;
  std::uint32_t n_peers = 1;
  std::uint32_t inner_rounds = 0;

  void validate() const {
    if (gamma <= 0.0) throw std::invalid_argument("OptimizerConfig: gamma > 0");
    if (tau < 1) throw std::invalid_argument("OptimizerConfig: tau >= 1");
    if (sigma < 0.0) throw std::invalid_argument("OptimizerConfig: sigma >= 0");
    grid.validate();
    if (n_peers < 1 || n_peers > grid.capacity())
      throw std::invalid_argument("OptimizerConfig: 1 <= N <= M^d");
  }
};

struct MembershipEvent {
  std::uint32_t step = 0;
  std::int32_t delta = 0;
};

struct AssumptionDiagnostics {
  std::vector<double> dispersion;
  double delta_aq_hat = 0.0;
  double sigma_hat = 0.0;
  double delta_pv1_hat = 0.0;
  double delta_pv2_hat = 0.0;
  std::uint32_t n_min = 0;
};

struct SgdResult {
  std::vector<double> f_gap;
  std::vector<double> grad_norm_sq;
  std::vector<double> f_gap_weighted;
  ParamVector final_mean;
  AssumptionDiagnostics diagnostics;
};

namespace b200_detail {
inline const Quadratic& as_quadratic(const Objective& o) {
  const auto* q = dynamic_cast<const Quadratic*>(&o);
  if (!q)
    throw std::invalid_argument(
        "B200 optimizer path: Quadratic and LogisticRegression objectives only");
  return *q;
}
inline double quad_l(const Quadratic& q) { return q.smoothness(); }
inline double quad_mu(const Quadratic& q) { return q.strong_convexity(); }
}  // namespace b200_detail

// GPU, noise from the caller's stream (optimizer.hpp:231-242).
inline void local_step(ParamVector& theta, const Objective& objective, double gamma, double sigma,
                       RngStream& noise) {
  if (const auto* lr = dynamic_cast<const LogisticRegression*>(&objective)) {
    b200::check(moshpit_local_step_logistic(MOSHPIT_F64, theta.data(), theta.size(),
                                            lr->flat_xs().data(), lr->ys().data(),
                                            lr->ys().size(), lr->l2(), gamma, sigma,
                                            &noise.state()));
    return;
  }
  const Quadratic& q = b200_detail::as_quadratic(objective);
  b200::check(moshpit_local_step_quadratic(MOSHPIT_F64, theta.data(), theta.size(), q.smoothness(),
                                           q.strong_convexity(), q.optimum().data(), gamma, sigma,
                                           &noise.state()));
}

// GPU, fp64, the reference's noise stream and diagnostic order: the
// SgdResult is bit-identical to the reference's (tests/test_cpp_dropin.py).
inline SgdResult run_moshpit_sgd(const OptimizerConfig& config, const Objective& objective,
                                 const ParamVector& theta0,
                                 const std::vector<MembershipEvent>& schedule, const Rng& rng) {
  config.validate();
  if (theta0.size() != objective.dim())
    throw std::invalid_argument("run_moshpit_sgd: theta0 dimension mismatch");
  const auto* lr = dynamic_cast<const LogisticRegression*>(&objective);
  const Quadratic* q = lr ? nullptr : &b200_detail::as_quadratic(objective);
  std::vector<std::uint32_t> st;
  std::vector<std::int32_t> dl;
  for (const auto& e : schedule) {
    st.push_back(e.step);
    dl.push_back(e.delta);
  }
  SgdResult r;
  const std::uint32_t K = config.steps;
  r.f_gap.resize(K);
  r.grad_norm_sq.resize(K);
  r.f_gap_weighted.resize(K);
  r.diagnostics.dispersion.resize(K);
  r.final_mean.resize(theta0.size());
  double d6[6] = {0, 0, 0, 0, 0, 0};
  if (lr)
    b200::check(moshpit_run_moshpit_sgd_logistic(
        MOSHPIT_F64, config.grid.peers_per_axis, config.grid.dims, config.grid.rounds,
        config.n_peers, theta0.size(), lr->flat_xs().data(), lr->ys().data(), lr->ys().size(),
        lr->l2(), theta0.data(), config.gamma, config.tau, config.steps, config.sigma,
        config.inner_rounds, rng.seed(), st.empty() ? nullptr : st.data(),
        dl.empty() ? nullptr : dl.data(), st.size(), MOSHPIT_DIAG_EXACT, 0, r.f_gap.data(),
        r.grad_norm_sq.data(), r.f_gap_weighted.data(), r.diagnostics.dispersion.data(),
        r.final_mean.data(), d6, nullptr, nullptr));
  else
    b200::check(moshpit_run_moshpit_sgd_quadratic(
        MOSHPIT_F64, config.grid.peers_per_axis, config.grid.dims, config.grid.rounds,
        config.n_peers, theta0.size(), q->smoothness(), q->strong_convexity(),
        q->optimum().data(), theta0.data(), config.gamma, config.tau, config.steps,
        config.sigma, config.inner_rounds, rng.seed(), st.empty() ? nullptr : st.data(),
        dl.empty() ? nullptr : dl.data(), st.size(), MOSHPIT_DIAG_EXACT, 0, r.f_gap.data(),
        r.grad_norm_sq.data(), r.f_gap_weighted.data(), r.diagnostics.dispersion.data(),
        r.final_mean.data(), d6, nullptr, nullptr));
  r.diagnostics.delta_aq_hat = d6[0];
  r.diagnostics.sigma_hat = d6[1];
  r.diagnostics.delta_pv1_hat = d6[2];
  r.diagnostics.delta_pv2_hat = d6[3];
  r.diagnostics.n_min = static_cast<std::uint32_t>(d6[4]);
  if (K == 0) r.final_mean.clear();
  return r;
}

}  // namespace optimizer

// ---- optimizer.hpp:249-284 ----------------------------------------------------
namespace optimizer::detail {

inline void moshpit_average(std::vector<ParamVector>& thetas, const GridConfig& grid,
                            std::uint32_t rounds, RngStream& stream) {
  const std::size_t n = thetas.size();
  if (n <= 1) return;
  const std::size_t dim = thetas.front().size();
  auto flat = b200::flatten(thetas, dim, "group_mean");
  b200::check(moshpit_moshpit_average(MOSHPIT_F64, flat.data(), n, dim, grid.peers_per_axis,
                                      grid.dims, rounds, &stream.state()));
  thetas = b200::unflatten(flat, n, dim);
}

}  // namespace optimizer::detail

}  // namespace MOSHPIT_B200_NS
