// capi.cu -- the C ABI (include/moshpit_b200.h) over the GPU kernels.
//
// Host responsibilities only: argument validation with the reference's error
// classes, the sequential RNG draws the reference makes (cells, failures,
// priorities: O(n) per round), buffer marshalling and kernel launches.  All
// arithmetic on peer vectors and all group formation run on the device.
#include <algorithm>
#include <cmath>
#include <memory>
#include <mutex>
#include <numeric>
#include <unordered_map>

#include "../../include/moshpit_b200.h"
#include "common.cuh"
#include "plane.cuh"

namespace mb200 {

thread_local std::string g_last_error;

double Xoshiro::normal() {  // rng.hpp:68-83
  if (have_spare) {
    have_spare = false;
    return spare;
  }
  double u, v, r2;
  do {
    u = 2.0 * uniform() - 1.0;
    v = 2.0 * uniform() - 1.0;
    r2 = u * u + v * v;
  } while (r2 >= 1.0 || r2 == 0.0);
  const double f = std::sqrt(-2.0 * std::log(r2) / r2);
  spare = v * f;
  have_spare = true;
  return u * f;
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw CudaError(std::string("no usable CUDA device (") +
                    (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                    "); the Moshpit B200 engine has no CPU fallback");
}

namespace {

Xoshiro from_state(const moshpit_rng_state* st) {
  Xoshiro r;
  std::memcpy(r.s, st->s, sizeof(r.s));
  r.have_spare = st->have_spare != 0;
  r.spare = st->spare;
  return r;
}

void to_state(const Xoshiro& r, moshpit_rng_state* st) {
  std::memcpy(st->s, r.s, sizeof(r.s));
  st->have_spare = r.have_spare ? 1 : 0;
  st->spare = r.spare;
}

}  // namespace

}  // namespace mb200

using namespace mb200;

namespace {
// record_round's second stream (column means -> drift, the critical path
// beside the distortion) at the device's highest stream priority: its CTAs
// go first when both kernels have CTAs pending (C2 round + FAST record 7.08-
// 7.18 -> 6.99 ms; profiles/r02/gpu_prio.sh).  MOSHPIT_DIAG_AUX_PRIORITY=0:
// default priority.
inline int aux_priority() {
  const char* e = std::getenv("MOSHPIT_DIAG_AUX_PRIORITY");
  if (e && std::atoi(e) == 0) return 0;
  int lo = 0, hi = 0;
  MB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  return hi;
}
}  // namespace

struct moshpit_engine {
  std::unique_ptr<Plane> plane;
  Xoshiro fail, clock;
  double p = 0.0;
  int variant = MOSHPIT_KERNEL_AUTO;
  // device-resident record_round (moshpit_engine_set_reference / _record)
  int diag = MOSHPIT_DIAG_NONE;
  std::uint64_t diag_dim = 0;
  DeviceBuffer ref, mean, sq, part, part2, log;  // log: [0] initial, then (dist, drift) pairs
  DeviceBuffer rep, rlist, rcount;               // representatives of the last round
  DeviceBuffer colsum;                          // launch_colmean_exactsum scratch
  RoundTables fused;                             // tables of moshpit_engine_rounds_fused
  std::uint64_t log_cap = 0, log_n = 0;
  std::unique_ptr<StreamHolder> aux;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ~moshpit_engine() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }
};

namespace {

void check_state(int dtype, const void* state, std::uint64_t dim, std::uint64_t ld) {
  const std::size_t es = elem_size(dtype);
  const std::uint64_t vec = 16 / es;
  if (reinterpret_cast<std::uintptr_t>(state) % 16 != 0)
    throw std::invalid_argument("peer state must be 16-byte aligned");
  if ((ld * es) % 16 != 0) throw std::invalid_argument("row stride must be a multiple of 16 bytes");
  if (ld < (dim + vec - 1) / vec * vec)
    throw std::invalid_argument("row stride must cover dim rounded up to 16 bytes");
}

}  // namespace

extern "C" {

const char* moshpit_last_error(void) { return g_last_error.c_str(); }

const char* moshpit_version(void) { return "moshpit-b200 0.1 (sm_100a)"; }

int moshpit_device_count(int* out) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    cudaGetLastError();
    *out = n;
  });
}

// ---------------------------------------------------------------------------
// RNG and key arithmetic (host)
// ---------------------------------------------------------------------------
int moshpit_rng_stream(std::uint64_t root, const char* name, std::int64_t index,
                       moshpit_rng_state* out) {
  return guarded([&] {
    if (!name || !out) throw std::invalid_argument("rng_stream: null argument");
    const Xoshiro r = index < 0 ? Xoshiro::named(root, name)
                                : Xoshiro::named(root, name, static_cast<std::uint64_t>(index));
    to_state(r, out);
  });
}

int moshpit_rng_seeded(std::uint64_t seed, moshpit_rng_state* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("rng_seeded: null argument");
    to_state(Xoshiro(seed), out);
  });
}

int moshpit_rng_draws(moshpit_rng_state* st, int kind, std::uint64_t arg, double p,
                      std::uint64_t n, void* out) {
  return guarded([&] {
    if (!st || (n && !out)) throw std::invalid_argument("rng_draws: null argument");
    if (kind == 2 && arg == 0) throw std::invalid_argument("rng_draws: below(0)");
    Xoshiro r = from_state(st);
    for (std::uint64_t i = 0; i < n; ++i) {
      switch (kind) {
        case 0: static_cast<std::uint64_t*>(out)[i] = r.next(); break;
        case 1: static_cast<double*>(out)[i] = r.uniform(); break;
        case 2: static_cast<std::uint64_t*>(out)[i] = r.below(arg); break;
        case 3: static_cast<double*>(out)[i] = r.normal(); break;
        case 4: static_cast<std::uint8_t*>(out)[i] = r.bernoulli(p) ? 1 : 0; break;
        default: throw std::invalid_argument("rng_draws: unknown kind");
      }
    }
    to_state(r, st);
  });
}

int moshpit_grid_validate(std::uint32_t M, std::uint32_t d, std::uint32_t T) {
  return guarded([&] {
    if (M < 1 || d < 1 || T < 1)
      throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
  });
}

std::uint64_t moshpit_grid_capacity(std::uint32_t M, std::uint32_t d) {
  std::uint64_t cap = 1;  // core.hpp:29-33 (wraps like the reference)
  for (std::uint32_t j = 0; j < d; ++j) cap *= M;
  return cap;
}

int moshpit_initial_index(std::uint64_t cell, std::uint32_t M, std::uint32_t d,
                          std::uint32_t* key_out) {
  return guarded([&] {
    if (M < 1 || d < 1) throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
    if (cell >= moshpit_grid_capacity(M, d))
      throw std::out_of_range("initial_index: cell index outside the grid");
    std::uint64_t rest = cell / M;
    for (std::uint32_t j = 1; j < d; ++j) {
      key_out[j - 1] = static_cast<std::uint32_t>(rest % M);
      rest /= M;
    }
  });
}

int moshpit_next_group_key(const std::uint32_t* key, std::uint32_t klen,
                           std::uint32_t chunk, std::uint32_t M, std::uint32_t* key_out) {
  return guarded([&] {
    if (chunk >= M) throw std::out_of_range("next_group_key: chunk index outside [0, M)");
    if (klen == 0) return;
    std::vector<std::uint32_t> tmp(key + 1, key + klen);
    tmp.push_back(chunk);
    std::copy(tmp.begin(), tmp.end(), key_out);
  });
}

int moshpit_chunk_sizes(std::uint64_t dim, const double* w, std::uint64_t n,
                        std::uint64_t* sizes) {
  return guarded([&] {
    double total = 0.0;
    for (std::uint64_t i = 0; i < n; ++i) {
      if (w[i] < 0.0) throw std::invalid_argument("PartitionWeights: w >= 0");
      total += w[i];
    }
    if (std::abs(total - 1.0) > 1e-9)
      throw std::invalid_argument("PartitionWeights: weights must sum to 1");
    std::vector<std::pair<double, std::uint64_t>> rem(n);
    std::uint64_t assigned = 0;
    for (std::uint64_t i = 0; i < n; ++i) {
      const double exact = w[i] * static_cast<double>(dim);
      sizes[i] = static_cast<std::uint64_t>(std::floor(exact));
      assigned += sizes[i];
      rem[i] = {exact - std::floor(exact), i};
    }
    std::sort(rem.begin(), rem.end(), [](const auto& a, const auto& b) {
      return std::tie(b.first, b.second) < std::tie(a.first, a.second);
    });
    for (std::uint64_t k = 0; assigned < dim; ++k, ++assigned) sizes[rem[k % n].second] += 1;
  });
}

double moshpit_complexity_estimate(std::uint32_t t, std::uint32_t n, std::uint32_t m,
                                   std::uint32_t dim) {
  if (t == 0) return 0.0;
  const double md = m;
  return t * (std::log2(static_cast<double>(n)) + md +
              std::max<double>(dim, md) * (md - 1.0) / md);
}

// ---------------------------------------------------------------------------
// form_groups_uncontested on the GPU (kernel 1, digit-key mode)
// ---------------------------------------------------------------------------
int moshpit_form_groups_uncontested(std::uint64_t n, const std::uint32_t* ids,
                                    const std::uint32_t* keys, std::uint32_t klen,
                                    const std::uint64_t* timestamps, std::uint32_t cap,
                                    std::uint32_t* members_out, std::uint32_t* group_off_out,
                                    std::uint64_t* n_groups_out) {
  return guarded([&] {
    if (cap == 0) throw std::invalid_argument("form_groups_uncontested: cap >= 1");
    if (n > 0x7fffffffull) throw std::invalid_argument("form_groups_uncontested: n too large");
    if (n == 0) {
      group_off_out[0] = 0;
      *n_groups_out = 0;
      return;
    }
    require_device();
    StreamHolder st;
    std::uint64_t np = 1;
    while (np < n) np <<= 1;
    DeviceBuffer d_ids(n * 4), d_keys(n * (klen ? klen : 1) * 4), d_ts(n * 8), d_mem(n * 4),
        d_goff((n + 1) * 4), d_void(n), d_counts(16), d_sidx(np * 4), d_scs(n * 4), d_sgi(n * 4);
    MB_CUDA(cudaMemcpyAsync(d_ids.ptr, ids, n * 4, cudaMemcpyHostToDevice, st.s));
    if (klen)
      MB_CUDA(cudaMemcpyAsync(d_keys.ptr, keys, n * klen * 4, cudaMemcpyHostToDevice, st.s));
    MB_CUDA(cudaMemcpyAsync(d_ts.ptr, timestamps, n * 8, cudaMemcpyHostToDevice, st.s));
    GroupArgs a;
    a.n = static_cast<std::uint32_t>(n);
    a.cap = cap;
    a.digit_keys = d_keys.as<std::uint32_t>();
    a.dklen = klen;
    a.ts = d_ts.as<std::uint64_t>();
    a.ids = d_ids.as<std::uint32_t>();
    a.members = d_mem.as<std::uint32_t>();
    a.goff = d_goff.as<std::uint32_t>();
    a.gvoid = d_void.as<std::uint8_t>();
    a.counts = d_counts.as<std::uint32_t>();
    a.sidx = d_sidx.as<std::uint32_t>();
    a.scs = d_scs.as<std::uint32_t>();
    a.sgi = d_sgi.as<std::uint32_t>();
    launch_form_groups(a, false, st.s);
    std::uint32_t counts[4];
    MB_CUDA(cudaMemcpyAsync(counts, d_counts.ptr, 16, cudaMemcpyDeviceToHost, st.s));
    MB_CUDA(cudaMemcpyAsync(members_out, d_mem.ptr, n * 4, cudaMemcpyDeviceToHost, st.s));
    MB_CUDA(cudaStreamSynchronize(st.s));
    MB_CUDA(cudaMemcpy(group_off_out, d_goff.ptr, (counts[0] + 1) * 4, cudaMemcpyDeviceToHost));
    *n_groups_out = counts[0];
  });
}

// ---------------------------------------------------------------------------
// numerics on host buffers
// ---------------------------------------------------------------------------
int moshpit_group_mean(int dtype, const void* rows, std::uint64_t n_rows, std::uint64_t dim,
                       const std::uint32_t* members, std::uint64_t n, void* mean_out) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    if (n == 0) throw std::invalid_argument("group_mean: empty group");
    if (members)
      for (std::uint64_t k = 0; k < n; ++k)
        if (members[k] >= n_rows) throw std::out_of_range("group_mean: member outside rows");
    if (!members && n > n_rows) throw std::out_of_range("group_mean: n exceeds rows");
    if (dim == 0) return;
    require_device();
    StreamHolder st;
    DeviceBuffer d_rows(n_rows * dim * es), d_mem(n * 4), d_out(dim * es);
    MB_CUDA(cudaMemcpyAsync(d_rows.ptr, rows, n_rows * dim * es, cudaMemcpyHostToDevice, st.s));
    if (members)
      MB_CUDA(cudaMemcpyAsync(d_mem.ptr, members, n * 4, cudaMemcpyHostToDevice, st.s));
    const std::uint32_t* m = members ? d_mem.as<std::uint32_t>() : nullptr;
    if (dtype == MOSHPIT_F32)
      launch_colmean<float, float>(d_rows.as<float>(), n, dim, dim, m, d_out.as<float>(), st.s);
    else
      launch_colmean<double, double>(d_rows.as<double>(), n, dim, dim, m, d_out.as<double>(),
                                     st.s);
    MB_CUDA(cudaMemcpyAsync(mean_out, d_out.ptr, dim * es, cudaMemcpyDeviceToHost, st.s));
    MB_CUDA(cudaStreamSynchronize(st.s));
  });
}

int moshpit_butterfly_allreduce(int dtype, const void* inputs, std::uint64_t n,
                                std::uint64_t dim, const double* weights,
                                std::uint64_t n_weights, const std::uint8_t* failed,
                                void* vectors_out, std::uint32_t* chunks_out,
                                std::int32_t* completed_out) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    // allreduce.hpp:82-89 validation order
    if (n == 0) throw std::invalid_argument("butterfly_allreduce: empty group");
    if (n_weights != n) throw std::invalid_argument("butterfly_allreduce: one weight per member");
    // chunk_sizes validates the weights (allreduce.hpp:48) on the success path
    for (std::uint64_t k = 0; k < n; ++k) chunks_out[k] = static_cast<std::uint32_t>(k);
    bool any = false;
    if (failed)
      for (std::uint64_t k = 0; k < n; ++k) any |= failed[k] != 0;
    if (any) {  // allreduce.hpp:95-102: the round is void, outputs = inputs
      std::memcpy(vectors_out, inputs, n * dim * es);
      *completed_out = 0;
      return;
    }
    std::vector<std::uint64_t> sizes(n);
    if (moshpit_chunk_sizes(dim, weights, n, sizes.data()) != MOSHPIT_OK)
      throw std::invalid_argument(g_last_error);
    *completed_out = 1;
    if (dim == 0) return;
    if (n > 0x7fffffffull) throw std::invalid_argument("butterfly_allreduce: group too large");
    require_device();
    StreamHolder st;
    const std::uint64_t ld = padded_ld(dim, es);
    DeviceBuffer d_x(n * ld * es), d_tab((n + 1) * 4 + n * 4 + 64);
    MB_CUDA(cudaMemcpy2DAsync(d_x.ptr, ld * es, inputs, dim * es, dim * es, n,
                              cudaMemcpyHostToDevice, st.s));
    // a single group {0..n-1}, active: kernel 2 averages it in place
    std::vector<std::uint32_t> tab((n + 1) + n + 16, 0);
    std::uint32_t* h_mem = tab.data();
    std::uint32_t* h_goff = h_mem + n;
    std::iota(h_mem, h_mem + n, 0u);
    h_goff[0] = 0;
    h_goff[1] = static_cast<std::uint32_t>(n);
    std::uint32_t* h_act = h_goff + 2;
    h_act[0] = 0;
    std::uint32_t* h_counts = h_act + 1;
    h_counts[0] = 1;
    h_counts[1] = 1;
    h_counts[2] = static_cast<std::uint32_t>(n);
    MB_CUDA(cudaMemcpyAsync(d_tab.ptr, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, st.s));
    const std::uint32_t* dm = d_tab.as<std::uint32_t>();
    if (dtype == MOSHPIT_F32)
      launch_group_mean<float>(d_x.as<float>(), ld, dim, dm, dm + n, dm + n + 2, dm + n + 3,
                               static_cast<std::uint32_t>(n), 0, st.s);
    else
      launch_group_mean<double>(d_x.as<double>(), ld, dim, dm, dm + n, dm + n + 2, dm + n + 3,
                                static_cast<std::uint32_t>(n), 0, st.s);
    MB_CUDA(cudaMemcpy2DAsync(vectors_out, dim * es, d_x.ptr, ld * es, dim * es, n,
                              cudaMemcpyDeviceToHost, st.s));
    MB_CUDA(cudaStreamSynchronize(st.s));
  });
}

int moshpit_distortion(int dtype, const void* peers, std::uint64_t n, std::uint64_t dim,
                       const double* ref, double* out) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    if (n == 0) {  // core.hpp:113
      *out = 0.0;
      return;
    }
    require_device();
    StreamHolder st;
    DeviceBuffer d_x(n * dim * es + 16), d_ref(dim * 8 + 16), d_sq(n * 8), d_out(16);
    MB_CUDA(cudaMemcpyAsync(d_x.ptr, peers, n * dim * es, cudaMemcpyHostToDevice, st.s));
    MB_CUDA(cudaMemcpyAsync(d_ref.ptr, ref, dim * 8, cudaMemcpyHostToDevice, st.s));
    if (dtype == MOSHPIT_F32)
      launch_distortion<float>(d_x.as<float>(), n, dim, dim, d_ref.as<double>(),
                               d_sq.as<double>(), nullptr, d_out.as<double>(), 1, st.s);
    else
      launch_distortion<double>(d_x.as<double>(), n, dim, dim, d_ref.as<double>(),
                                d_sq.as<double>(), nullptr, d_out.as<double>(), 1, st.s);
    MB_CUDA(cudaMemcpyAsync(out, d_out.ptr, 8, cudaMemcpyDeviceToHost, st.s));
    MB_CUDA(cudaStreamSynchronize(st.s));
  });
}

int moshpit_mean_of(int dtype, const void* peers, std::uint64_t n, std::uint64_t dim,
                    void* mean_out) {
  return moshpit_group_mean(dtype, peers, n, dim, nullptr, n, mean_out);
}

// ---------------------------------------------------------------------------
// run_moshpit (protocols.hpp:108-179) with host buffers
// ---------------------------------------------------------------------------
int moshpit_run_moshpit(int dtype, std::uint32_t M, std::uint32_t d, std::uint32_t T,
                        const void* initial, std::uint64_t n, std::uint64_t dim,
                        double p_round, std::uint64_t seed, std::uint32_t rounds, int diag,
                        double* initial_distortion, double* distortion, double* mean_drift,
                        std::uint32_t* active_counts, double* cost_units, void* final_out) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    // protocols.hpp:112-117, in order
    if (M < 1 || d < 1 || T < 1)
      throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
    if (p_round < 0.0 || p_round > 1.0)
      throw std::invalid_argument("FailureModel: p_round must be in [0,1]");
    if (n == 0) throw std::invalid_argument("run_moshpit: no peers");
    if (n > moshpit_grid_capacity(M, d))
      throw std::invalid_argument("run_moshpit: N exceeds grid capacity M^d");
    if (diag < MOSHPIT_DIAG_NONE || diag > MOSHPIT_DIAG_EXACT)
      throw std::invalid_argument("run_moshpit: unknown diagnostics mode");
    require_device();
    int dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    // Large states stream through the GPU in D-slabs (stream_run.cu): H2D,
    // rounds and D2H overlap; results are identical to the resident path.
    const std::uint64_t W = stream_slab_cols(n, es, dim);
    if (dim > W) {
      HostRows src;
      src.base = initial;
      src.pitch_bytes = dim * es;
      if (dtype == MOSHPIT_F32)
        run_moshpit_streamed<float>(M, d, src, n, dim, p_round, seed, rounds, diag,
                                    initial_distortion, distortion, mean_drift, active_counts,
                                    static_cast<float*>(final_out), W);
      else
        run_moshpit_streamed<double>(M, d, src, n, dim, p_round, seed, rounds, diag,
                                     initial_distortion, distortion, mean_drift, active_counts,
                                     static_cast<double*>(final_out), W);
      *cost_units = moshpit_complexity_estimate(rounds, static_cast<std::uint32_t>(n), M,
                                                static_cast<std::uint32_t>(dim));
      return;
    }
    StreamHolder st, aux(aux_priority());
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    MB_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    MB_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    struct EvG {
      cudaEvent_t a, b;
      ~EvG() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
    } evg{ev_fork, ev_join};
    const std::uint64_t ld = padded_ld(dim, es);
    DeviceBuffer d_x(n * ld * es), d_ref(dim * 8 + 16), d_mean(dim * 8 + 16), d_sq(n * 8),
        d_part(diag_partial_elems(n, dim) * 8 + 16), d_part2(diag_partial_elems(n, dim) * 8 + 16),
        d_out((2 * rounds + 2) * 8);
    MB_CUDA(cudaMemcpy2DAsync(d_x.ptr, ld * es, initial, dim * es, dim * es, n,
                              cudaMemcpyHostToDevice, st.s));
    const int exact = diag == MOSHPIT_DIAG_EXACT;
    // record_round: the distortion (st; EXACT j-chains or FAST chunk
    // partials) and colmean + drift (aux) only read the state, so they run
    // side by side; the next round waits for both.
    // after a round, the rows of each averaged group are identical: the
    // per-row diagnostics read one representative row per such group
    // (RepRows; bit-identical results, fewer HBM bytes)
    DeviceBuffer d_rep(n * 4 + 16), d_rlist(n * 4 + 16), d_rcount(16);
    const RepRows reps{d_rep.as<std::uint32_t>(), d_rlist.as<std::uint32_t>(),
                       d_rcount.as<std::uint32_t>()};
    auto record = [&](double* dist_slot, double* drift_slot) {
      const RepRows* rr = drift_slot ? &reps : nullptr;  // the initial record has no round
      const std::uint32_t* rows = rr ? reps.rep : nullptr;
      if (drift_slot) {
        MB_CUDA(cudaEventRecord(ev_fork, st.s));
        MB_CUDA(cudaStreamWaitEvent(aux.s, ev_fork, 0));
      }
      if (dtype == MOSHPIT_F32) {
        launch_distortion<float>(d_x.as<float>(), n, ld, dim, d_ref.as<double>(),
                                 d_sq.as<double>(), d_part.as<double>(), dist_slot, exact, st.s,
                                 rr);
        if (drift_slot)
          launch_colmean<float, double>(d_x.as<float>(), n, ld, dim, rows,
                                        d_mean.as<double>(), aux.s, true);
      } else {
        launch_distortion<double>(d_x.as<double>(), n, ld, dim, d_ref.as<double>(),
                                  d_sq.as<double>(), d_part.as<double>(), dist_slot, exact, st.s,
                                  rr);
        if (drift_slot)
          launch_colmean<double, double>(d_x.as<double>(), n, ld, dim, rows,
                                         d_mean.as<double>(), aux.s, true);
      }
      if (drift_slot) {
        launch_drift(d_mean.as<double>(), d_ref.as<double>(), dim, d_part2.as<double>(),
                     drift_slot, exact, aux.s);
        MB_CUDA(cudaEventRecord(ev_join, aux.s));
        MB_CUDA(cudaStreamWaitEvent(st.s, ev_join, 0));
      }
    };
    double* outp = d_out.as<double>();
    if (diag != MOSHPIT_DIAG_NONE) {
      // reference = mean_of(initial) (protocols.hpp:119), in fp64
      if (dtype == MOSHPIT_F32)
        launch_colmean<float, double>(d_x.as<float>(), n, ld, dim, nullptr, d_ref.as<double>(),
                                      st.s);
      else
        launch_colmean<double, double>(d_x.as<double>(), n, ld, dim, nullptr,
                                       d_ref.as<double>(), st.s);
      record(outp, nullptr);
    }
    Plane plane(M, d, n, dev);
    Xoshiro cells = Xoshiro::named(seed, "cells");
    plane.init_cells(cells, st.s);
    Xoshiro fail = Xoshiro::named(seed, "failures");
    Xoshiro clock = Xoshiro::named(seed, "priorities");
    for (std::uint32_t r = 0; r < rounds; ++r) {
      active_counts[r] = plane.round(&fail, p_round, clock, dtype, d_x.ptr, dim, ld, st.s,
                                     MOSHPIT_KERNEL_AUTO);
      if (diag != MOSHPIT_DIAG_NONE) {
        launch_build_reps(plane.members.as<std::uint32_t>(), plane.goff.as<std::uint32_t>(),
                          plane.gvoid.as<std::uint8_t>(), plane.counts.as<std::uint32_t>(), n,
                          d_rep.as<std::uint32_t>(), d_rlist.as<std::uint32_t>(),
                          d_rcount.as<std::uint32_t>(), st.s);
        record(outp + 2 + r, outp + 2 + rounds + r);
      }
    }
    if (diag != MOSHPIT_DIAG_NONE) {
      std::vector<double> h(2 * rounds + 2);
      MB_CUDA(cudaMemcpyAsync(h.data(), outp, h.size() * 8, cudaMemcpyDeviceToHost, st.s));
      MB_CUDA(cudaStreamSynchronize(st.s));
      *initial_distortion = h[0];
      for (std::uint32_t r = 0; r < rounds; ++r) {
        distortion[r] = h[2 + r];
        mean_drift[r] = h[2 + rounds + r];
      }
    } else {
      *initial_distortion = std::nan("");
      for (std::uint32_t r = 0; r < rounds; ++r) distortion[r] = mean_drift[r] = std::nan("");
    }
    if (final_out)
      MB_CUDA(cudaMemcpy2DAsync(final_out, dim * es, d_x.ptr, ld * es, dim * es, n,
                                cudaMemcpyDeviceToHost, st.s));
    MB_CUDA(cudaStreamSynchronize(st.s));
    *cost_units = moshpit_complexity_estimate(rounds, static_cast<std::uint32_t>(n), M,
                                              static_cast<std::uint32_t>(dim));
  });
}

// run_moshpit over an array of row pointers (the drop-in's
// std::vector<ParamVector>): large states are packed slab by slab from the
// rows into a pinned ring by host threads (no flattened copy of the state);
// small ones are flattened and take the resident path.
int moshpit_run_moshpit_rows(int dtype, std::uint32_t M, std::uint32_t d, std::uint32_t T,
                             const void* const* rows, std::uint64_t n, std::uint64_t dim,
                             double p_round, std::uint64_t seed, std::uint32_t rounds, int diag,
                             double* initial_distortion, double* distortion, double* mean_drift,
                             std::uint32_t* active_counts, double* cost_units) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    if (M < 1 || d < 1 || T < 1)
      throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
    if (p_round < 0.0 || p_round > 1.0)
      throw std::invalid_argument("FailureModel: p_round must be in [0,1]");
    if (n == 0) throw std::invalid_argument("run_moshpit: no peers");
    if (!rows) throw std::invalid_argument("run_moshpit: null rows");
    if (n > moshpit_grid_capacity(M, d))
      throw std::invalid_argument("run_moshpit: N exceeds grid capacity M^d");
    if (diag < MOSHPIT_DIAG_NONE || diag > MOSHPIT_DIAG_EXACT)
      throw std::invalid_argument("run_moshpit: unknown diagnostics mode");
    const std::uint64_t W = stream_slab_cols(n, es, dim);
    if (dim <= W) {
      std::vector<char> flat(n * dim * es + 16);
      for (std::uint64_t i = 0; i < n; ++i)
        if (dim) std::memcpy(flat.data() + i * dim * es, rows[i], dim * es);
      const int rc = moshpit_run_moshpit(dtype, M, d, T, flat.data(), n, dim, p_round, seed,
                                         rounds, diag, initial_distortion, distortion, mean_drift,
                                         active_counts, cost_units, nullptr);
      if (rc != MOSHPIT_OK) {
        const std::string msg = g_last_error;
        if (rc == MOSHPIT_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
        if (rc == MOSHPIT_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
        if (rc == MOSHPIT_ERR_CUDA) throw CudaError(msg);
        throw std::runtime_error(msg);
      }
      return;
    }
    require_device();
    HostRows src;
    src.rows = rows;
    if (dtype == MOSHPIT_F32)
      run_moshpit_streamed<float>(M, d, src, n, dim, p_round, seed, rounds, diag,
                                  initial_distortion, distortion, mean_drift, active_counts,
                                  nullptr, W);
    else
      run_moshpit_streamed<double>(M, d, src, n, dim, p_round, seed, rounds, diag,
                                   initial_distortion, distortion, mean_drift, active_counts,
                                   nullptr, W);
    *cost_units = moshpit_complexity_estimate(rounds, static_cast<std::uint32_t>(n), M,
                                              static_cast<std::uint32_t>(dim));
  });
}

// ---------------------------------------------------------------------------
// one round over an externally formed group table (e.g. the reference's
// contested form_groups, matchmaking.hpp:104-294 / 325-333): kernel 2 over
// the table; voided groups (any member failed, allreduce.hpp:95-102) keep
// their rows.  SURVEY 8f rank 4: the control plane stays on the CPU.
// ---------------------------------------------------------------------------
namespace {

struct GroupTable {
  std::vector<std::uint32_t> tab;  // members | goff | act | counts(4)
  std::uint32_t n_members = 0, n_groups = 0, max_group = 1;
};

GroupTable build_group_table(std::uint64_t n_rows, const std::uint32_t* members,
                             const std::uint32_t* group_off, std::uint64_t n_groups,
                             const std::uint8_t* void_flags) {
  if (n_groups > 0x7fffffffull) throw std::invalid_argument("round_from_groups: too many groups");
  if (n_groups && (!members || !group_off))
    throw std::invalid_argument("round_from_groups: null table");
  GroupTable t;
  t.n_groups = static_cast<std::uint32_t>(n_groups);
  if (n_groups && group_off[0] != 0)
    throw std::invalid_argument("round_from_groups: group_off[0] must be 0");
  const std::uint32_t m = n_groups ? group_off[n_groups] : 0;
  t.n_members = m;
  std::vector<std::uint8_t> seen(n_rows, 0);
  std::uint32_t active = 0, rows = 0;
  for (std::uint64_t g = 0; g < n_groups; ++g) {
    if (group_off[g + 1] < group_off[g])
      throw std::invalid_argument("round_from_groups: group_off must be non-decreasing");
    if (group_off[g + 1] == group_off[g])
      throw std::invalid_argument("butterfly_allreduce: empty group");
    t.max_group = std::max(t.max_group, group_off[g + 1] - group_off[g]);
  }
  for (std::uint32_t k = 0; k < m; ++k) {
    if (members[k] >= n_rows) throw std::out_of_range("round_from_groups: member outside rows");
    if (seen[members[k]]++) throw std::invalid_argument("round_from_groups: a row in two groups");
  }
  t.tab.resize(m + (n_groups + 1) + n_groups + 4 + 4);
  std::copy(members, members + m, t.tab.begin());
  std::copy(group_off, group_off + n_groups + 1, t.tab.begin() + m);
  std::uint32_t* act = t.tab.data() + m + n_groups + 1;
  for (std::uint64_t g = 0; g < n_groups; ++g)
    if (!(void_flags && void_flags[g])) {
      act[active++] = static_cast<std::uint32_t>(g);
      rows += group_off[g + 1] - group_off[g];
    }
  std::uint32_t* cnt = act + n_groups;
  cnt[0] = t.n_groups;
  cnt[1] = active;
  cnt[2] = rows;
  cnt[3] = 0;
  return t;
}

void launch_table_round(int dtype, void* state, std::uint64_t dim, std::uint64_t ld,
                        const GroupTable& t, cudaStream_t s) {
  if (dim == 0 || t.n_groups == 0) return;
  void* d_tab = nullptr;
  MB_CUDA(cudaMallocAsync(&d_tab, t.tab.size() * 4, s));
  MB_CUDA(cudaMemcpyAsync(d_tab, t.tab.data(), t.tab.size() * 4, cudaMemcpyHostToDevice, s));
  const auto* dm = static_cast<const std::uint32_t*>(d_tab);
  const std::uint32_t* goff = dm + t.n_members;
  const std::uint32_t* act = goff + t.n_groups + 1;
  const std::uint32_t* cnt = act + t.n_groups;
  if (dtype == MOSHPIT_F32)
    launch_group_mean<float>(static_cast<float*>(state), ld, dim, dm, goff, act, cnt,
                             t.max_group, 0, s);
  else
    launch_group_mean<double>(static_cast<double*>(state), ld, dim, dm, goff, act, cnt,
                              t.max_group, 0, s);
  MB_CUDA(cudaFreeAsync(d_tab, s));
}

}  // namespace

extern "C" {

int moshpit_round_from_groups(int dtype, void* state, std::uint64_t n_rows, std::uint64_t dim,
                              std::uint64_t ld, const std::uint32_t* members,
                              const std::uint32_t* group_off, std::uint64_t n_groups,
                              const std::uint8_t* void_flags, void* stream) {
  return guarded([&] {
    elem_size(dtype);
    if (state) check_state(dtype, state, dim, ld);
    const GroupTable t = build_group_table(n_rows, members, group_off, n_groups, void_flags);
    require_device();
    launch_table_round(dtype, state, dim, ld, t, static_cast<cudaStream_t>(stream));
  });
}

int moshpit_round_from_groups_host(int dtype, void* vectors, std::uint64_t n_rows,
                                   std::uint64_t dim, const std::uint32_t* members,
                                   const std::uint32_t* group_off, std::uint64_t n_groups,
                                   const std::uint8_t* void_flags) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    const GroupTable t = build_group_table(n_rows, members, group_off, n_groups, void_flags);
    if (dim == 0 || n_rows == 0 || t.n_groups == 0) return;
    require_device();
    StreamHolder st;
    const std::uint64_t ld = padded_ld(dim, es);
    DeviceBuffer d_x(n_rows * ld * es);
    MB_CUDA(cudaMemcpy2DAsync(d_x.ptr, ld * es, vectors, dim * es, dim * es, n_rows,
                              cudaMemcpyHostToDevice, st.s));
    launch_table_round(dtype, d_x.ptr, dim, ld, t, st.s);
    MB_CUDA(cudaMemcpy2DAsync(vectors, dim * es, d_x.ptr, ld * es, dim * es, n_rows,
                              cudaMemcpyDeviceToHost, st.s));
    MB_CUDA(cudaStreamSynchronize(st.s));
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// optimizer::detail::moshpit_average (optimizer.hpp:249-284) with host buffers
// ---------------------------------------------------------------------------
int moshpit_moshpit_average(int dtype, void* thetas, std::uint64_t n, std::uint64_t dim,
                            std::uint32_t M, std::uint32_t d, std::uint32_t rounds,
                            moshpit_rng_state* stream) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    if (n <= 1) return;  // optimizer.hpp:253: no draws at all
    if (M < 1 || d < 1) throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
    require_device();
    int dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    StreamHolder st;
    const std::uint64_t ld = padded_ld(dim, es);
    DeviceBuffer d_x(n * ld * es);
    MB_CUDA(cudaMemcpy2DAsync(d_x.ptr, ld * es, thetas, dim * es, dim * es, n,
                              cudaMemcpyHostToDevice, st.s));
    Xoshiro s = from_state(stream);
    Plane plane(M, d, n, dev);
    plane.init_cells(s, st.s);
    for (std::uint32_t r = 0; r < rounds; ++r)
      plane.round(nullptr, 0.0, s, dtype, d_x.ptr, dim, ld, st.s, MOSHPIT_KERNEL_AUTO);
    MB_CUDA(cudaMemcpy2DAsync(thetas, dim * es, d_x.ptr, ld * es, dim * es, n,
                              cudaMemcpyDeviceToHost, st.s));
    MB_CUDA(cudaStreamSynchronize(st.s));
    to_state(s, stream);
  });
}

// ---------------------------------------------------------------------------
// device-resident engine
// ---------------------------------------------------------------------------
int moshpit_engine_create(std::uint32_t M, std::uint32_t d, std::uint64_t n, double p_round,
                          std::uint64_t seed, int device, moshpit_engine** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("engine_create: null out");
    if (M < 1 || d < 1) throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
    if (p_round < 0.0 || p_round > 1.0)
      throw std::invalid_argument("FailureModel: p_round must be in [0,1]");
    require_device();
    DeviceGuard g(device);
    int dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    auto e = std::make_unique<moshpit_engine>();
    e->plane = std::make_unique<Plane>(M, d, n, dev);
    e->p = p_round;
    Xoshiro cells = Xoshiro::named(seed, "cells");
    e->fail = Xoshiro::named(seed, "failures");
    e->clock = Xoshiro::named(seed, "priorities");
    StreamHolder st;
    e->plane->init_cells(cells, st.s);
    MB_CUDA(cudaStreamSynchronize(st.s));
    *out = e.release();
  });
}

int moshpit_engine_destroy(moshpit_engine* e) {
  return guarded([&] {
    if (!e) return;
    if (e->plane) {
      DeviceGuard g(e->plane->device);
      cudaDeviceSynchronize();
      e->plane.reset();
    }
    delete e;
  });
}

int moshpit_engine_set_kernel(moshpit_engine* e, int variant) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    if (variant < MOSHPIT_KERNEL_AUTO || variant > MOSHPIT_KERNEL_BULK)
      throw std::invalid_argument("unknown kernel variant");
    e->variant = variant;
  });
}

int moshpit_engine_round(moshpit_engine* e, int dtype, void* state, std::uint64_t dim,
                         std::uint64_t ld, void* stream, std::uint32_t* active_out) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    if (state) check_state(dtype, state, dim, ld);
    DeviceGuard g(e->plane->device);
    const std::uint32_t a = e->plane->round(&e->fail, e->p, e->clock, dtype, state, dim, ld,
                                            static_cast<cudaStream_t>(stream), e->variant);
    if (active_out) *active_out = a;
  });
}

// Several rounds in one pass over the state (temporal blocking, a separate
// mode from the per-round path): kernel 1 for each round, then one fused
// kernel per chunk of at most fused_rounds_max(n, M^(d-1)) rounds.  Bit-identical to
// `rounds` calls of moshpit_engine_round.
int moshpit_engine_rounds_fused(moshpit_engine* e, int dtype, void* state, std::uint64_t dim,
                                std::uint64_t ld, std::uint32_t rounds, void* stream,
                                std::uint32_t* active_out) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    if (!state) throw std::invalid_argument("fused rounds: null state");
    check_state(dtype, state, dim, ld);
    Plane& p = *e->plane;
    const auto gcap = (std::uint32_t)std::min<std::uint64_t>(p.grid.lines(), p.n);
    const std::uint32_t cap = fused_rounds_max(p.n, gcap);
    if (cap == 0) throw std::invalid_argument("fused rounds: too many peers for one pass");
    DeviceGuard g(p.device);
    auto s = static_cast<cudaStream_t>(stream);
    for (std::uint32_t done = 0; done < rounds;) {
      const std::uint32_t R = std::min(cap, rounds - done);
      e->fused.form(p, R, &e->fail, e->p, e->clock, s, active_out ? active_out + done : nullptr);
      if (dtype == MOSHPIT_F32)
        launch_rounds_fused<float>(static_cast<float*>(state), ld, dim, (std::uint32_t)p.n, gcap,
                                   e->fused.dev(), R, nullptr, s);
      else
        launch_rounds_fused<double>(static_cast<double*>(state), ld, dim, (std::uint32_t)p.n, gcap,
                                    e->fused.dev(), R, nullptr, s);
      p.mark_done(s);
      done += R;
    }
  });
}

int moshpit_engine_stats(moshpit_engine* e, std::uint64_t* rounds,
                         std::uint64_t* active_rows_total) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    DeviceGuard g(e->plane->device);
    e->plane->sync_done();
    unsigned long long t[2];
    MB_CUDA(cudaMemcpy(t, e->plane->totals.ptr, 16, cudaMemcpyDeviceToHost));
    if (rounds) *rounds = e->plane->rounds_done;
    if (active_rows_total) *active_rows_total = t[0];
  });
}

int moshpit_engine_set_timing(moshpit_engine* e, int enable) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    e->plane->timing = enable != 0;
    e->plane->tev_used = 0;
  });
}

int moshpit_engine_kernel_time(moshpit_engine* e, double* total_ms, std::uint64_t* launches) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    Plane& p = *e->plane;
    DeviceGuard g(p.device);
    double t = 0.0;
    for (std::size_t i = 0; i < p.tev_used; ++i) {
      MB_CUDA(cudaEventSynchronize(p.tev[i].second));
      float ms = 0.f;
      MB_CUDA(cudaEventElapsedTime(&ms, p.tev[i].first, p.tev[i].second));
      t += ms;
    }
    if (total_ms) *total_ms = t;
    if (launches) *launches = p.tev_used;
    p.tev_used = 0;
  });
}

int moshpit_engine_tables(moshpit_engine* e, std::uint32_t* members, std::uint32_t* group_off,
                          std::uint32_t* n_groups, std::uint8_t* void_flags,
                          std::uint32_t* ranks, std::uint32_t* keys) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    Plane& p = *e->plane;
    DeviceGuard g(p.device);
    p.sync_done();
    std::uint32_t counts[4];
    MB_CUDA(cudaMemcpy(counts, p.counts.ptr, 16, cudaMemcpyDeviceToHost));
    if (n_groups) *n_groups = counts[0];
    if (members) MB_CUDA(cudaMemcpy(members, p.members.ptr, p.n * 4, cudaMemcpyDeviceToHost));
    if (group_off)
      MB_CUDA(cudaMemcpy(group_off, p.goff.ptr, (counts[0] + 1) * 4, cudaMemcpyDeviceToHost));
    if (void_flags) MB_CUDA(cudaMemcpy(void_flags, p.gvoid.ptr, counts[0], cudaMemcpyDeviceToHost));
    if (ranks) MB_CUDA(cudaMemcpy(ranks, p.rank.ptr, p.n * 4, cudaMemcpyDeviceToHost));
    if (keys && p.grid.klen) {
      std::vector<std::uint64_t> packed(p.n);
      MB_CUDA(cudaMemcpy(packed.data(), p.keys.ptr, p.n * 8, cudaMemcpyDeviceToHost));
      for (std::uint64_t i = 0; i < p.n; ++i) p.grid.unpack(packed[i], keys + i * p.grid.klen);
    }
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// device-resident record_round for engine callers (protocols.hpp:68-84)
// ---------------------------------------------------------------------------
namespace {

// cached: FAST with representatives, the row-partial cache kept warm
// (launch_distortion_fast_cached; reps lists only what changed)
template <typename T>
void engine_diag(moshpit_engine* e, const T* x, std::uint64_t ld, std::uint64_t dim,
                 double* dist_slot, double* drift_slot, cudaStream_t s,
                 const RepRows* reps = nullptr, bool cached = false) {
  const std::uint64_t n = e->plane->n;
  const int exact = e->diag == MOSHPIT_DIAG_EXACT;
  if (drift_slot) {
    MB_CUDA(cudaEventRecord(e->ev_fork, s));
    MB_CUDA(cudaStreamWaitEvent(e->aux->s, e->ev_fork, 0));
  }
  if (cached && reps && !exact)
    launch_distortion_fast_cached<T>(x, n, ld, dim, e->ref.as<double>(), e->sq.as<double>(),
                                     e->part.as<double>(), dist_slot, s, *reps);
  else
    launch_distortion<T>(x, n, ld, dim, e->ref.as<double>(), e->sq.as<double>(),
                         e->part.as<double>(), dist_slot, exact, s, reps);
  if (drift_slot) {
    bool done = false;
    if constexpr (std::is_same<T, float>::value) {
      if (reps && reps->rep) {
        e->colsum.resize(colsum_scratch_bytes(n, dim));
        done = launch_colmean_exactsum(x, n, ld, dim, reps->rep, e->mean.as<double>(),
                                       e->colsum.ptr, e->aux->s);
      }
    }
    if (!done)
      launch_colmean<T, double>(x, n, ld, dim, reps ? reps->rep : nullptr, e->mean.as<double>(),
                                e->aux->s, true);
    launch_drift(e->mean.as<double>(), e->ref.as<double>(), dim, e->part2.as<double>(),
                 drift_slot, exact, e->aux->s);
    MB_CUDA(cudaEventRecord(e->ev_join, e->aux->s));
    MB_CUDA(cudaStreamWaitEvent(s, e->ev_join, 0));
  }
}

}  // namespace

extern "C" {

int moshpit_engine_set_reference(moshpit_engine* e, int dtype, const void* state,
                                 std::uint64_t dim, std::uint64_t ld, int diag, void* stream) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    if (diag < MOSHPIT_DIAG_NONE || diag > MOSHPIT_DIAG_EXACT)
      throw std::invalid_argument("engine: unknown diagnostics mode");
    check_state(dtype, state, dim, ld);
    DeviceGuard g(e->plane->device);
    auto s = static_cast<cudaStream_t>(stream);
    e->plane->order_after(s);
    const std::uint64_t n = e->plane->n;
    e->diag = diag;
    e->diag_dim = dim;
    e->log_n = 0;
    if (diag == MOSHPIT_DIAG_NONE) return;
    if (!e->aux) {
      e->aux = std::make_unique<StreamHolder>(aux_priority());
      MB_CUDA(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
      MB_CUDA(cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
    }
    e->ref.resize(dim * 8 + 16);
    e->mean.resize(dim * 8 + 16);
    e->sq.resize(n * 8 + 16);
    e->part.resize(diag_partial_elems(n, dim) * 8 + 16);
    e->part2.resize(diag_partial_elems(n, dim) * 8 + 16);
    if (e->log_cap < 1024) {
      e->log.resize((1 + 2 * 1024) * 8);
      e->log_cap = 1024;
    }
    // reference = mean_of(initial) (protocols.hpp:119), then the initial distortion
    if (dtype == MOSHPIT_F32) {
      launch_colmean<float, double>(static_cast<const float*>(state), n, ld, dim, nullptr,
                                    e->ref.as<double>(), s);
      engine_diag<float>(e, static_cast<const float*>(state), ld, dim, e->log.as<double>(),
                         nullptr, s);
    } else {
      launch_colmean<double, double>(static_cast<const double*>(state), n, ld, dim, nullptr,
                                     e->ref.as<double>(), s);
      engine_diag<double>(e, static_cast<const double*>(state), ld, dim, e->log.as<double>(),
                          nullptr, s);
    }
    e->plane->mark_done(s);
  });
}

namespace {

// record_round after the state's latest change; with `after_round` the
// state is exactly the output of the engine's last round, so its averaged
// groups' rows are identical and only representative rows are read.
// cache_warm (FAST, after_round, within one moshpit_engine_rounds_record
// call): every row's FAST partials are in its slot from the previous round's
// record, so only the averaged groups' representatives are re-read.
void engine_record_impl(moshpit_engine* e, int dtype, const void* state, std::uint64_t dim,
                        std::uint64_t ld, cudaStream_t s, bool after_round,
                        bool use_cache = false, bool cache_warm = false) {
  if (e->diag == MOSHPIT_DIAG_NONE)
    throw std::invalid_argument("engine_record: set_reference with a diagnostics mode first");
  if (dim != e->diag_dim) throw std::invalid_argument("engine_record: dim changed");
  e->plane->order_after(s);
  if (e->log_n == e->log_cap) {  // grow the device log (rare: synchronises)
    DeviceBuffer bigger((1 + 4 * e->log_cap) * 8);
    MB_CUDA(cudaStreamSynchronize(s));
    MB_CUDA(cudaMemcpy(bigger.ptr, e->log.ptr, (1 + 2 * e->log_cap) * 8,
                       cudaMemcpyDeviceToDevice));
    std::swap(e->log.ptr, bigger.ptr);
    std::swap(e->log.bytes, bigger.bytes);
    e->log_cap *= 2;
  }
  RepRows reps;
  if (after_round) {
    const std::uint64_t n = e->plane->n;
    e->rep.resize(n * 4 + 16);
    e->rlist.resize(n * 4 + 16);
    e->rcount.resize(16);
    Plane& p = *e->plane;
    launch_build_reps(p.members.as<std::uint32_t>(), p.goff.as<std::uint32_t>(),
                      p.gvoid.as<std::uint8_t>(), p.counts.as<std::uint32_t>(), n,
                      e->rep.as<std::uint32_t>(), e->rlist.as<std::uint32_t>(),
                      e->rcount.as<std::uint32_t>(), s, use_cache && cache_warm ? 0 : 1);
    reps = RepRows{e->rep.as<std::uint32_t>(), e->rlist.as<std::uint32_t>(),
                   e->rcount.as<std::uint32_t>()};
  }
  double* slot = e->log.as<double>() + 1 + 2 * e->log_n;
  const bool cached = use_cache && after_round;
  if (dtype == MOSHPIT_F32)
    engine_diag<float>(e, static_cast<const float*>(state), ld, dim, slot, slot + 1, s,
                       after_round ? &reps : nullptr, cached);
  else
    engine_diag<double>(e, static_cast<const double*>(state), ld, dim, slot, slot + 1, s,
                        after_round ? &reps : nullptr, cached);
  ++e->log_n;
  e->plane->mark_done(s);
}

}  // namespace

int moshpit_engine_record(moshpit_engine* e, int dtype, const void* state, std::uint64_t dim,
                          std::uint64_t ld, void* stream) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    check_state(dtype, state, dim, ld);
    DeviceGuard g(e->plane->device);
    engine_record_impl(e, dtype, state, dim, ld, static_cast<cudaStream_t>(stream), false);
  });
}

// One round and its record_round in one call (protocols.hpp:142-173): the
// diagnostics read one representative row per averaged group.
int moshpit_engine_round_record(moshpit_engine* e, int dtype, void* state, std::uint64_t dim,
                                std::uint64_t ld, void* stream, std::uint32_t* active_out) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    if (!state) throw std::invalid_argument("engine_round_record: null state");
    check_state(dtype, state, dim, ld);
    if (e->diag == MOSHPIT_DIAG_NONE)
      throw std::invalid_argument("engine_record: set_reference with a diagnostics mode first");
    DeviceGuard g(e->plane->device);
    auto s = static_cast<cudaStream_t>(stream);
    const std::uint32_t a =
        e->plane->round(&e->fail, e->p, e->clock, dtype, state, dim, ld, s, e->variant);
    if (active_out) *active_out = a;
    engine_record_impl(e, dtype, state, dim, ld, s, true);
  });
}

// `rounds` rounds, each followed by its record_round, in one call (the
// protocols.hpp:142-173 loop on device-resident state).  Between the rounds
// of one call nothing else touches the state, so with FAST diagnostics the
// rows of voided groups -- unchanged by their round -- keep their FAST row
// partials from the previous record and only the averaged groups'
// representatives are re-read (the first round of the call reads every
// representative).  TrialReport bits are those of `rounds` round_record
// calls.  active_out: [rounds] (optional).
int moshpit_engine_rounds_record(moshpit_engine* e, int dtype, void* state, std::uint64_t dim,
                                 std::uint64_t ld, std::uint32_t rounds, void* stream,
                                 std::uint32_t* active_out) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    if (!state) throw std::invalid_argument("engine_rounds_record: null state");
    check_state(dtype, state, dim, ld);
    if (e->diag == MOSHPIT_DIAG_NONE)
      throw std::invalid_argument("engine_record: set_reference with a diagnostics mode first");
    DeviceGuard g(e->plane->device);
    auto s = static_cast<cudaStream_t>(stream);
    const bool fast = e->diag == MOSHPIT_DIAG_FAST;
    for (std::uint32_t r = 0; r < rounds; ++r) {
      const std::uint32_t a =
          e->plane->round(&e->fail, e->p, e->clock, dtype, state, dim, ld, s, e->variant);
      if (active_out) active_out[r] = a;
      engine_record_impl(e, dtype, state, dim, ld, s, true, fast, r > 0);
    }
  });
}

int moshpit_engine_report(moshpit_engine* e, double* initial_distortion, double* distortion,
                          double* mean_drift, std::uint64_t cap, std::uint64_t* count) {
  return guarded([&] {
    if (!e) throw std::invalid_argument("null engine");
    DeviceGuard g(e->plane->device);
    e->plane->sync_done();
    const std::uint64_t k = std::min<std::uint64_t>(cap, e->log_n);
    if (count) *count = e->log_n;
    if (e->diag == MOSHPIT_DIAG_NONE) {
      if (initial_distortion) *initial_distortion = std::nan("");
      return;
    }
    std::vector<double> h(1 + 2 * k);
    MB_CUDA(cudaMemcpy(h.data(), e->log.ptr, h.size() * 8, cudaMemcpyDeviceToHost));
    if (initial_distortion) *initial_distortion = h[0];
    for (std::uint64_t t = 0; t < k; ++t) {
      if (distortion) distortion[t] = h[1 + 2 * t];
      if (mean_drift) mean_drift[t] = h[2 + 2 * t];
    }
  });
}

int moshpit_fill_synthetic(int dtype, void* state, std::uint64_t n, std::uint64_t dim,
                           std::uint64_t ld, std::uint64_t seed, std::uint64_t col0,
                           void* stream) {
  return guarded([&] {
    elem_size(dtype);
    if (ld < dim) throw std::invalid_argument("fill_synthetic: ld < dim");
    require_device();
    if (dtype == MOSHPIT_F32)
      launch_fill_synthetic<float>(static_cast<float*>(state), n, dim, ld, seed, col0,
                                   static_cast<cudaStream_t>(stream));
    else
      launch_fill_synthetic<double>(static_cast<double*>(state), n, dim, ld, seed, col0,
                                    static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
