// plane.cuh -- the device-resident integer plane of one Moshpit trial: the
// reference's sequential RNG draws (host), group formation (kernel 1) and the
// group-mean launch (kernel 2) for one round.  Shared by the single-GPU engine
// (capi.cu) and the peer-sharded engine (shard.cu).
#pragma once

#include <cstring>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/moshpit_b200.h"
#include "common.cuh"

namespace mb200 {

extern thread_local std::string g_last_error;

// Runs f, mapping the reference's exception classes onto MOSHPIT_ERR_*.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return MOSHPIT_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return MOSHPIT_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return MOSHPIT_ERR_OUT_OF_RANGE;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return MOSHPIT_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MOSHPIT_ERR_RUNTIME;
  } catch (...) {
    g_last_error = "unknown error";
    return MOSHPIT_ERR_RUNTIME;
  }
}

inline std::size_t elem_size(int dtype) {
  if (dtype == MOSHPIT_F32) return 4;
  if (dtype == MOSHPIT_F64) return 8;
  throw std::invalid_argument("dtype must be MOSHPIT_F32 or MOSHPIT_F64");
}

// Row pitch of engine-owned peer state: 16-byte multiples, and 4 KB
// multiples for rows of 64 KB or more -- measured on B200
// (profiles/ld_sweep.py): Kernel 2 on 4096 x 6e6 fp32 runs at 92.4 % of the
// HBM peak with a 24,000,000-byte pitch and 96.4 % with a 4 KB-multiple one.
inline std::uint64_t padded_ld(std::uint64_t dim, std::size_t elem) {
  const std::uint64_t v = (dim * elem >= (64u << 10)) ? 4096 / elem : 16 / elem;
  const std::uint64_t ld = (dim + v - 1) / v * v;
  return ld ? ld : v;
}

struct StreamHolder {
  cudaStream_t s = nullptr;
  StreamHolder() { MB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  // priority: lower numbers are higher priority (cudaDeviceGetStreamPriorityRange)
  explicit StreamHolder(int priority) {
    MB_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority));
  }
  ~StreamHolder() {
    if (s) cudaStreamDestroy(s);
  }
};


// Partial Fisher-Yates over [0, capacity) (protocols.hpp:124-130,
// optimizer.hpp:254-259): a dense permutation when the grid is at most ~8n
// cells, else a sparse map, so memory stays O(n) rather than O(M^d); either
// way the draws and swaps are exactly the reference's.
inline std::vector<std::uint64_t> draw_cells(Xoshiro& st, std::uint64_t capacity,
                                      std::uint64_t n) {
  std::vector<std::uint64_t> cells(n);
  if (capacity <= 8 * n + 4096) {  // dense permutation: same draws, same swaps
    std::vector<std::uint64_t> perm(capacity);
    for (std::uint64_t i = 0; i < capacity; ++i) perm[i] = i;
    for (std::uint64_t i = 0; i < n; ++i) {
      const std::uint64_t j = i + st.below(capacity - i);
      std::swap(perm[i], perm[j]);
      cells[i] = perm[i];
    }
    return cells;
  }
  std::unordered_map<std::uint64_t, std::uint64_t> moved;
  moved.reserve(2 * n);
  auto at = [&](std::uint64_t i) {
    auto it = moved.find(i);
    return it == moved.end() ? i : it->second;
  };
  for (std::uint64_t i = 0; i < n; ++i) {
    const std::uint64_t j = i + st.below(capacity - i);
    const std::uint64_t vi = at(i), vj = at(j);
    moved[i] = vj;
    moved[j] = vi;
    cells[i] = vj;
  }
  return cells;
}

// ---------------------------------------------------------------------------
// The device-resident integer plane of one trial (keys, tables, draws).
// ---------------------------------------------------------------------------
struct Plane {
  Grid grid;
  std::uint64_t n = 0;
  int device = 0;
  DeviceBuffer keys, draws, members, goff, gvoid, rank, act, counts, totals,
      sidx, scs, sgi, cellbuf;
  static constexpr int kStages = 4;
  PinnedBuffer stage[kStages];
  cudaEvent_t ev[kStages] = {};
  int slot = 0;
  std::uint32_t last_active = 0;
  std::uint64_t rounds_done = 0;
  // Cross-stream ordering: the tables above are reused every round, so a
  // round issued on a different stream than the last one first waits for the
  // last round's end (`done`, recorded by mark_done at the end of a round).
  cudaStream_t last_stream = nullptr;
  cudaEvent_t done = nullptr;
  bool have_done = false;
  // optional CUDA-event bracketing of kernel 2 on its launch stream
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
  std::size_t tev_used = 0;

  Plane(std::uint32_t M, std::uint32_t d, std::uint64_t n_, int dev)
      : grid(M, d), n(n_), device(dev) {
    if (n == 0) throw std::invalid_argument("run_moshpit: no peers");
    if (n > grid.capacity)
      throw std::invalid_argument("run_moshpit: N exceeds grid capacity M^d");
    if (n > 0x7fffffffull)
      throw std::invalid_argument("moshpit engine: more than 2^31 peers");
    std::uint64_t np = 1;
    while (np < n) np <<= 1;
    keys.resize(n * 8);
    draws.resize(n * 9 + 16);
    members.resize(n * 4);
    goff.resize((n + 1) * 4);
    gvoid.resize(n);
    rank.resize(n * 4);
    act.resize(n * 4);
    counts.resize(16);
    totals.resize(16);
    sidx.resize(np * 4);
    scs.resize(n * 4);
    sgi.resize(n * 4);
    cellbuf.resize(n * 8);
    {
      // zeroed on a private stream and waited for: a plain cudaMemset goes to
      // the legacy stream, which the engines' non-blocking streams do not
      // order against -- kernel 1 could write `counts` before the memset
      // lands (seen with concurrent host threads)
      StreamHolder z;
      MB_CUDA(cudaMemsetAsync(totals.ptr, 0, 16, z.s));
      MB_CUDA(cudaMemsetAsync(counts.ptr, 0, 16, z.s));
      MB_CUDA(cudaStreamSynchronize(z.s));
    }
    for (int i = 0; i < kStages; ++i) {
      stage[i].resize(n * 9 + 16);
      MB_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    MB_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  }
  ~Plane() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (done) cudaEventDestroy(done);
    for (auto& pr : tev) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  }

  std::pair<cudaEvent_t, cudaEvent_t> timing_pair() {
    if (tev_used == tev.size()) {
      cudaEvent_t a, b;
      MB_CUDA(cudaEventCreate(&a));
      MB_CUDA(cudaEventCreate(&b));
      tev.emplace_back(a, b);
    }
    return tev[tev_used++];
  }

  // cells -> initial keys (matchmaking.hpp:46-59), on the device.
  void init_cells(Xoshiro& cell_stream, cudaStream_t s) {
    const auto cells = draw_cells(cell_stream, grid.capacity, n);
    order_after(s);
    const int k = next_slot();
    std::memcpy(stage[k].ptr, cells.data(), n * 8);
    MB_CUDA(cudaMemcpyAsync(cellbuf.ptr, stage[k].ptr, n * 8, cudaMemcpyHostToDevice, s));
    MB_CUDA(cudaEventRecord(ev[k], s));
    launch_initial_keys(cellbuf.as<std::uint64_t>(), keys.as<std::uint64_t>(), n,
                        grid.M, grid.d, s);
    mark_done(s);
  }

  // Work on `s` that touches the plane's tables starts after the last round.
  void order_after(cudaStream_t s) {
    if (have_done && s != last_stream) MB_CUDA(cudaStreamWaitEvent(s, done, 0));
  }
  // End of a round (or of any work using the tables) on `s`.
  void mark_done(cudaStream_t s) {
    MB_CUDA(cudaEventRecord(done, s));
    have_done = true;
    last_stream = s;
  }
  // Host wait for the last round (stats / table reads).
  void sync_done() {
    if (have_done) MB_CUDA(cudaEventSynchronize(done));
    else MB_CUDA(cudaDeviceSynchronize());
  }

  int next_slot() {
    const int k = slot;
    slot = (slot + 1) % kStages;
    MB_CUDA(cudaEventSynchronize(ev[k]));  // host staging slot reusable
    return k;
  }

  // One round: host draws (protocols.hpp:143-150), group formation (kernel 1),
  // group mean (kernel 2).  fail == nullptr or p <= 0: no failure draws.
  std::uint32_t round(Xoshiro* fail, double p, Xoshiro& clock, int dtype,
                      void* state, std::uint64_t dim, std::uint64_t ld,
                      cudaStream_t s, int variant,
                      const StepPrologue<float>* step_f = nullptr,
                      const StepPrologue<double>* step_d = nullptr) {
    order_after(s);
    const int k = next_slot();
    auto* ts = stage[k].as<std::uint64_t>();
    auto* failed = reinterpret_cast<std::uint8_t*>(ts + n);
    std::memset(failed, 0, n);
    std::uint32_t active = 0;
    if (fail && p > 0.0) {
      for (std::uint64_t i = 0; i < n; ++i) failed[i] = fail->bernoulli(p) ? 1 : 0;
    }
    for (std::uint64_t i = 0; i < n; ++i) active += failed[i] == 0;
    for (std::uint64_t i = 0; i < n; ++i) ts[i] = clock.next() >> 16;
    MB_CUDA(cudaMemcpyAsync(draws.ptr, ts, n * 9, cudaMemcpyHostToDevice, s));
    MB_CUDA(cudaEventRecord(ev[k], s));

    GroupArgs a;
    a.n = static_cast<std::uint32_t>(n);
    a.cap = grid.M;
    a.M = grid.M;
    a.pow_drop = grid.pow_drop;
    a.advance_keys = 1;
    a.klen_zero = grid.klen == 0;
    a.keys = keys.as<std::uint64_t>();
    a.ts = draws.as<std::uint64_t>();
    a.failed = draws.as<std::uint8_t>() + n * 8;
    a.members = members.as<std::uint32_t>();
    a.goff = goff.as<std::uint32_t>();
    a.gvoid = gvoid.as<std::uint8_t>();
    a.rank = rank.as<std::uint32_t>();
    a.act = act.as<std::uint32_t>();
    a.counts = counts.as<std::uint32_t>();
    a.totals = totals.as<unsigned long long>();
    a.sidx = sidx.as<std::uint32_t>();
    a.scs = scs.as<std::uint32_t>();
    a.sgi = sgi.as<std::uint32_t>();
    launch_form_groups(a, true, s);
    if (state && dim) {
      std::pair<cudaEvent_t, cudaEvent_t> te{};
      if (timing) {
        te = timing_pair();
        MB_CUDA(cudaEventRecord(te.first, s));
      }
      if (dtype == MOSHPIT_F32)
        launch_group_mean<float>(static_cast<float*>(state), ld, dim, a.members, a.goff,
                                 a.act, a.counts, grid.M, variant, s, step_f);
      else
        launch_group_mean<double>(static_cast<double*>(state), ld, dim, a.members, a.goff,
                                  a.act, a.counts, grid.M, variant, s, step_d);
      if (timing) MB_CUDA(cudaEventRecord(te.second, s));
    }
    last_active = active;
    ++rounds_done;
    mark_done(s);
    return active;
  }
};


// The tables of R consecutive rounds of a Plane (kernel 1 each, no data
// pass) copied aside for the fused-rounds kernel (fused_rounds.cu).
struct RoundTables {
  DeviceBuffer members, goff, act, counts, rounds, scratch;
  std::vector<FusedRound> host;  // the same tables' device pointers, per round
  void form(Plane& p, std::uint32_t R, Xoshiro* fail, double prob, Xoshiro& clock,
            cudaStream_t s, std::uint32_t* active_out = nullptr) {
    const std::uint64_t n = p.n;
    members.resize(R * n * 4 + 16);
    goff.resize(R * (n + 1) * 4 + 16);
    act.resize(R * n * 4 + 16);
    counts.resize(R * 16 + 16);
    rounds.resize(R * sizeof(FusedRound) + 16);
    std::vector<FusedRound> h(R);
    for (std::uint32_t r = 0; r < R; ++r) {
      const std::uint32_t a = p.round(fail, prob, clock, MOSHPIT_F32, nullptr, 0, 0, s, 0);
      if (active_out) active_out[r] = a;
      auto* m = members.as<std::uint32_t>() + r * n;
      auto* g = goff.as<std::uint32_t>() + r * (n + 1);
      auto* ac = act.as<std::uint32_t>() + r * n;
      auto* c = counts.as<std::uint32_t>() + r * 4;
      MB_CUDA(cudaMemcpyAsync(m, p.members.ptr, n * 4, cudaMemcpyDeviceToDevice, s));
      MB_CUDA(cudaMemcpyAsync(g, p.goff.ptr, (n + 1) * 4, cudaMemcpyDeviceToDevice, s));
      MB_CUDA(cudaMemcpyAsync(ac, p.act.ptr, n * 4, cudaMemcpyDeviceToDevice, s));
      MB_CUDA(cudaMemcpyAsync(c, p.counts.ptr, 16, cudaMemcpyDeviceToDevice, s));
      h[r] = FusedRound{m, g, ac, c};
    }
    // pageable source: staged before the call returns
    MB_CUDA(cudaMemcpyAsync(rounds.ptr, h.data(), R * sizeof(FusedRound),
                            cudaMemcpyHostToDevice, s));
    host = h;
  }
  const FusedRound* dev() const { return static_cast<const FusedRound*>(rounds.ptr); }
};

// Slab-pipelined run_moshpit over host buffers (stream_run.cu).  The initial
// state is either one buffer (row i at base + i * pitch_bytes) or an array of
// row pointers (the drop-in's std::vector<ParamVector>, no flattening).
struct HostRows {
  const void* base = nullptr;
  std::uint64_t pitch_bytes = 0;
  const void* const* rows = nullptr;
};
std::uint64_t stream_slab_cols(std::uint64_t n, std::size_t es, std::uint64_t dim);
template <typename T>
void run_moshpit_streamed(std::uint32_t M, std::uint32_t d, const HostRows& src, std::uint64_t n,
                          std::uint64_t dim, double p, std::uint64_t seed, std::uint32_t rounds,
                          int diag, double* init_dist, double* dist, double* drift,
                          std::uint32_t* active, T* final_out, std::uint64_t W);

}  // namespace mb200
