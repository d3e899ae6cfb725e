// stream_run.cu -- run_moshpit (protocols.hpp:108-179) on HOST buffers as a
// D-slab pipeline.
//
// Group formation never depends on vector values and coordinates are
// independent, so the trial's integer plane is computed once
// (host draws + kernel 1 for all R rounds, tables kept on the device) and
// replayed on every D-slab: slab s+1 is copied host->device while slab s runs
// its R rounds (kernel 2 + diagnostics) and slab s-1 is copied back.  The
// j-sums of record_round continue across slabs (EXACT: per-peer running
// accumulators in j order; FAST: 64 Ki-element chunk partials at their global
// chunk index), so the TrialReport is identical to the resident path's.  The
// end-to-end time approaches max(H2D, D2H, compute) instead of their sum, and
// the device footprint is three slabs instead of the whole state.
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>

#include "plane.cuh"

namespace mb200 {

std::uint64_t stream_slab_cols(std::uint64_t n, std::size_t es, std::uint64_t dim) {
  const std::uint64_t chunk = diag_chunk();
  std::uint64_t budget = 256ull << 20;
  if (const char* e = std::getenv("MOSHPIT_SLAB_BYTES")) budget = std::strtoull(e, nullptr, 10);
  std::uint64_t w = budget / (n * es);
  w = w / chunk * chunk;
  if (w < chunk) w = chunk;
  if (w > dim) w = (dim + chunk - 1) / chunk * chunk;
  return w;
}

namespace {

// A small persistent pool of host threads for packing pageable caller memory
// into the pinned staging ring (one memcpy per row segment, rows split across
// the threads).  run(f) calls f(t, T) on all T threads and waits.
class HostPool {
 public:
  explicit HostPool(unsigned n) {
    for (unsigned t = 1; t < n; ++t) th_.emplace_back([this, t] { loop(t); });
    n_ = n;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  unsigned size() const { return n_; }
  void run(const std::function<void(unsigned, unsigned)>& f) {
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &f;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0, n_);
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(unsigned t) {
    std::uint64_t seen = 0;
    for (;;) {
      const std::function<void(unsigned, unsigned)>* f;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        f = job_;
      }
      (*f)(t, n_);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(unsigned, unsigned)>* job_ = nullptr;
  unsigned n_ = 1, pending_ = 0;
  std::uint64_t gen_ = 0;
  bool stop_ = false;
};

bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Grow-only per-thread workspace: repeated host-buffer calls (the harness
// runs many trials per thread) reuse the slab ring, tables, diagnostics
// buffers, streams and -- for the same (M, d, n) -- the integer plane, instead
// of paying cudaMalloc/cudaFree/cudaMallocHost on every call.
struct StreamWorkspace {
  int dev = -1;
  std::unique_ptr<DeviceBuffer> ring[3];
  DeviceBuffer t_mem, t_goff, t_act, t_cnt, ref, mean_s, acc, acc2, rpart, dpart, out;
  DeviceBuffer t_rep, t_rlist, t_rcount;  // representatives of every round (RepRows)
  std::unique_ptr<Plane> plane;
  std::uint32_t pM = 0, pd = 0;
  std::uint64_t pn = 0;
  std::unique_ptr<StreamHolder> s_in, s_cmp, s_out, s_aux;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // pageable callers: pinned staging rings (in, out) and the packing threads
  PinnedBuffer hin[3], hout[3];
  std::unique_ptr<HostPool> pool;
  ~StreamWorkspace() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }
};
thread_local std::unique_ptr<StreamWorkspace> tl_ws;

StreamWorkspace& workspace(int dev) {
  if (!tl_ws || tl_ws->dev != dev) {
    tl_ws = std::make_unique<StreamWorkspace>();
    tl_ws->dev = dev;
    for (auto& r : tl_ws->ring) r = std::make_unique<DeviceBuffer>();
    tl_ws->s_in = std::make_unique<StreamHolder>();
    tl_ws->s_cmp = std::make_unique<StreamHolder>();
    tl_ws->s_out = std::make_unique<StreamHolder>();
    tl_ws->s_aux = std::make_unique<StreamHolder>();
    MB_CUDA(cudaEventCreateWithFlags(&tl_ws->ev_fork, cudaEventDisableTiming));
    MB_CUDA(cudaEventCreateWithFlags(&tl_ws->ev_join, cudaEventDisableTiming));
  }
  return *tl_ws;
}

}  // namespace

template <typename T>
void run_moshpit_streamed(std::uint32_t M, std::uint32_t d, const HostRows& src, std::uint64_t n,
                          std::uint64_t dim, double p, std::uint64_t seed, std::uint32_t rounds,
                          int diag, double* init_dist, double* dist, double* drift,
                          std::uint32_t* active, T* final_out, std::uint64_t W) {
  const std::size_t es = sizeof(T);
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  StreamWorkspace& ws = workspace(dev);
  // Pageable (or row-pointer) sources are packed by host threads into a
  // pinned ring and copied with one contiguous async copy per slab; pinned
  // contiguous sources are copied directly (2-D copy).
  const bool stage_in = src.rows || !is_pinned(src.base);
  const bool stage_out = final_out && !is_pinned(final_out);
  if ((stage_in || stage_out) && !ws.pool) {
    unsigned hc = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("MOSHPIT_HOST_THREADS")) hc = (unsigned)std::atoi(e);
    ws.pool = std::make_unique<HostPool>(std::max(1u, std::min(hc ? hc : 1u, 32u)));
  }
  auto row_ptr = [&](std::uint64_t i) -> const char* {
    return src.rows ? static_cast<const char*>(src.rows[i])
                    : static_cast<const char*>(src.base) + i * src.pitch_bytes;
  };
  StreamHolder &s_in = *ws.s_in, &s_cmp = *ws.s_cmp, &s_out = *ws.s_out;
  const std::uint64_t R = rounds;
  // 1. the integer plane of every round (identical for all slabs)
  if (!ws.plane || ws.pM != M || ws.pd != d || ws.pn != n) {
    ws.plane.reset();
    ws.plane = std::make_unique<Plane>(M, d, n, dev);
    ws.pM = M;
    ws.pd = d;
    ws.pn = n;
  }
  Plane& plane = *ws.plane;
  Xoshiro cells = Xoshiro::named(seed, "cells");
  plane.init_cells(cells, s_cmp.s);
  Xoshiro fail = Xoshiro::named(seed, "failures");
  Xoshiro clock = Xoshiro::named(seed, "priorities");
  DeviceBuffer &t_mem = ws.t_mem, &t_goff = ws.t_goff, &t_act = ws.t_act, &t_cnt = ws.t_cnt;
  t_mem.resize(R * n * 4 + 16);
  t_goff.resize(R * (n + 1) * 4 + 16);
  t_act.resize(R * n * 4 + 16);
  t_cnt.resize(R * 16 + 16);
  const bool dgr = diag != MOSHPIT_DIAG_NONE;
  if (dgr) {
    ws.t_rep.resize(R * n * 4 + 16);
    ws.t_rlist.resize(R * n * 4 + 16);
    ws.t_rcount.resize(R * 4 + 16);
  }
  for (std::uint64_t r = 0; r < R; ++r) {
    active[r] = plane.round(&fail, p, clock, 0, nullptr, 0, 0, s_cmp.s, 0);
    if (dgr)  // the rows of every averaged group are identical after round r
      launch_build_reps(plane.members.as<std::uint32_t>(), plane.goff.as<std::uint32_t>(),
                        plane.gvoid.as<std::uint8_t>(), plane.counts.as<std::uint32_t>(), n,
                        ws.t_rep.as<std::uint32_t>() + r * n,
                        ws.t_rlist.as<std::uint32_t>() + r * n,
                        ws.t_rcount.as<std::uint32_t>() + r, s_cmp.s);
    MB_CUDA(cudaMemcpyAsync(t_mem.as<std::uint32_t>() + r * n, plane.members.ptr, n * 4,
                            cudaMemcpyDeviceToDevice, s_cmp.s));
    MB_CUDA(cudaMemcpyAsync(t_goff.as<std::uint32_t>() + r * (n + 1), plane.goff.ptr,
                            (n + 1) * 4, cudaMemcpyDeviceToDevice, s_cmp.s));
    MB_CUDA(cudaMemcpyAsync(t_act.as<std::uint32_t>() + r * n, plane.act.ptr, n * 4,
                            cudaMemcpyDeviceToDevice, s_cmp.s));
    MB_CUDA(cudaMemcpyAsync(t_cnt.as<std::uint32_t>() + r * 4, plane.counts.ptr, 16,
                            cudaMemcpyDeviceToDevice, s_cmp.s));
  }
  // 2. slab ring
  const std::uint64_t nslab = (dim + W - 1) / W;
  const std::uint64_t chunk = diag_chunk();
  const std::uint64_t nch = (dim + chunk - 1) / chunk;
  const int exact = diag == MOSHPIT_DIAG_EXACT;
  const bool dg = diag != MOSHPIT_DIAG_NONE;
  constexpr int kRing = 3;
  std::unique_ptr<DeviceBuffer>* buf = ws.ring;
  for (int k = 0; k < kRing; ++k) buf[k]->resize(n * W * es + 16);
  DeviceBuffer &ref = ws.ref, &mean_s = ws.mean_s, &acc = ws.acc, &acc2 = ws.acc2,
               &rpart = ws.rpart, &dpart = ws.dpart, &out = ws.out;
  if (dg) {
    ref.resize(dim * 8 + 16);
    mean_s.resize(W * 8 + 16);
    acc.resize((R + 1) * n * 8);
    acc2.resize((R + 1) * 16 + 16);
    if (!exact) {
      rpart.resize((R + 1) * n * nch * 8 + 16);
      dpart.resize((R + 1) * 2 * nch * 8 + 16);
    }
    out.resize((2 * R + 2) * 8);
    MB_CUDA(cudaMemsetAsync(acc.ptr, 0, (R + 1) * n * 8, s_cmp.s));
    MB_CUDA(cudaMemsetAsync(acc2.ptr, 0, (R + 1) * 16 + 16, s_cmp.s));
  }
  cudaEvent_t ev_in[kRing], ev_cmp[kRing], ev_out[kRing];
  for (int k = 0; k < kRing; ++k) {
    MB_CUDA(cudaEventCreateWithFlags(&ev_in[k], cudaEventDisableTiming));
    MB_CUDA(cudaEventCreateWithFlags(&ev_cmp[k], cudaEventDisableTiming));
    MB_CUDA(cudaEventCreateWithFlags(&ev_out[k], cudaEventDisableTiming));
  }
  struct EvGuard {
    cudaEvent_t* e[3];
    ~EvGuard() {
      for (auto* a : e)
        for (int k = 0; k < kRing; ++k) cudaEventDestroy(a[k]);
    }
  } guard{{ev_in, ev_cmp, ev_out}};
  if (stage_in)
    for (int k = 0; k < kRing; ++k) ws.hin[k].resize(n * W * es + 16);
  if (stage_out)
    for (int k = 0; k < kRing; ++k) ws.hout[k].resize(n * W * es + 16);
  bool in_used[kRing] = {}, out_pending[kRing] = {};
  std::uint64_t out_j0[kRing] = {}, out_w[kRing] = {};
  // copy a finished slab from the pinned out-ring into the caller's rows
  auto unpack = [&](int b) {
    MB_CUDA(cudaEventSynchronize(ev_out[b]));
    const char* h = ws.hout[b].as<char>();
    const std::uint64_t j0 = out_j0[b], w = out_w[b];
    ws.pool->run([&](unsigned t, unsigned T_) {
      for (std::uint64_t i = n * t / T_; i < n * (t + 1) / T_; ++i)
        std::memcpy(reinterpret_cast<char*>(final_out) + (i * dim + j0) * es, h + i * W * es,
                    w * es);
    });
    out_pending[b] = false;
  };
  for (std::uint64_t sl = 0; sl < nslab; ++sl) {
    const int b = (int)(sl % kRing);
    const std::uint64_t j0 = sl * W, w = (dim - j0) < W ? (dim - j0) : W;
    T* x = buf[b]->as<T>();
    if (sl >= (std::uint64_t)kRing) MB_CUDA(cudaStreamWaitEvent(s_in.s, ev_out[b], 0));
    if (stage_in) {
      // the previous H2D out of this pinned slot must be done before refilling it
      if (in_used[b]) MB_CUDA(cudaEventSynchronize(ev_in[b]));
      char* h = ws.hin[b].as<char>();
      ws.pool->run([&](unsigned t, unsigned T_) {
        for (std::uint64_t i = n * t / T_; i < n * (t + 1) / T_; ++i)
          std::memcpy(h + i * W * es, row_ptr(i) + j0 * es, w * es);
      });
      MB_CUDA(cudaMemcpy2DAsync(x, W * es, h, W * es, w * es, n, cudaMemcpyHostToDevice,
                                s_in.s));
      in_used[b] = true;
    } else {
      MB_CUDA(cudaMemcpy2DAsync(x, W * es, row_ptr(0) + j0 * es, src.pitch_bytes, w * es, n,
                                cudaMemcpyHostToDevice, s_in.s));
    }
    MB_CUDA(cudaEventRecord(ev_in[b], s_in.s));
    MB_CUDA(cudaStreamWaitEvent(s_cmp.s, ev_in[b], 0));
    const std::uint64_t c0 = j0 / chunk;
    double* refj = dg ? ref.as<double>() + j0 : nullptr;
    if (dg) {
      launch_colmean<T, double>(x, n, W, w, nullptr, refj, s_cmp.s);
      launch_dist_slab<T>(x, n, W, w, refj, exact, acc.as<double>(), rpart.as<double>(), nch, c0,
                          s_cmp.s);
    }
    for (std::uint64_t r = 0; r < R; ++r) {
      launch_group_mean<T>(x, W, w, t_mem.as<std::uint32_t>() + r * n,
                           t_goff.as<std::uint32_t>() + r * (n + 1),
                           t_act.as<std::uint32_t>() + r * n, t_cnt.as<std::uint32_t>() + r * 4,
                           M, MOSHPIT_KERNEL_AUTO, s_cmp.s);
      if (dg) {
        // the distortion j-chains (s_cmp) and colmean + drift (s_aux) only
        // read the slab: run them side by side, join before the next round
        MB_CUDA(cudaEventRecord(ws.ev_fork, s_cmp.s));
        MB_CUDA(cudaStreamWaitEvent(ws.s_aux->s, ws.ev_fork, 0));
        const RepRows rr{ws.t_rep.as<std::uint32_t>() + r * n,
                         ws.t_rlist.as<std::uint32_t>() + r * n,
                         ws.t_rcount.as<std::uint32_t>() + r};
        launch_dist_slab<T>(x, n, W, w, refj, exact, acc.as<double>() + (r + 1) * n,
                            rpart.as<double>() + (r + 1) * n * nch, nch, c0, s_cmp.s, &rr);
        launch_colmean<T, double>(x, n, W, w, rr.rep, mean_s.as<double>(), ws.s_aux->s, true);
        launch_drift_slab(mean_s.as<double>(), refj, w, exact, acc2.as<double>() + 2 * (r + 1),
                          dpart.as<double>() + (r + 1) * 2 * nch, c0, ws.s_aux->s);
        MB_CUDA(cudaEventRecord(ws.ev_join, ws.s_aux->s));
        MB_CUDA(cudaStreamWaitEvent(s_cmp.s, ws.ev_join, 0));
      }
    }
    MB_CUDA(cudaEventRecord(ev_cmp[b], s_cmp.s));
    MB_CUDA(cudaStreamWaitEvent(s_out.s, ev_cmp[b], 0));
    if (stage_out) {
      if (out_pending[b]) unpack(b);  // slot reused: drain slab sl - kRing first
      MB_CUDA(cudaMemcpy2DAsync(ws.hout[b].ptr, W * es, x, W * es, w * es, n,
                                cudaMemcpyDeviceToHost, s_out.s));
      out_pending[b] = true;
      out_j0[b] = j0;
      out_w[b] = w;
    } else if (final_out) {
      MB_CUDA(cudaMemcpy2DAsync(final_out + j0, dim * es, x, W * es, w * es, n,
                                cudaMemcpyDeviceToHost, s_out.s));
    }
    MB_CUDA(cudaEventRecord(ev_out[b], s_out.s));
    // drain the oldest finished slab while the GPU works on the newer ones
    if (stage_out && sl >= 1) {
      const int pb = (int)((sl - 1) % kRing);
      if (out_pending[pb]) unpack(pb);
    }
  }
  if (stage_out)
    for (std::uint64_t k = 0; k < (std::uint64_t)kRing; ++k) {
      const int b = (int)((nslab + k) % kRing);
      if (out_pending[b]) unpack(b);
    }
  if (dg) {
    double* o = out.as<double>();
    for (std::uint64_t r = 0; r <= R; ++r)
      launch_diag_finish(n, nch, exact, acc.as<double>() + r * n,
                         exact ? nullptr : rpart.as<double>() + r * n * nch,
                         acc2.as<double>() + 2 * r,
                         exact ? nullptr : dpart.as<double>() + r * 2 * nch,
                         r == 0 ? o : o + 2 + (r - 1), r == 0 ? nullptr : o + 2 + R + (r - 1),
                         s_cmp.s, r == 0 ? nullptr : ws.t_rep.as<std::uint32_t>() + (r - 1) * n);
    std::vector<double> h(2 * R + 2);
    MB_CUDA(cudaMemcpyAsync(h.data(), o, h.size() * 8, cudaMemcpyDeviceToHost, s_cmp.s));
    MB_CUDA(cudaStreamSynchronize(s_cmp.s));
    *init_dist = h[0];
    for (std::uint64_t r = 0; r < R; ++r) {
      dist[r] = h[2 + r];
      drift[r] = h[2 + R + r];
    }
  } else {
    *init_dist = std::nan("");
    for (std::uint64_t r = 0; r < R; ++r) dist[r] = drift[r] = std::nan("");
  }
  MB_CUDA(cudaStreamSynchronize(s_cmp.s));
  MB_CUDA(cudaStreamSynchronize(s_out.s));
  MB_CUDA(cudaStreamSynchronize(s_in.s));
}

// Frees the calling thread's workspace (slab ring, tables, plane, streams).
void release_stream_workspace() {
  if (!tl_ws) return;
  DeviceGuard g(tl_ws->dev);
  for (auto* h : {tl_ws->s_in.get(), tl_ws->s_cmp.get(), tl_ws->s_out.get(), tl_ws->s_aux.get()})
    if (h) MB_CUDA(cudaStreamSynchronize(h->s));
  tl_ws.reset();
}

template void run_moshpit_streamed<float>(std::uint32_t, std::uint32_t, const HostRows&,
                                          std::uint64_t, std::uint64_t, double, std::uint64_t,
                                          std::uint32_t, int, double*, double*, double*,
                                          std::uint32_t*, float*, std::uint64_t);
template void run_moshpit_streamed<double>(std::uint32_t, std::uint32_t, const HostRows&,
                                           std::uint64_t, std::uint64_t, double, std::uint64_t,
                                           std::uint32_t, int, double*, double*, double*,
                                           std::uint32_t*, double*, std::uint64_t);

}  // namespace mb200

extern "C" int moshpit_release_workspace(void) {
  return mb200::guarded([] { mb200::release_stream_workspace(); });
}
