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
#include <cstdlib>
#include <memory>

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

// Grow-only per-thread workspace: repeated host-buffer calls (the harness
// runs many trials per thread) reuse the slab ring, tables, diagnostics
// buffers, streams and -- for the same (M, d, n) -- the integer plane, instead
// of paying cudaMalloc/cudaFree/cudaMallocHost on every call.
struct StreamWorkspace {
  int dev = -1;
  std::unique_ptr<DeviceBuffer> ring[3];
  DeviceBuffer t_mem, t_goff, t_act, t_cnt, ref, mean_s, acc, acc2, rpart, dpart, out;
  std::unique_ptr<Plane> plane;
  std::uint32_t pM = 0, pd = 0;
  std::uint64_t pn = 0;
  std::unique_ptr<StreamHolder> s_in, s_cmp, s_out;
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
  }
  return *tl_ws;
}

}  // namespace

template <typename T>
void run_moshpit_streamed(std::uint32_t M, std::uint32_t d, const T* initial, std::uint64_t n,
                          std::uint64_t dim, double p, std::uint64_t seed, std::uint32_t rounds,
                          int diag, double* init_dist, double* dist, double* drift,
                          std::uint32_t* active, T* final_out, std::uint64_t W) {
  const std::size_t es = sizeof(T);
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  StreamWorkspace& ws = workspace(dev);
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
  for (std::uint64_t r = 0; r < R; ++r) {
    active[r] = plane.round(&fail, p, clock, 0, nullptr, 0, 0, s_cmp.s, 0);
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
  for (std::uint64_t sl = 0; sl < nslab; ++sl) {
    const int b = (int)(sl % kRing);
    const std::uint64_t j0 = sl * W, w = (dim - j0) < W ? (dim - j0) : W;
    T* x = buf[b]->as<T>();
    if (sl >= (std::uint64_t)kRing) MB_CUDA(cudaStreamWaitEvent(s_in.s, ev_out[b], 0));
    MB_CUDA(cudaMemcpy2DAsync(x, W * es, initial + j0, dim * es, w * es, n,
                              cudaMemcpyHostToDevice, s_in.s));
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
        launch_dist_slab<T>(x, n, W, w, refj, exact, acc.as<double>() + (r + 1) * n,
                            rpart.as<double>() + (r + 1) * n * nch, nch, c0, s_cmp.s);
        launch_colmean<T, double>(x, n, W, w, nullptr, mean_s.as<double>(), s_cmp.s);
        launch_drift_slab(mean_s.as<double>(), refj, w, exact, acc2.as<double>() + 2 * (r + 1),
                          dpart.as<double>() + (r + 1) * 2 * nch, c0, s_cmp.s);
      }
    }
    MB_CUDA(cudaEventRecord(ev_cmp[b], s_cmp.s));
    MB_CUDA(cudaStreamWaitEvent(s_out.s, ev_cmp[b], 0));
    if (final_out)
      MB_CUDA(cudaMemcpy2DAsync(final_out + j0, dim * es, x, W * es, w * es, n,
                                cudaMemcpyDeviceToHost, s_out.s));
    MB_CUDA(cudaEventRecord(ev_out[b], s_out.s));
  }
  if (dg) {
    double* o = out.as<double>();
    for (std::uint64_t r = 0; r <= R; ++r)
      launch_diag_finish(n, nch, exact, acc.as<double>() + r * n,
                         exact ? nullptr : rpart.as<double>() + r * n * nch,
                         acc2.as<double>() + 2 * r,
                         exact ? nullptr : dpart.as<double>() + r * 2 * nch,
                         r == 0 ? o : o + 2 + (r - 1), r == 0 ? nullptr : o + 2 + R + (r - 1),
                         s_cmp.s);
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

template void run_moshpit_streamed<float>(std::uint32_t, std::uint32_t, const float*,
                                          std::uint64_t, std::uint64_t, double, std::uint64_t,
                                          std::uint32_t, int, double*, double*, double*,
                                          std::uint32_t*, float*, std::uint64_t);
template void run_moshpit_streamed<double>(std::uint32_t, std::uint32_t, const double*,
                                           std::uint64_t, std::uint64_t, double, std::uint64_t,
                                           std::uint32_t, int, double*, double*, double*,
                                           std::uint32_t*, double*, std::uint64_t);

}  // namespace mb200
