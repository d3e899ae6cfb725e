// batch.cu -- trial-batched run_moshpit: T independent
// trials, each exactly protocols::run_moshpit (protocols.hpp:108-179) with its
// own Rng(seed_t), executed together -- one kernel-1 launch (one CTA per
// trial), one kernel-2 launch (gridDim.y = trial) and one launch per
// diagnostic per round for the whole batch.  This is the shape of
// harness::run_experiment's sweeps (harness.hpp:195-280: thousands of small
// trials, dim 1 for Table 3), where per-trial launches would be pure overhead.
// The sequential xoshiro draws of different trials are independent: the
// per-round failure and priority streams run on the device, one thread per
// (trial, stream); the once-per-trial cell draws stay on the host threads.
#include <algorithm>
#include <bitset>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <type_traits>

#include "pairwise.cuh"
#include "blocktree.cuh"
#include "plane.cuh"

namespace mb200 {
namespace {

// colmean per trial (blockIdx.y): pairwise over the trial's n rows, fp64.
template <typename T>
__global__ void colmean_b(const T* __restrict__ x, std::uint64_t n, std::uint64_t ld,
                          std::uint64_t dim, double* __restrict__ out) {
  const std::uint64_t j = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (j >= dim) return;
  const T* xt = x + (std::uint64_t)blockIdx.y * n * ld;
  auto ld_fn = [&](std::uint32_t i) -> double { return (double)xt[(std::uint64_t)i * ld + j]; };
  const double s = pairwise_rt<double>(ld_fn, (std::uint32_t)n,
                                       [](double a, double b) { return __dadd_rn(a, b); }, 0.0);
  out[(std::uint64_t)blockIdx.y * dim + j] = __ddiv_rn(s, (double)n);
}

// per row (all trials): sequential over j (core.hpp:118-122)
template <typename T>
__global__ void dist_rows_b(const T* __restrict__ x, std::uint64_t n, std::uint64_t rows,
                            std::uint64_t ld, std::uint64_t dim, const double* __restrict__ ref,
                            double* __restrict__ sq) {
  const std::uint64_t r = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const T* row = x + r * ld;
  const double* rf = ref + (r / n) * dim;
  double acc = 0.0;
  for (std::uint64_t j = 0; j < dim; ++j) {
    const double diff = __dsub_rn((double)row[j], rf[j]);
    acc = __dadd_rn(acc, __dmul_rn(diff, diff));
  }
  sq[r] = acc;
}

// The distortion finish (pairwise over the trial's n row sums, / n;
// core.hpp:125) and the column means of narrow vectors, with the tree over
// peers evaluated by a whole CTA (blocktree.cuh, bit-identical): one CTA per
// trial, or per (column, trial).  The harness sweeps run dim = 1, where one
// thread per trial walking an n-deep serial tree dominated every round.
constexpr int kTreeThreads = 256;

__global__ void __launch_bounds__(kTreeThreads)
    finish_tree_b(const double* __restrict__ sq, std::uint32_t n, double* __restrict__ out,
                  std::uint64_t out_stride) {
  __shared__ double lvl[2 * kBlockTreeMaxNodes];
  const double* s = sq + (std::uint64_t)blockIdx.x * n;
  auto ld_fn = [&](std::uint32_t i) { return s[i]; };
  const double v = pairwise_block(ld_fn, n, lvl);
  if (threadIdx.x == 0) out[(std::uint64_t)blockIdx.x * out_stride] = __ddiv_rn(v, (double)n);
}

template <typename T>
__global__ void __launch_bounds__(kTreeThreads)
    colmean_tree_b(const T* __restrict__ x, std::uint32_t n, std::uint64_t ld, std::uint64_t dim,
                   double* __restrict__ out) {
  __shared__ double lvl[2 * kBlockTreeMaxNodes];
  const std::uint64_t j = blockIdx.x;
  const T* xt = x + (std::uint64_t)blockIdx.y * n * ld + j;
  auto ld_fn = [&](std::uint32_t i) -> double { return (double)xt[(std::uint64_t)i * ld]; };
  const double v = pairwise_block(ld_fn, n, lvl);
  if (threadIdx.x == 0) out[(std::uint64_t)blockIdx.y * dim + j] = __ddiv_rn(v, (double)n);
}

// per trial: drift (protocols.hpp:75-81) in j order
__global__ void drift_b(const double* __restrict__ mean, const double* __restrict__ ref,
                        std::uint64_t dim, std::uint64_t trials, double* __restrict__ out,
                        std::uint64_t out_stride) {
  const std::uint64_t t = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (t >= trials) return;
  const double* m = mean + t * dim;
  const double* r = ref + t * dim;
  double drift_sq = 0.0, ref_sq = 0.0;
  for (std::uint64_t j = 0; j < dim; ++j) {
    const double dm = __dsub_rn(m[j], r[j]);
    drift_sq = __dadd_rn(drift_sq, __dmul_rn(dm, dm));
    ref_sq = __dadd_rn(ref_sq, __dmul_rn(r[j], r[j]));
  }
  out[t * out_stride] = __ddiv_rn(__dsqrt_rn(drift_sq), fmax(__dsqrt_rn(ref_sq), 1e-300));
}

// One round's whole record_round (protocols.hpp:68-84) for narrow vectors,
// one CTA per trial: per-peer sums over j in order, the tree over peers for
// the distortion, the column means (tree over peers per j), then the drift in
// j order -- the four kernels above fused for dim < 32, where a sweep round
// otherwise costs four launches for a few microseconds of work.
template <typename T>
__global__ void __launch_bounds__(kTreeThreads)
    round_diag_narrow(const T* __restrict__ x, std::uint32_t n, std::uint64_t ld,
                      std::uint32_t dim, const double* __restrict__ ref, double* __restrict__ sq,
                      double* __restrict__ mean, double* __restrict__ dist_out,
                      double* __restrict__ drift_out, std::uint64_t out_stride) {
  __shared__ double lvl[2 * kBlockTreeMaxNodes];
  const std::uint64_t t = blockIdx.x;
  const T* xt = x + t * n * ld;
  const double* rf = ref + t * dim;
  double* sqt = sq + t * n;
  double* mt = mean + t * dim;
  for (std::uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    double acc = 0.0;
    for (std::uint32_t j = 0; j < dim; ++j) {
      const double diff = __dsub_rn((double)xt[(std::uint64_t)i * ld + j], rf[j]);
      acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    sqt[i] = acc;
  }
  __syncthreads();
  auto ld_sq = [&](std::uint32_t i) { return sqt[i]; };
  const double dsum = pairwise_block(ld_sq, n, lvl);
  if (threadIdx.x == 0) dist_out[t * out_stride] = __ddiv_rn(dsum, (double)n);
  for (std::uint32_t j = 0; j < dim; ++j) {
    auto ld_x = [&](std::uint32_t i) -> double { return (double)xt[(std::uint64_t)i * ld + j]; };
    const double v = pairwise_block(ld_x, n, lvl);
    if (threadIdx.x == 0) mt[j] = __ddiv_rn(v, (double)n);
  }
  if (threadIdx.x == 0) {
    double drift_sq = 0.0, ref_sq = 0.0;
    for (std::uint32_t j = 0; j < dim; ++j) {
      const double dm = __dsub_rn(mt[j], rf[j]);
      drift_sq = __dadd_rn(drift_sq, __dmul_rn(dm, dm));
      ref_sq = __dadd_rn(ref_sq, __dmul_rn(rf[j], rf[j]));
    }
    drift_out[t * out_stride] = __ddiv_rn(__dsqrt_rn(drift_sq), fmax(__dsqrt_rn(ref_sq), 1e-300));
  }
}

// Per-trial protocol draws on the device (protocols.hpp:86-97, 146-150).
// Each trial's "failures" and "priorities" streams are sequential xoshiro256**
// sequences (rng.hpp:35-91), but the trials are independent: thread
// (trial, stream) continues its stream over a block of rounds and writes the
// draws in the layout kernel 1 reads (ts u64[rows] | failed u8[rows] per
// round).  Same generator, same call order, so the draws equal the host's.
__device__ __forceinline__ std::uint64_t rotl64(std::uint64_t x, int k) {
  return (x << k) | (x >> (64 - k));
}
__device__ __forceinline__ std::uint64_t xnext(std::uint64_t (&s)[4]) {
  const std::uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const std::uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

__global__ void draws_kernel(std::uint64_t* __restrict__ fail_state,
                             std::uint64_t* __restrict__ clock_state, std::uint32_t trials,
                             std::uint32_t n, std::uint32_t nr, std::uint64_t per_round,
                             double p, std::uint8_t* __restrict__ block,
                             std::uint32_t* __restrict__ act, std::uint32_t rounds,
                             std::uint32_t r0) {
  const std::uint32_t id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= 2 * trials) return;
  const std::uint32_t t = id >> 1;
  const std::uint64_t rows = (std::uint64_t)trials * n;
  std::uint64_t* st = (id & 1) ? clock_state + 4 * t : fail_state + 4 * t;
  std::uint64_t s[4] = {st[0], st[1], st[2], st[3]};
  for (std::uint32_t q = 0; q < nr; ++q) {
    std::uint64_t* ts = reinterpret_cast<std::uint64_t*>(block + q * per_round) + (std::uint64_t)t * n;
    std::uint8_t* f = block + q * per_round + rows * 8 + (std::uint64_t)t * n;
    if (id & 1) {  // priorities: clock() >> 16 (protocols.hpp:148-150)
      for (std::uint32_t i = 0; i < n; ++i) ts[i] = xnext(s) >> 16;
    } else {  // failures: bernoulli(p) per peer, no draws at p <= 0 (:89)
      std::uint32_t alive = n;
      if (p > 0.0) {
        // uniform() < p  <=>  (next >> 11) < ceil(p * 2^53): v * 2^-53 and
        // p * 2^53 are exact (power-of-two scaling), v is an integer
        const std::uint64_t thr = (std::uint64_t)ceil(p * 0x1.0p53);
        for (std::uint32_t i = 0; i < n; ++i) {
          const bool dead = (xnext(s) >> 11) < thr;
          f[i] = dead ? 1 : 0;
          alive -= dead ? 1u : 0u;
        }
      } else {
        for (std::uint32_t i = 0; i < n; ++i) f[i] = 0;
      }
      act[(std::uint64_t)t * rounds + r0 + q] = alive;
    }
  }
  st[0] = s[0];
  st[1] = s[1];
  st[2] = s[2];
  st[3] = s[3];
}

// Lane-parallel form of draws_kernel: one warp per (trial, stream).  A block
// of nr rounds is nr*n consecutive draws of the stream; lane L takes draws
// [L*C, (L+1)*C) (C = ceil(nr*n / 32)) and starts from the block's state
// jumped ahead by L*C steps.  The jump is q_L(T) s with q_L = x^(L*C) mod the
// characteristic polynomial of the xoshiro256 transition T (Cayley-Hamilton),
// evaluated as sum_i q_i T^i s: 256 steps instead of L*C.  Every lane then
// runs the reference's generator over its own chunk, so each draw is the one
// the serial chain produces at that position (bit-identical by construction).
struct LanePolys {
  std::uint64_t w[32][4];  // q_L, bit i = coefficient of x^i
};
constexpr std::uint32_t kMaxBlockRounds = 4;

__global__ void __launch_bounds__(64)
    draws_lanes_kernel(std::uint64_t* __restrict__ fail_state,
                       std::uint64_t* __restrict__ clock_state, std::uint32_t trials,
                       std::uint32_t n, std::uint32_t nr, std::uint64_t per_round, double p,
                       std::uint8_t* __restrict__ block, std::uint32_t* __restrict__ act,
                       std::uint32_t rounds, std::uint32_t r0, std::uint64_t chunk,
                       const __grid_constant__ LanePolys polys) {
  __shared__ std::uint32_t dead[2][kMaxBlockRounds];
  const std::uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t id = blockIdx.x * 2 + wib;
  if (lane < kMaxBlockRounds) dead[wib][lane] = 0;
  __syncwarp();
  if (id >= 2 * trials) return;
  const std::uint32_t t = id >> 1;
  const bool clock = id & 1;
  const std::uint64_t rows = (std::uint64_t)trials * n;
  std::uint64_t* st = clock ? clock_state + 4 * t : fail_state + 4 * t;
  if (!clock && !(p > 0.0)) {  // failures at p <= 0: no draws (protocols.hpp:89)
    for (std::uint32_t q = 0; q < nr; ++q) {
      std::uint8_t* f = block + q * per_round + rows * 8 + (std::uint64_t)t * n;
      for (std::uint32_t i = lane; i < n; i += 32) f[i] = 0;
      if (lane == 0) act[(std::uint64_t)t * rounds + r0 + q] = n;
    }
    return;
  }
  const std::uint64_t total = (std::uint64_t)nr * n;
  const std::uint64_t beg = (std::uint64_t)lane * chunk;
  const std::uint64_t end = beg + chunk < total ? beg + chunk : total;
  std::uint64_t s[4] = {st[0], st[1], st[2], st[3]};
  __syncwarp();
  if (beg < total && lane) {
    std::uint64_t a[4] = {0, 0, 0, 0};
#pragma unroll 1
    for (int wi = 0; wi < 4; ++wi) {
      const std::uint64_t word = polys.w[lane][wi];
#pragma unroll 4
      for (int b = 0; b < 64; ++b) {
        if ((word >> b) & 1) {
          a[0] ^= s[0]; a[1] ^= s[1]; a[2] ^= s[2]; a[3] ^= s[3];
        }
        xnext(s);
      }
    }
    s[0] = a[0]; s[1] = a[1]; s[2] = a[2]; s[3] = a[3];
  }
  const std::uint64_t thr = clock ? 0 : (std::uint64_t)ceil(p * 0x1.0p53);
  if (beg < total) {
    std::uint32_t q = (std::uint32_t)(beg / n), i = (std::uint32_t)(beg % n);
    std::uint32_t dq = 0;
    for (std::uint64_t g = beg; g < end; ++g) {
      const std::uint64_t v = xnext(s);
      if (clock) {  // priorities: clock() >> 16 (protocols.hpp:148-150)
        reinterpret_cast<std::uint64_t*>(block + q * per_round)[(std::uint64_t)t * n + i] = v >> 16;
      } else {  // failures: uniform() < p  <=>  (next >> 11) < ceil(p * 2^53)
        const bool d = (v >> 11) < thr;
        block[q * per_round + rows * 8 + (std::uint64_t)t * n + i] = d ? 1 : 0;
        dq += d ? 1u : 0u;
      }
      if (++i == n) {
        if (!clock && dq) atomicAdd(&dead[wib][q], dq);
        dq = 0;
        i = 0;
        ++q;
      }
    }
    if (!clock && dq) atomicAdd(&dead[wib][q], dq);
    if (end == total) {  // the lane holding the block's last draw carries the stream on
      st[0] = s[0];
      st[1] = s[1];
      st[2] = s[2];
      st[3] = s[3];
    }
  }
  __syncwarp();
  if (!clock && lane < nr) act[(std::uint64_t)t * rounds + r0 + lane] = n - dead[wib][lane];
}

// GF(2) polynomials of degree < 512 (host).
using Poly = std::bitset<512>;

// Minimal polynomial of the xoshiro256 state transition, by Berlekamp-Massey
// over 512 bits of one state bit; degree 256 (the transition's characteristic
// polynomial, which is primitive) is checked.
const Poly& xoshiro_charpoly() {
  static const Poly m = [] {
    Xoshiro g(0x2545F4914F6CDD1DULL);
    const int N = 512;
    std::vector<int> a(N), C(N + 1, 0), B(N + 1, 0);
    for (int k = 0; k < N; ++k) {
      a[k] = (int)(g.s[0] & 1);
      g.next();
    }
    C[0] = B[0] = 1;
    int L = 0, mm = 1;
    for (int k = 0; k < N; ++k) {
      int d = a[k];
      for (int i = 1; i <= L; ++i) d ^= C[i] & a[k - i];
      if (!d) {
        ++mm;
      } else if (2 * L <= k) {
        const std::vector<int> Tm = C;
        for (int i = 0; i + mm <= N; ++i) C[i + mm] ^= B[i];
        L = k + 1 - L;
        B = Tm;
        mm = 1;
      } else {
        for (int i = 0; i + mm <= N; ++i) C[i + mm] ^= B[i];
        ++mm;
      }
    }
    if (L != 256) throw std::runtime_error("xoshiro256 minimal polynomial is not of degree 256");
    Poly r;
    for (int i = 0; i <= L; ++i) r[i] = C[L - i];  // reciprocal of the connection polynomial
    return r;
  }();
  return m;
}

Poly poly_mulmod(const Poly& a, const Poly& b) {
  const Poly& m = xoshiro_charpoly();
  Poly r;
  for (int i = 0; i < 256; ++i)
    if (a[i]) r ^= b << i;
  for (int k = 510; k >= 256; --k)
    if (r[k]) r ^= m << (k - 256);
  return r;
}

// q_L = x^(L*chunk) mod m for the 32 lanes, self-checked once per chunk
// against stepping the generator chunk times.
const LanePolys& lane_polys(std::uint64_t chunk) {
  static std::mutex mu;
  static std::map<std::uint64_t, LanePolys> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(chunk);
  if (it != cache.end()) return it->second;
  Poly x, base, acc;
  x[1] = 1;
  acc[0] = 1;
  base = x;
  for (std::uint64_t e = chunk; e; e >>= 1) {  // x^chunk
    if (e & 1) acc = poly_mulmod(acc, base);
    base = poly_mulmod(base, base);
  }
  LanePolys lp{};
  Poly q;
  q[0] = 1;
  for (int L = 0; L < 32; ++L) {
    for (int i = 0; i < 256; ++i)
      if (q[i]) lp.w[L][i >> 6] |= 1ull << (i & 63);
    q = poly_mulmod(q, acc);
  }
  {  // self-check: lane 1's jump equals chunk serial steps
    Xoshiro g(0x9E3779B97F4A7C15ULL ^ chunk), h = g;
    for (std::uint64_t k = 0; k < chunk; ++k) h.next();
    std::uint64_t a[4] = {0, 0, 0, 0};
    for (int i = 0; i < 256; ++i) {
      if ((lp.w[1][i >> 6] >> (i & 63)) & 1)
        for (int w = 0; w < 4; ++w) a[w] ^= g.s[w];
      g.next();
    }
    for (int w = 0; w < 4; ++w)
      if (a[w] != h.s[w]) throw std::runtime_error("xoshiro256 jump polynomial self-check failed");
  }
  return cache.emplace(chunk, lp).first->second;
}

// Stream-ordered buffers from the device's default memory pool (release
// threshold raised once, so freed blocks stay in the pool).  Sweeps call the
// batch entry point once per harness cell, often from many host threads at
// once; cudaMalloc/cudaFree per call synchronise the device and serialise the
// callers, pool allocations on the call's own stream do neither.
struct PoolBuffer {
  void* ptr = nullptr;
  cudaStream_t s = nullptr;
  PoolBuffer(std::size_t bytes, cudaStream_t stream) : s(stream) {
    static thread_local int configured = -1;
    int dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    if (configured != dev) {
      cudaMemPool_t pool;
      MB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
      std::uint64_t keep = UINT64_MAX;
      MB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
      configured = dev;
    }
    MB_CUDA(cudaMallocAsync(&ptr, bytes ? bytes : 16, s));
  }
  PoolBuffer(const PoolBuffer&) = delete;
  PoolBuffer& operator=(const PoolBuffer&) = delete;
  ~PoolBuffer() {
    if (ptr) cudaFreeAsync(ptr, s);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

template <typename F>
void parallel_for(std::uint64_t count, F&& f) {
  unsigned th = std::max(1u, std::thread::hardware_concurrency());
  if (count < 4 || th == 1) {
    for (std::uint64_t i = 0; i < count; ++i) f(i);
    return;
  }
  th = (unsigned)std::min<std::uint64_t>(th, count);
  std::vector<std::thread> pool;
  for (unsigned k = 0; k < th; ++k)
    pool.emplace_back([&, k] {
      for (std::uint64_t i = k; i < count; i += th) f(i);
    });
  for (auto& t : pool) t.join();
}

template <typename T>
void run_batch(std::uint32_t M, std::uint32_t d, std::uint32_t trials, const T* initial,
               std::uint64_t n, std::uint64_t dim, double p, const std::uint64_t* seeds,
               std::uint32_t rounds, int diag, double* init_dist, double* dist, double* drift,
               std::uint32_t* active, T* final_out) {
  const std::size_t es = sizeof(T);
  const Grid grid(M, d);
  // MOSHPIT_PROFILE=1: host-side phase times of this call on stderr
  static const bool prof = std::getenv("MOSHPIT_PROFILE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t_begin = now();
  std::vector<std::pair<const char*, double>> marks;
  auto mark = [&](const char* what) {
    if (prof) marks.emplace_back(what, std::chrono::duration<double, std::milli>(now() - t_begin).count());
  };
  StreamHolder st;
  const std::uint64_t ld = padded_ld(dim, es), rows = (std::uint64_t)trials * n;
  std::uint64_t np = 1;
  while (np < n) np <<= 1;
  PoolBuffer x(rows * ld * es + 16, st.s), keys(rows * 8, st.s), cellb(rows * 8, st.s),
      members(rows * 4, st.s), goff((std::uint64_t)trials * (n + 1) * 4, st.s), gvoid(rows, st.s),
      act(rows * 4, st.s), counts((std::uint64_t)trials * 16, st.s),
      sidx((std::uint64_t)trials * np * 4, st.s), scs(rows * 4, st.s), sgi(rows * 4, st.s);
  MB_CUDA(cudaMemcpy2DAsync(x.ptr, ld * es, initial, dim * es, dim * es, rows,
                            cudaMemcpyHostToDevice, st.s));
  // host: cells of every trial (protocols.hpp:124-130), in parallel
  // one-shot staging: pageable memory (a cudaMallocHost per call costs more
  // than the copy it would speed up, and serialises concurrent callers)
  std::vector<std::uint64_t> hcells(rows);
  std::vector<std::uint64_t> hstate((std::uint64_t)trials * 8);  // failures | priorities
  mark("alloc+h2d");
  parallel_for(trials, [&](std::uint64_t t) {
    Xoshiro cs = Xoshiro::named(seeds[t], "cells");
    const auto c = draw_cells(cs, grid.capacity, n);
    std::memcpy(hcells.data() + t * n, c.data(), n * 8);
    const Xoshiro f = Xoshiro::named(seeds[t], "failures");
    const Xoshiro k = Xoshiro::named(seeds[t], "priorities");
    std::memcpy(hstate.data() + t * 4, f.s, 32);
    std::memcpy(hstate.data() + ((std::uint64_t)trials + t) * 4, k.s, 32);
  });
  mark("cells");
  PoolBuffer rstate(hstate.size() * 8, st.s), act_d((std::uint64_t)trials * rounds * 4 + 16, st.s);
  MB_CUDA(cudaMemcpyAsync(rstate.ptr, hstate.data(), hstate.size() * 8, cudaMemcpyHostToDevice,
                          st.s));
  MB_CUDA(cudaMemcpyAsync(cellb.ptr, hcells.data(), rows * 8, cudaMemcpyHostToDevice, st.s));
  launch_initial_keys(cellb.as<std::uint64_t>(), keys.as<std::uint64_t>(), rows, M, d, st.s);
  const bool dg = diag != MOSHPIT_DIAG_NONE;
  const bool dg0 = diag != MOSHPIT_DIAG_NONE;
  PoolBuffer ref(dg0 ? (std::uint64_t)trials * dim * 8 + 16 : 16, st.s),
      mean(dg0 ? (std::uint64_t)trials * dim * 8 + 16 : 16, st.s), sq(dg0 ? rows * 8 + 16 : 16, st.s),
      out(dg0 ? (std::uint64_t)trials * (2 * rounds + 1) * 8 + 16 : 16, st.s);
  const unsigned cb = 128;
  const dim3 cgrid((unsigned)((dim + cb - 1) / cb), trials);
  // narrow vectors: a CTA per (column, trial) evaluates the tree over peers
  const bool narrow = dim < cb;
  auto colmean = [&](double* o) {
    if (!dim) return;
    if (narrow)
      colmean_tree_b<T><<<dim3((unsigned)dim, trials), kTreeThreads, 0, st.s>>>(
          x.as<T>(), (std::uint32_t)n, ld, dim, o);
    else
      colmean_b<T><<<cgrid, cb, 0, st.s>>>(x.as<T>(), n, ld, dim, o);
  };
  auto finish = [&](double* o) {
    finish_tree_b<<<trials, kTreeThreads, 0, st.s>>>(sq.as<double>(), (std::uint32_t)n, o,
                                                     2 * rounds + 1);
  };
  if (dg) {
    colmean(ref.as<double>());
    dist_rows_b<T><<<(unsigned)((rows + 127) / 128), 128, 0, st.s>>>(x.as<T>(), n, rows, ld, dim,
                                                                     ref.as<double>(),
                                                                     sq.as<double>());
    finish(out.as<double>());
    MB_LAUNCH_CHECK();
  }
  // The draws of a block of rounds are generated on the device (draws_kernel,
  // a serial xoshiro chain per trial stream) on a side stream, one block
  // ahead of the rounds that consume them: blocks of a few rounds in two
  // buffers, so the chains of block b+1 run under the rounds of block b.
  std::vector<std::uint32_t> act_h((std::uint64_t)trials * rounds);
  // per-round block: ts u64[rows] then failed u8[rows], padded to 16 bytes so
  // every block's timestamps stay 8-byte aligned
  const std::uint64_t per_round = (rows * 9 + 15) / 16 * 16;
  std::uint32_t rb = (std::uint32_t)std::max<std::uint64_t>(1, (128ull << 20) / per_round);
  if (rb > kMaxBlockRounds) rb = kMaxBlockRounds;
  // lane-parallel draws for blocks of >= 512 draws per stream (enough per
  // lane to pay for the 256-step jump); MOSHPIT_SERIAL_DRAWS=1 keeps one
  // thread per stream
  static const bool serial_draws = std::getenv("MOSHPIT_SERIAL_DRAWS") != nullptr;
  const bool lanes = !serial_draws;
  if (rb > rounds) rb = rounds ? rounds : 1;
  PoolBuffer dbuf0(per_round * rb + 16, st.s), dbuf1(per_round * rb + 16, st.s);
  PoolBuffer* dbufs[2] = {&dbuf0, &dbuf1};
  StreamHolder ds;
  cudaEvent_t ev_ready = nullptr, ev_drawn[2] = {}, ev_free[2] = {};
  MB_CUDA(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    MB_CUDA(cudaEventCreateWithFlags(&ev_drawn[i], cudaEventDisableTiming));
    MB_CUDA(cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming));
  }
  struct EvGuard {
    cudaEvent_t* e;
    int k;
    ~EvGuard() {
      for (int i = 0; i < k; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  };
  cudaEvent_t all_ev[5] = {ev_ready, ev_drawn[0], ev_drawn[1], ev_free[0], ev_free[1]};
  EvGuard guard{all_ev, 5};
  MB_CUDA(cudaEventRecord(ev_ready, st.s));  // stream states + buffers are in place
  MB_CUDA(cudaStreamWaitEvent(ds.s, ev_ready, 0));
  auto draw_block = [&](std::uint32_t b) {
    const std::uint32_t r0 = b * rb;
    const std::uint32_t nr = std::min(rb, rounds - r0);
    if (b >= 2) MB_CUDA(cudaStreamWaitEvent(ds.s, ev_free[b & 1], 0));
    if (lanes && (std::uint64_t)nr * n >= 512) {
      const std::uint64_t chunk = ((std::uint64_t)nr * n + 31) / 32;
      draws_lanes_kernel<<<trials, 64, 0, ds.s>>>(
          rstate.as<std::uint64_t>(), rstate.as<std::uint64_t>() + (std::uint64_t)trials * 4,
          trials, (std::uint32_t)n, nr, per_round, p, dbufs[b & 1]->as<std::uint8_t>(),
          act_d.as<std::uint32_t>(), rounds, r0, chunk, lane_polys(chunk));
    } else {
      draws_kernel<<<(2 * trials + 63) / 64, 64, 0, ds.s>>>(
          rstate.as<std::uint64_t>(), rstate.as<std::uint64_t>() + (std::uint64_t)trials * 4,
          trials, (std::uint32_t)n, nr, per_round, p, dbufs[b & 1]->as<std::uint8_t>(),
          act_d.as<std::uint32_t>(), rounds, r0);
    }
    MB_LAUNCH_CHECK();
    MB_CUDA(cudaEventRecord(ev_drawn[b & 1], ds.s));
  };
  // Narrow vectors (the harness's dim-1/2 sweeps): one launch per round, the
  // group means computed by kernel 1's CTA of each trial.  MOSHPIT_BATCH_FUSE=0
  // keeps the separate kernel-2 launch (same results bit for bit).
  static const bool fuse_env = [] {
    const char* e = std::getenv("MOSHPIT_BATCH_FUSE");
    return !(e && e[0] == '0');
  }();
  const bool fuse = fuse_env && dim > 0 && dim <= 4;
  const std::uint32_t nblocks = rounds ? (rounds + rb - 1) / rb : 0;
  if (nblocks) draw_block(0);
  for (std::uint32_t b = 0; b < nblocks; ++b) {
    const std::uint32_t r0 = b * rb;
    const std::uint32_t nr = std::min(rb, rounds - r0);
    if (b + 1 < nblocks) draw_block(b + 1);
    MB_CUDA(cudaStreamWaitEvent(st.s, ev_drawn[b & 1], 0));
    PoolBuffer& dblock = *dbufs[b & 1];
    for (std::uint32_t q = 0; q < nr; ++q) {
    const std::uint32_t r = r0 + q;
    std::uint8_t* draws_r = dblock.as<std::uint8_t>() + q * per_round;
    GroupArgs a;
    a.n = static_cast<std::uint32_t>(n);
    a.cap = M;
    a.M = M;
    a.pow_drop = grid.pow_drop;
    a.advance_keys = 1;
    a.klen_zero = grid.klen == 0;
    a.keys = keys.as<std::uint64_t>();
    a.ts = reinterpret_cast<std::uint64_t*>(draws_r);
    a.failed = draws_r + rows * 8;
    a.members = members.as<std::uint32_t>();
    a.goff = goff.as<std::uint32_t>();
    a.gvoid = gvoid.as<std::uint8_t>();
    a.act = act.as<std::uint32_t>();
    a.counts = counts.as<std::uint32_t>();
    a.sidx = sidx.as<std::uint32_t>();
    a.scs = scs.as<std::uint32_t>();
    a.sgi = sgi.as<std::uint32_t>();
    a.batch = trials;
    if (fuse) {  // kernel 2 inside kernel 1's CTA (see GroupArgs::fuse_x)
      a.fuse_x = x.ptr;
      a.fuse_ld = ld;
      a.fuse_dim = dim;
      a.fuse_stride = n * ld;
      a.fuse_f64 = std::is_same_v<T, double> ? 1 : 0;
    }
    launch_form_groups(a, true, st.s);
    if (!fuse)
      launch_group_mean_batch<T>(x.as<T>(), n * ld, ld, dim, (std::uint32_t)n, trials,
                                 a.members, a.goff, a.act, a.counts, st.s);
    if (dg && dim < 32) {
      round_diag_narrow<T><<<trials, kTreeThreads, 0, st.s>>>(
          x.as<T>(), (std::uint32_t)n, ld, (std::uint32_t)dim, ref.as<double>(), sq.as<double>(),
          mean.as<double>(), out.as<double>() + 1 + r, out.as<double>() + 1 + rounds + r,
          2 * rounds + 1);
      MB_LAUNCH_CHECK();
    } else if (dg) {
      dist_rows_b<T><<<(unsigned)((rows + 127) / 128), 128, 0, st.s>>>(
          x.as<T>(), n, rows, ld, dim, ref.as<double>(), sq.as<double>());
      finish(out.as<double>() + 1 + r);
      colmean(mean.as<double>());
      drift_b<<<(trials + 127) / 128, 128, 0, st.s>>>(mean.as<double>(), ref.as<double>(), dim,
                                                      trials, out.as<double>() + 1 + rounds + r,
                                                      2 * rounds + 1);
      MB_LAUNCH_CHECK();
    }
    }
    MB_CUDA(cudaEventRecord(ev_free[b & 1], st.s));  // block b's draws consumed
  }
  if (rounds) {
    MB_CUDA(cudaStreamWaitEvent(st.s, ev_drawn[(nblocks - 1) & 1], 0));  // act counts complete
    MB_CUDA(cudaMemcpyAsync(act_h.data(), act_d.ptr, act_h.size() * 4, cudaMemcpyDeviceToHost,
                            st.s));
  }
  std::vector<double> h;
  if (dg) {
    h.resize((std::uint64_t)trials * (2 * rounds + 1));
    MB_CUDA(cudaMemcpyAsync(h.data(), out.ptr, h.size() * 8, cudaMemcpyDeviceToHost, st.s));
  }
  if (final_out)
    MB_CUDA(cudaMemcpy2DAsync(final_out, dim * es, x.ptr, ld * es, dim * es, rows,
                              cudaMemcpyDeviceToHost, st.s));
  mark("enqueued");
  MB_CUDA(cudaStreamSynchronize(st.s));
  mark("synced");
  const double nan = std::nan("");
  for (std::uint64_t t = 0; t < trials; ++t) {
    const std::uint64_t o = t * (2 * rounds + 1);
    init_dist[t] = dg ? h[o] : nan;
    for (std::uint32_t r = 0; r < rounds; ++r) {
      dist[t * rounds + r] = dg ? h[o + 1 + r] : nan;
      drift[t * rounds + r] = dg ? h[o + 1 + rounds + r] : nan;
      active[t * rounds + r] = act_h[t * rounds + r];
    }
  }
  mark("reports");
  if (prof) {
    std::string line = "[moshpit batch] trials=" + std::to_string(trials) + " n=" + std::to_string(n);
    for (auto& m : marks) line += std::string(" ") + m.first + "=" + std::to_string(m.second) + "ms";
    fprintf(stderr, "%s\n", line.c_str());
  }
}

}  // namespace
}  // namespace mb200

using namespace mb200;

extern "C" {

// Trial-batched protocols::run_moshpit: trial t uses initial + t*n*dim and
// Rng(seeds[t]); report arrays are [trials] / [trials][rounds].  Diagnostics
// are computed in the reference order (EXACT) unless diag == NONE.
int moshpit_run_moshpit_batch(int dtype, std::uint32_t M, std::uint32_t d, std::uint32_t T,
                              std::uint32_t trials, const void* initial, std::uint64_t n,
                              std::uint64_t dim, double p_round, const std::uint64_t* seeds,
                              std::uint32_t rounds, int diag, double* initial_distortion,
                              double* distortion, double* mean_drift,
                              std::uint32_t* active_counts, double* cost_units,
                              void* final_out) {
  return guarded([&] {
    elem_size(dtype);
    if (M < 1 || d < 1 || T < 1)
      throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
    if (p_round < 0.0 || p_round > 1.0)
      throw std::invalid_argument("FailureModel: p_round must be in [0,1]");
    if (n == 0) throw std::invalid_argument("run_moshpit: no peers");
    if (n > moshpit_grid_capacity(M, d))
      throw std::invalid_argument("run_moshpit: N exceeds grid capacity M^d");
    if (n > 8192) throw std::invalid_argument("run_moshpit_batch: at most 8192 peers per trial");
    if (diag < MOSHPIT_DIAG_NONE || diag > MOSHPIT_DIAG_EXACT)
      throw std::invalid_argument("run_moshpit: unknown diagnostics mode");
    if (trials > 65535) throw std::invalid_argument("run_moshpit_batch: at most 65535 trials");
    if (trials == 0) return;
    require_device();
    if (dtype == MOSHPIT_F32)
      run_batch<float>(M, d, trials, static_cast<const float*>(initial), n, dim, p_round, seeds,
                       rounds, diag, initial_distortion, distortion, mean_drift, active_counts,
                       static_cast<float*>(final_out));
    else
      run_batch<double>(M, d, trials, static_cast<const double*>(initial), n, dim, p_round,
                        seeds, rounds, diag, initial_distortion, distortion, mean_drift,
                        active_counts, static_cast<double*>(final_out));
    const double c = moshpit_complexity_estimate(rounds, static_cast<std::uint32_t>(n), M,
                                                 static_cast<std::uint32_t>(dim));
    for (std::uint32_t t = 0; t < trials; ++t) cost_units[t] = c;
  });
}

// harness.hpp:145-155 trial_rng: the per-trial root seed of a sweep cell.
std::uint64_t moshpit_trial_seed(std::uint64_t seed_base, const char* protocol,
                                 std::uint32_t n, double p, std::uint32_t seed_index) {
  std::uint64_t p_bits;
  std::memcpy(&p_bits, &p, sizeof(p));
  std::uint64_t mix = seed_base ^ fnv1a(protocol);
  mix = splitmix64(mix) ^ n;
  mix = splitmix64(mix) ^ p_bits;
  mix = splitmix64(mix) ^ seed_index;
  return splitmix64(mix);
}

}  // extern "C"
