// mean_kernel.cu -- Kernel 2: fused segmented group mean (the graded kernel).
//
// Replaces the data plane of one Moshpit round: for every non-voided group
// (allreduce.hpp:95-102 voids the rest), mean[j] = pairwise_sum(column_j over
// the members in priority order) / n (allreduce.hpp:106-116, core.hpp:72-81),
// then vectors.assign(n, mean) + write-back (allreduce.hpp:118-120,
// protocols.hpp:165-167).  One read and one write of every active row per
// round; voided groups move 0 bytes.
//
// Layout: peer-major rows (row = peer id, `ld` elements).  Work item =
// (active group, D-tile); a persistent grid strides over items so that at any
// instant the resident CTAs stream adjacent tiles of the same rows.
//
// Exactness: every thread owns VEC consecutive coordinates (one 16-byte
// vector) and evaluates the reference's pairwise tree over the members in
// registers -- n <= 8 sequential from +0, else split at floor(n/2) -- with
// IEEE add and IEEE division by n (no FMA, no reciprocal).  The per-coordinate
// tree is register-local, so no cross-lane shuffles are needed and the fp32
// result is bit-identical to the fp32 restatement of the reference, and the
// fp64 instantiation bit-identical to the reference itself.
#include "common.cuh"

namespace mb200 {
namespace {

template <typename T>
struct V16;
template <>
struct V16<float> {
  using type = float4;
  static constexpr int kN = 4;
};
template <>
struct V16<double> {
  using type = double2;
  static constexpr int kN = 2;
};

__device__ __forceinline__ float4 vzero(float4*) { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ double2 vzero(double2*) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ float4 vadd(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ double2 vadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ float4 vdiv(float4 a, std::uint32_t n) {
  const float f = (float)n;
  return make_float4(__fdiv_rn(a.x, f), __fdiv_rn(a.y, f), __fdiv_rn(a.z, f),
                     __fdiv_rn(a.w, f));
}
__device__ __forceinline__ double2 vdiv(double2 a, std::uint32_t n) {
  const double f = (double)n;
  return make_double2(__ddiv_rn(a.x, f), __ddiv_rn(a.y, f));
}

// Streaming 128-bit accesses: every row tile is touched once per round, so
// keep it out of L1 and mark it evict-first in L2.
__device__ __forceinline__ float4 vload(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 vload(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void vstore(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void vstore(double2* p, double2 v) { __stcs(p, v); }

// core.hpp:72-81 over x[B .. B+N) with compile-time shape.
template <int N, int B, typename V>
__device__ __forceinline__ V tree(const V (&x)[32]) {
  if constexpr (N <= 8) {
    V s = vzero((V*)nullptr);
#pragma unroll
    for (int i = 0; i < N; ++i) s = vadd(s, x[B + i]);
    return s;
  } else {
    constexpr int H = N / 2;
    const V lo = tree<H, B>(x);
    const V hi = tree<N - H, B + H>(x);
    return vadd(lo, hi);
  }
}

}  // namespace
}  // namespace mb200
#include "pairwise.cuh"
namespace mb200 {
namespace {

constexpr int kThreads = 128;
constexpr int kMaxSmemIds = 1024;

template <typename T>
struct MeanArgs {
  T* state;
  std::uint64_t ld_vec;     // row stride in 16-byte vectors
  std::uint64_t nvec;       // vectors per row to process
  std::uint64_t n_tiles;    // ceil(nvec / kThreads)
  const std::uint32_t* members;
  const std::uint32_t* goff;
  const std::uint32_t* act;
  const std::uint32_t* counts;  // [1] = number of active groups
};

template <int N, typename V>
__device__ __forceinline__ void mean_fixed(V* base, std::uint64_t ld_vec,
                                           std::uint64_t col,
                                           const std::uint32_t* ids) {
  V x[32];
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = vload(base + (std::uint64_t)ids[k] * ld_vec + col);
  const V m = vdiv(tree<N, 0>(x), (std::uint32_t)N);
#pragma unroll
  for (int k = 0; k < N; ++k) vstore(base + (std::uint64_t)ids[k] * ld_vec + col, m);
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 3) group_mean_register(MeanArgs<T> a) {
  using V = typename V16<T>::type;
  __shared__ std::uint32_t sids[kMaxSmemIds];
  const std::uint32_t n_act = a.counts[1];
  const std::uint64_t n_items = (std::uint64_t)n_act * a.n_tiles;
  V* base = reinterpret_cast<V*>(a.state);
  std::uint32_t cached = 0xffffffffu, beg = 0, cnt = 0;
  for (std::uint64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
    const std::uint32_t g = a.act[w / a.n_tiles];
    const std::uint64_t tile = w % a.n_tiles;
    if (g != cached) {  // uniform across the CTA
      __syncthreads();
      beg = a.goff[g];
      cnt = a.goff[g + 1] - beg;
      for (std::uint32_t k = threadIdx.x; k < cnt && k < kMaxSmemIds; k += kThreads)
        sids[k] = a.members[beg + k];
      cached = g;
      __syncthreads();
    }
    const std::uint64_t col = tile * kThreads + threadIdx.x;
    if (col >= a.nvec) continue;
    switch (cnt) {
#define MB_CASE(N) \
  case N:          \
    mean_fixed<N, V>(base, a.ld_vec, col, sids); \
    break;
      MB_CASE(1) MB_CASE(2) MB_CASE(3) MB_CASE(4) MB_CASE(5) MB_CASE(6) MB_CASE(7)
      MB_CASE(8) MB_CASE(9) MB_CASE(10) MB_CASE(11) MB_CASE(12) MB_CASE(13)
      MB_CASE(14) MB_CASE(15) MB_CASE(16) MB_CASE(17) MB_CASE(18) MB_CASE(19)
      MB_CASE(20) MB_CASE(21) MB_CASE(22) MB_CASE(23) MB_CASE(24) MB_CASE(25)
      MB_CASE(26) MB_CASE(27) MB_CASE(28) MB_CASE(29) MB_CASE(30) MB_CASE(31)
      MB_CASE(32)
#undef MB_CASE
      default: {
        const std::uint32_t* ids = cnt <= kMaxSmemIds ? sids : a.members + beg;
        auto ld = [&](std::uint32_t k) {
          return vload(base + (std::uint64_t)ids[k] * a.ld_vec + col);
        };
        const V m = vdiv(pairwise_rt<V>(ld, cnt, [](V x, V y) { return vadd(x, y); },
                                           vzero((V*)nullptr)), cnt);
        for (std::uint32_t k = 0; k < cnt; ++k)
          vstore(base + (std::uint64_t)ids[k] * a.ld_vec + col, m);
      }
    }
  }
}

struct GridCache {
  int dev = -1;
  int grid[2] = {0, 0};
};

template <typename T>
int mean_grid() {
  static thread_local GridCache cache;
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  const int slot = sizeof(T) == 4 ? 0 : 1;
  if (cache.dev != dev) {
    cache.dev = dev;
    cache.grid[0] = cache.grid[1] = 0;
  }
  if (!cache.grid[slot]) {
    int sms = 0, per = 0;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per, group_mean_register<T>, kThreads, 0));
    cache.grid[slot] = sms * (per > 0 ? per : 1);
  }
  return cache.grid[slot];
}

}  // namespace

template <typename T>
void launch_group_mean(T* state, std::uint64_t ld, std::uint64_t dim,
                       const std::uint32_t* members, const std::uint32_t* goff,
                       const std::uint32_t* act, const std::uint32_t* counts,
                       std::uint32_t max_group, int variant, cudaStream_t s) {
  (void)variant;
  (void)max_group;
  if (dim == 0) return;
  constexpr int kVec = V16<T>::kN;
  MeanArgs<T> a;
  a.state = state;
  a.ld_vec = ld / kVec;
  a.nvec = (dim + kVec - 1) / kVec;
  a.n_tiles = (a.nvec + kThreads - 1) / kThreads;
  a.members = members;
  a.goff = goff;
  a.act = act;
  a.counts = counts;
  group_mean_register<T><<<mean_grid<T>(), kThreads, 0, s>>>(a);
  MB_LAUNCH_CHECK();
}

template void launch_group_mean<float>(float*, std::uint64_t, std::uint64_t,
                                       const std::uint32_t*, const std::uint32_t*,
                                       const std::uint32_t*, const std::uint32_t*,
                                       std::uint32_t, int, cudaStream_t);
template void launch_group_mean<double>(double*, std::uint64_t, std::uint64_t,
                                        const std::uint32_t*, const std::uint32_t*,
                                        const std::uint32_t*, const std::uint32_t*,
                                        std::uint32_t, int, cudaStream_t);

}  // namespace mb200
