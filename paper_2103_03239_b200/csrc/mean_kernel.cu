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
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "philox.cuh"

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

// Plain 128-bit LDG/STG.  Measured on B200 (profiles/k2_variants.cu): with one
// CTA per SM the default cache policy beats the streaming (.cs) and .nc hints
// by ~2-5 % on this access pattern.
__device__ __forceinline__ float4 vload(const float4* p) { return *p; }
__device__ __forceinline__ double2 vload(const double2* p) { return *p; }
__device__ __forceinline__ void vstore(float4* p, float4 v) { *p = v; }
__device__ __forceinline__ void vstore(double2* p, double2 v) { *p = v; }

// core.hpp:72-81 over x[B .. B+N) with compile-time shape.
template <int N, int B, typename V, int S>
__device__ __forceinline__ V tree(const V (&x)[S]) {
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

__device__ __forceinline__ float4 vshfl_xor16(float4 v) {
  return make_float4(__shfl_xor_sync(0xffffffffu, v.x, 16), __shfl_xor_sync(0xffffffffu, v.y, 16),
                     __shfl_xor_sync(0xffffffffu, v.z, 16), __shfl_xor_sync(0xffffffffu, v.w, 16));
}
__device__ __forceinline__ double2 vshfl_xor16(double2 v) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 16),
                      __shfl_xor_sync(0xffffffffu, v.y, 16));
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
  StepPrologue<T> step;     // kernel 3: local SGD step fused into the loads
  T* state;
  std::uint64_t ld_vec;     // row stride in 16-byte vectors
  std::uint64_t nvec;       // vectors per row to process
  std::uint64_t n_tiles;    // ceil(nvec / kThreads)
  const std::uint32_t* members;
  const std::uint32_t* goff;
  const std::uint32_t* act;
  const std::uint32_t* counts;  // [1] = number of active groups
  std::uint64_t batch_state_stride;  // trial batching: state elements per trial
  std::uint32_t batch_n;             // peers per trial (0: no batching)
};

// Kernel 3 prologue (optimizer.hpp:356-373): g = c*(theta-t) [+ nj]; the
// non-finite check is on g; theta' = theta - gamma*g.  Same rounding and the
// same Philox noise per (step, peer, coordinate) as the standalone step kernel
// (sgd.cu), so fused == unfused bit for bit.
__device__ __forceinline__ float sgd_grad(float x, float c, float t, float nj, bool noisy) {
  float g = __fmul_rn(c, __fsub_rn(x, t));
  return noisy ? __fadd_rn(g, nj) : g;
}
__device__ __forceinline__ double sgd_grad(double x, double c, double t, double nj, bool noisy) {
  double g = __dmul_rn(c, __dsub_rn(x, t));
  return noisy ? __dadd_rn(g, nj) : g;
}
__device__ __forceinline__ float sgd_update(float x, float gm, float g) {
  return __fsub_rn(x, __fmul_rn(gm, g));
}
__device__ __forceinline__ double sgd_update(double x, double gm, double g) {
  return __dsub_rn(x, __dmul_rn(gm, g));
}

template <typename T, typename V>
__device__ __forceinline__ V apply_step(const StepPrologue<T>& sp, V v, std::uint32_t peer,
                                        std::uint64_t col, const V& c, const V& t, double& nsq,
                                        bool& bad) {
  constexpr int kV = sizeof(V) / sizeof(T);
  T* pv = reinterpret_cast<T*>(&v);
  const T* pc = reinterpret_cast<const T*>(&c);
  const T* pt = reinterpret_cast<const T*>(&t);
  const std::uint64_t j0 = col * kV;
  float z[4] = {0, 0, 0, 0};
  const bool noisy = sp.philox != 0;
  if (noisy) philox_normals4(sp.seed, sp.step_no, peer, j0 / 4, z);
  T q = T(0);
#pragma unroll
  for (int u = 0; u < kV; ++u) {
    const std::uint64_t j = j0 + u;
    if (j >= sp.dim) break;
    const T nj = noisy ? noise_component(z[j % 4], sp.coord_std, (T*)nullptr) : T(0);
    if (noisy) nsq_add(q, nj);
    const T g = sgd_grad(pv[u], pc[u], pt[u], nj, noisy);
    bad |= !isfinite(g);
    pv[u] = sgd_update(pv[u], sp.gamma, g);
  }
  if (noisy) nsq += (double)q;
  return v;
}

template <int N, bool STEP, typename T, typename V>
__device__ __forceinline__ void mean_fixed(V* base, std::uint64_t ld_vec,
                                           std::uint64_t col,
                                           const std::uint32_t* ids,
                                           const StepPrologue<T>& sp, double& nsq, bool& bad) {
  V x[32];
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = vload(base + (std::uint64_t)ids[k] * ld_vec + col);
  if constexpr (STEP) {
    // curvature / target of this column: loaded once per item, not per member
    const V c = __ldg(reinterpret_cast<const V*>(sp.curv) + col);
    const V t = __ldg(reinterpret_cast<const V*>(sp.tgt) + col);
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = apply_step(sp, x[k], ids[k], col, c, t, nsq, bad);
  }
  const V m = vdiv(tree<N, 0>(x), (std::uint32_t)N);
#pragma unroll
  for (int k = 0; k < N; ++k) vstore(base + (std::uint64_t)ids[k] * ld_vec + col, m);
}

template <typename T, bool STEP>
__global__ void __launch_bounds__(kThreads, 3) group_mean_register(MeanArgs<T> a) {
  using V = typename V16<T>::type;
  double nsq = 0.0;
  bool bad = false;
  if (a.batch_n) {  // trial = blockIdx.y
    const std::uint64_t t = blockIdx.y, n = a.batch_n;
    a.state += t * a.batch_state_stride;
    a.members += t * n;
    a.goff += t * (n + 1);
    a.act += t * n;
    a.counts += t * 4;
  }
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
    // with the step fused (groups > 32 only: kernel 3 takes the rest) just
    // the generic tree -- no 32 specialised step bodies in the binary
    switch (STEP ? 0u : cnt) {
#define MB_CASE(N) \
  case N:          \
    mean_fixed<N, STEP, T, V>(base, a.ld_vec, col, sids, a.step, nsq, bad); \
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
          V v = vload(base + (std::uint64_t)ids[k] * a.ld_vec + col);
          if constexpr (STEP)
            v = apply_step(a.step, v, ids[k], col,
                           __ldg(reinterpret_cast<const V*>(a.step.curv) + col),
                           __ldg(reinterpret_cast<const V*>(a.step.tgt) + col), nsq, bad);
          return v;
        };
        const V m = vdiv(pairwise_rt<V>(ld, cnt, [](V x, V y) { return vadd(x, y); },
                                           vzero((V*)nullptr)), cnt);
        for (std::uint32_t k = 0; k < cnt; ++k)
          vstore(base + (std::uint64_t)ids[k] * a.ld_vec + col, m);
      }
    }
  }
  if constexpr (STEP) {
    __shared__ double red[kThreads];
    red[threadIdx.x] = nsq;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0 && a.step.noise_partial) a.step.noise_partial[blockIdx.x] = red[0];
    if (bad) atomicOr(a.step.nonfinite, 1u);
  }
}

// ---------------------------------------------------------------------------
// Bulk (TMA) variant: one producer warp streams every member-row tile of an
// item into a shared-memory ring with cp.async.bulk (global -> shared, mbarrier
// complete_tx, L2 evict-first), consumer warps evaluate the same register tree
// from shared memory and store the mean with 128-bit streaming stores.  One
// CTA per SM; the ring keeps `stages` items (up to ~190 KB) of loads in flight.
// ---------------------------------------------------------------------------
__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ std::uint64_t evict_first_policy() {
  std::uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes,
                                         std::uint64_t* bar, std::uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

constexpr int kBulkTileVec = 128;  // 16-byte vectors per row tile (2 KB)
constexpr int kBulkConsumerWarps = kBulkTileVec / 32;
constexpr int kBulkThreads = kBulkTileVec + 32;
constexpr int kBulkMaxRows = 32;

struct BulkHdr {
  std::uint32_t ids[kBulkMaxRows];
  std::uint32_t n;
  std::uint32_t nv;
  std::uint64_t col;
};

template <int N, typename V>
__device__ __forceinline__ void mean_fixed_smem(const V* in, V* base, std::uint64_t ld_vec,
                                                std::uint64_t col, const std::uint32_t* ids) {
  V x[32];
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = in[k * kBulkTileVec];
  const V m = vdiv(tree<N, 0>(x), (std::uint32_t)N);
#pragma unroll
  for (int k = 0; k < N; ++k) vstore(base + (std::uint64_t)ids[k] * ld_vec + col, m);
}

template <typename T>
__global__ void __launch_bounds__(kBulkThreads, 1)
    group_mean_bulk(MeanArgs<T> a, int stages, int srows) {
  using V = typename V16<T>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  V* data = reinterpret_cast<V*>(smem);
  BulkHdr* hdr = reinterpret_cast<BulkHdr*>(data + (std::size_t)stages * srows * kBulkTileVec);
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(hdr + stages);
  std::uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBulkConsumerWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const std::uint32_t n_act = a.counts[1];
  const std::uint64_t n_items = (std::uint64_t)n_act * a.n_tiles;
  V* base = reinterpret_cast<V*>(a.state);
  int s = 0;
  std::uint32_t ph = 0;
  if (warp == kBulkConsumerWarps) {
    // Producer warp: lane k owns member row k of the current group (ids
    // cached in registers across the items of one group) and issues its own
    // bulk copy; lane 0 arms the stage's full barrier first.
    const std::uint64_t pol = evict_first_policy();
    std::uint32_t cached = 0xffffffffu, n = 0, my_id = 0;
    for (std::uint64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const std::uint32_t g = a.act[w / a.n_tiles];
      if (g != cached) {
        const std::uint32_t beg = a.goff[g];
        n = a.goff[g + 1] - beg;
        my_id = (std::uint32_t)lane < n ? a.members[beg + lane] : 0u;
        cached = g;
      }
      const std::uint64_t col = (w % a.n_tiles) * kBulkTileVec;
      const std::uint64_t left = a.nvec - col;
      const std::uint32_t nv = left < (std::uint64_t)kBulkTileVec ? (std::uint32_t)left
                                                                  : (std::uint32_t)kBulkTileVec;
      if (lane == 0) mbar_wait(&empty[s], ph ^ 1);
      __syncwarp();
      BulkHdr& h = hdr[s];
      if ((std::uint32_t)lane < n) h.ids[lane] = my_id;
      if (lane == 0) {
        h.n = n;
        h.nv = nv;
        h.col = col;
        mbar_arrive_expect_tx(&full[s], n * nv * 16u);
      }
      __syncwarp();
      if ((std::uint32_t)lane < n)
        bulk_g2s(data + ((std::size_t)s * srows + lane) * kBulkTileVec,
                 base + (std::uint64_t)my_id * a.ld_vec + col, nv * 16u, &full[s], pol);
      if (++s == stages) {
        s = 0;
        ph ^= 1;
      }
    }
    return;
  }
  const int t = threadIdx.x;  // consumer: one 16-byte column of the tile
  for (std::uint64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
    mbar_wait(&full[s], ph);
    const BulkHdr& h = hdr[s];
    const std::uint32_t n = h.n;
    if ((std::uint32_t)t < h.nv) {
      const V* in = data + (std::size_t)s * srows * kBulkTileVec + t;
      const std::uint64_t col = h.col + t;
      switch (n) {
#define MB_BCASE(N) \
  case N:           \
    mean_fixed_smem<N, V>(in, base, a.ld_vec, col, h.ids); \
    break;
        MB_BCASE(1) MB_BCASE(2) MB_BCASE(3) MB_BCASE(4) MB_BCASE(5) MB_BCASE(6) MB_BCASE(7)
        MB_BCASE(8) MB_BCASE(9) MB_BCASE(10) MB_BCASE(11) MB_BCASE(12) MB_BCASE(13)
        MB_BCASE(14) MB_BCASE(15) MB_BCASE(16) MB_BCASE(17) MB_BCASE(18) MB_BCASE(19)
        MB_BCASE(20) MB_BCASE(21) MB_BCASE(22) MB_BCASE(23) MB_BCASE(24) MB_BCASE(25)
        MB_BCASE(26) MB_BCASE(27) MB_BCASE(28) MB_BCASE(29) MB_BCASE(30) MB_BCASE(31)
        MB_BCASE(32)
#undef MB_BCASE
        default: break;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == stages) {
      s = 0;
      ph ^= 1;
    }
  }
}

// Grid cap (in SMs' worth of CTAs) for kernel 2 launched from this thread; 0 =
// every SM.  The peer-sharded slab pipeline lowers it while a cross round of
// another slab shares the GPU.
thread_local int t_k2_grid_sms = 0;

struct GridCache {
  int dev = -1;
  int grid[4] = {0, 0, 0, 0};
};

template <typename T, bool STEP>
int mean_grid() {
  static thread_local GridCache cache;
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  const int slot = (sizeof(T) == 4 ? 0 : 1) + (STEP ? 2 : 0);
  if (cache.dev != dev) {
    cache.dev = dev;
    cache.grid[0] = cache.grid[1] = cache.grid[2] = cache.grid[3] = 0;
  }
  if (!cache.grid[slot]) {
    int sms = 0, per = 0;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per, group_mean_register<T, STEP>, kThreads, 0));
    cache.grid[slot] = sms * (per > 0 ? per : 1);
  }
  return cache.grid[slot];
}

bool bulk_default() {
  static const bool on = [] {
    const char* e = std::getenv("MOSHPIT_KERNEL");
    return e && std::string(e) == "bulk";
  }();
  return on;
}

}  // namespace

void set_k2_grid_sms(int sms) { t_k2_grid_sms = sms; }

template <typename T>
void launch_group_mean(T* state, std::uint64_t ld, std::uint64_t dim,
                       const std::uint32_t* members, const std::uint32_t* goff,
                       const std::uint32_t* act, const std::uint32_t* counts,
                       std::uint32_t max_group, int variant, cudaStream_t s,
                       const StepPrologue<T>* step) {
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
  a.batch_state_stride = 0;
  a.batch_n = 0;
  if (step) {
    a.step = *step;
    // Kernel 3 (step_kernel.cu: leaf-streamed step + round 1) for groups of
    // <= 32; larger groups take the register form's generic tree.
    if (max_group <= 32) {
      launch_group_mean_step<T>(state, ld, dim, members, goff, act, counts, *step, s);
      return;
    }
    group_mean_register<T, true><<<mean_grid<T, true>(), kThreads, 0, s>>>(a);
    MB_LAUNCH_CHECK();
    return;
  }
  const bool bulk_ok = max_group <= (std::uint32_t)kBulkMaxRows;
  if (variant == 2 || (variant == 0 && bulk_ok && bulk_default())) {
    if (!bulk_ok) throw std::invalid_argument("bulk kernel: groups larger than 32 members");
    const std::uint32_t srows = max_group;
    const std::size_t row_bytes = (std::size_t)kBulkTileVec * 16;
    const std::size_t budget = 200 * 1024;
    int stages = (int)(budget / (srows * row_bytes + sizeof(BulkHdr) + 16));
    if (stages > 8) stages = 8;
    if (stages < 2) stages = 2;
    const std::size_t smem = (std::size_t)stages * (srows * row_bytes + sizeof(BulkHdr) + 16) + 128;
    static thread_local int configured_dev[2] = {-1, -1};
    int dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    const int slot = sizeof(T) == 4 ? 0 : 1;
    if (configured_dev[slot] != dev) {
      MB_CUDA(cudaFuncSetAttribute(group_mean_bulk<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   227 * 1024));
      configured_dev[slot] = dev;
    }
    int sms = 0;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    a.n_tiles = (a.nvec + kBulkTileVec - 1) / kBulkTileVec;
    group_mean_bulk<T><<<sms, kBulkThreads, smem, s>>>(a, stages, (int)srows);
  } else {
    // Fewer concurrent row streams keep DRAM pages open: measured on B200
    // (profiles/r01/k2_grid_sweep.txt) two 128-thread CTAs per SM are best for
    // groups of 16-32 members (0.95-0.96 of the copy peak vs 0.91-0.92 at full
    // occupancy); groups of <= 8 need full occupancy for bytes in flight.
    int sms = 0, dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int occ = mean_grid<T, false>() / (sms ? sms : 1);
    int per = max_group > 8 ? 2 : occ;
    if (const char* e = std::getenv("MOSHPIT_K2_CTAS_PER_SM")) per = std::atoi(e);
    if (per < 1) per = 1;
    if (per > occ) per = occ;
    // Pin residency to exactly `per` CTAs per SM: reserve enough dynamic shared
    // memory that a (per+1)-th CTA cannot fit, so the grid of sms*per CTAs is
    // spread evenly instead of stacking up to the register limit on some SMs.
    std::size_t pin = 0;
    if (per < occ) {
      int smem_sm = 0;
      MB_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
      pin = (std::size_t)smem_sm / (per + 1) + 1024;
      static thread_local int set_dev[2] = {-1, -1};
      const int slot = sizeof(T) == 4 ? 0 : 1;
      if (set_dev[slot] != dev) {
        MB_CUDA(cudaFuncSetAttribute(group_mean_register<T, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        set_dev[slot] = dev;
      }
    }
    if (std::getenv("MOSHPIT_DEBUG")) {
      static thread_local int once = 0;
      if (!once++)
        fprintf(stderr, "[moshpit] kernel2 max_group=%u occ=%d per=%d pin=%zu grid=%d\n",
                max_group, occ, per, pin, sms * per);
    }
    const int gsms = t_k2_grid_sms > 0 && t_k2_grid_sms < sms ? t_k2_grid_sms : sms;
    group_mean_register<T, false><<<gsms * per, kThreads, pin, s>>>(a);
  }
  MB_LAUNCH_CHECK();
}

template <typename T>
void launch_group_mean_batch(T* state, std::uint64_t state_stride, std::uint64_t ld,
                             std::uint64_t dim, std::uint32_t n, std::uint32_t trials,
                             const std::uint32_t* members, const std::uint32_t* goff,
                             const std::uint32_t* act, const std::uint32_t* counts,
                             cudaStream_t s) {
  if (dim == 0 || trials == 0) return;
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
  a.batch_state_stride = state_stride;
  a.batch_n = n;
  // per trial: at most n groups x n_tiles items; spread ~2 waves of CTAs
  int sms = 0, dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  std::uint64_t gx = ((std::uint64_t)sms * 2 + trials - 1) / trials;
  const std::uint64_t items = (std::uint64_t)n * a.n_tiles;
  if (gx > items) gx = items;
  if (gx < 1) gx = 1;
  for (std::uint32_t t0 = 0; t0 < trials; t0 += 65535) {
    const std::uint32_t tb = trials - t0 < 65535 ? trials - t0 : 65535;
    MeanArgs<T> b = a;
    b.state += (std::uint64_t)t0 * state_stride;
    b.members += (std::uint64_t)t0 * n;
    b.goff += (std::uint64_t)t0 * (n + 1);
    b.act += (std::uint64_t)t0 * n;
    b.counts += (std::uint64_t)t0 * 4;
    group_mean_register<T, false><<<dim3((unsigned)gx, tb), kThreads, 0, s>>>(b);
    MB_LAUNCH_CHECK();
  }
}

template void launch_group_mean_batch<float>(float*, std::uint64_t, std::uint64_t,
                                             std::uint64_t, std::uint32_t, std::uint32_t,
                                             const std::uint32_t*, const std::uint32_t*,
                                             const std::uint32_t*, const std::uint32_t*,
                                             cudaStream_t);
template void launch_group_mean_batch<double>(double*, std::uint64_t, std::uint64_t,
                                              std::uint64_t, std::uint32_t, std::uint32_t,
                                              const std::uint32_t*, const std::uint32_t*,
                                              const std::uint32_t*, const std::uint32_t*,
                                              cudaStream_t);

template void launch_group_mean<float>(float*, std::uint64_t, std::uint64_t,
                                       const std::uint32_t*, const std::uint32_t*,
                                       const std::uint32_t*, const std::uint32_t*,
                                       std::uint32_t, int, cudaStream_t,
                                       const StepPrologue<float>*);
template void launch_group_mean<double>(double*, std::uint64_t, std::uint64_t,
                                        const std::uint32_t*, const std::uint32_t*,
                                        const std::uint32_t*, const std::uint32_t*,
                                        std::uint32_t, int, cudaStream_t,
                                        const StepPrologue<double>*);

int group_mean_grid_size(bool f64, bool step) {
  if (f64) return step ? mean_grid<double, true>() : mean_grid<double, false>();
  return step ? mean_grid<float, true>() : mean_grid<float, false>();
}

}  // namespace mb200
