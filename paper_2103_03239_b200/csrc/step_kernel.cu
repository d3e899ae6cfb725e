// step_kernel.cu -- Kernel 3: the local Moshpit-SGD step fused into the first
// averaging round (optimizer.hpp:356-381 then 249-284), for groups of at most
// 32 members.
//
// Same data plane as Kernel 2 (mean_kernel.cu): work item = (active group,
// D-tile of 128 x 16-byte vectors), one read and one write of every active
// row.  Each member vector is stepped as it is loaded,
//     g = c * (theta - t) [+ n_j],   theta' = theta - gamma * g
// (separately rounded, no FMA; optimizer.hpp:356-373), then enters the
// reference pairwise tree (core.hpp:72-81).
//
// Why a separate kernel.  The tree over n <= 32 members is a fixed set of at
// most four sequential LEAVES of <= 8 consecutive members (n <= 8: one leaf;
// n <= 16: two, split at floor(n/2); n <= 32: the two halves split again,
// a half of exactly 8 staying one leaf), joined as L0 | L0+L1 | L0+(L1+L2) |
// (L0+L1)+(L2+L3).  Streaming leaf by leaf (a few loads in flight per thread, many
// warps per SM) needs a fraction of the registers of holding all 32 member
// vectors, and one runtime-n code body
// replaces 32 unrolled specialisations -- the fully unrolled step+Philox form
// was 2.3 MB of SASS, and instruction-cache misses ("no_instruction" stalls,
// 34 % of samples) held it at ~50 % of HBM bandwidth.
//
// Bit-exactness: leaf sums start from +0 and add members in priority order;
// the joins are the reference's; the step matches sgd_step_kernel (sgd.cu)
// and the Philox noise per (step, peer, coordinate quad) is the same function,
// so this kernel, the register form and step-then-average are bit-identical.
#include <algorithm>
#include <stdexcept>

#include "common.cuh"
#include "philox.cuh"

namespace mb200 {
namespace {

constexpr int kLThreads = 128;
#ifndef MB_K3_ILP
#define MB_K3_ILP 4
#endif
constexpr int kIlp = MB_K3_ILP;  // members whose Philox chains interleave
#ifndef MB_K3_MINB
#define MB_K3_MINB 5
#endif
constexpr int kNoisyMinB = MB_K3_MINB;  // CTAs/SM of the noisy 4-wide form


template <typename T>
struct LVec;
template <>
struct LVec<float> {
  using V = float4;
  static constexpr int kN = 4;
};
template <>
struct LVec<double> {
  using V = double2;
  static constexpr int kN = 2;
};

__device__ __forceinline__ float lsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float lmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float ladd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float lfma0(float g, float acc) { return __fmaf_rn(g, 0.f, acc); }
__device__ __forceinline__ double lsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double lmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ladd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double lfma0(double g, double acc) { return __fma_rn(g, 0.0, acc); }
__device__ __forceinline__ float ldiv(float a, float n) { return __fdiv_rn(a, n); }
__device__ __forceinline__ double ldiv(double a, double n) { return __ddiv_rn(a, n); }

template <typename T>
struct LArgs {
  T* state;
  std::uint64_t ld_vec, nvec, n_tiles;
  const std::uint32_t* members;
  const std::uint32_t* goff;
  const std::uint32_t* act;
  const std::uint32_t* counts;
  const T* curv;
  const T* tgt;
  T gamma;
  double coord_std;
  std::uint64_t seed, step_no, dim;
  std::uint32_t* nonfinite;
  double* noise_partial;
  PhiloxKeys pk;  // Philox round keys of `seed` (constant-bank operands)
};

// Leaf boundaries of the reference tree for n <= 32 (see header comment).
__device__ __forceinline__ int leaf_bounds(std::uint32_t n, std::uint32_t* b) {
  if (n <= 8) {
    b[0] = 0; b[1] = n;
    return 1;
  }
  const std::uint32_t h = n / 2;
  if (n <= 16) {
    b[0] = 0; b[1] = h; b[2] = n;
    return 2;
  }
  const std::uint32_t n2 = n - h;  // >= 9: always split
  if (h <= 8) {                    // n == 17: left half is one leaf
    b[0] = 0; b[1] = h; b[2] = h + n2 / 2; b[3] = n;
    return 3;
  }
  b[0] = 0; b[1] = h / 2; b[2] = h; b[3] = h + n2 / 2; b[4] = n;
  return 4;
}

// One member vector: the step, lane by lane (element j of the row).  `cst`
// is coord_std in the state's precision ((T)coord_std, hoisted), so
// cst * z is noise_component() exactly.  Full vectors (every thread but the
// row tail's) run the lanes without per-lane exits: the Box-Muller SFU ops
// and the lane steps schedule as one block instead of four.
// The lanes of one member vector given its four normals z (unused when
// !NOISY).
template <typename T, bool NOISY, typename V>
__device__ __forceinline__ void step_lanes(V& v, const V& c, const V& t, T gamma, T cst,
                                           const float (&z)[4], std::uint64_t j0, bool full,
                                           std::uint64_t dim, T& chk, double& nsq) {
  constexpr int kV = LVec<T>::kN;
  T* pv = reinterpret_cast<T*>(&v);
  const T* pc = reinterpret_cast<const T*>(&c);
  const T* pt = reinterpret_cast<const T*>(&t);
  T q = T(0);
  auto lane = [&](int u) {
    T g = lmul(pc[u], lsub(pv[u], pt[u]));
    if constexpr (NOISY) {
      const T nj = lmul(cst, (T)z[(j0 + u) & 3]);
      nsq_add(q, nj);
      g = ladd(g, nj);
    }
    chk = lfma0(g, chk);  // stays 0 unless some g is inf/NaN
    pv[u] = lsub(pv[u], lmul(gamma, g));
  };
  if (full) {
#pragma unroll
    for (int u = 0; u < kV; ++u) lane(u);
  } else {
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      if (j0 + u >= dim) break;
      lane(u);
    }
  }
  if constexpr (NOISY) nsq += (double)q;
}

template <typename T, bool NOISY, typename V>
__device__ __forceinline__ void step_vec(V& v, const V& c, const V& t, T gamma, T cst,
                                         const PhiloxKeys& seed, std::uint64_t step_no,
                                         std::uint32_t peer, std::uint64_t j0, bool full,
                                         std::uint64_t dim, T& chk, double& nsq) {
  float z[4] = {0.f, 0.f, 0.f, 0.f};
  if constexpr (NOISY) philox_normals4(seed, step_no, peer, j0 / 4, z);
  step_lanes<T, NOISY>(v, c, t, gamma, cst, z, j0, full, dim, chk, nsq);
}

template <typename V>
__device__ __forceinline__ V vz() {
  V v;
  if constexpr (sizeof(V) == 16 && sizeof(v.x) == 4) v = make_float4(0.f, 0.f, 0.f, 0.f);
  else v = make_double2(0.0, 0.0);
  return v;
}
__device__ __forceinline__ float4 vsum(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ double2 vsum(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ float4 vdivn(float4 a, std::uint32_t n) {
  const float f = (float)n;
  return make_float4(ldiv(a.x, f), ldiv(a.y, f), ldiv(a.z, f), ldiv(a.w, f));
}
__device__ __forceinline__ double2 vdivn(double2 a, std::uint32_t n) {
  const double f = (double)n;
  return make_double2(ldiv(a.x, f), ldiv(a.y, f));
}

// 4-member load batches.  Without noise: 64 registers, 8 CTAs/SM (warps
// hide the load latency).  With device noise the batch's four Philox chains
// are computed together (kIlp) so their dependent IMAD/LOP3 rounds
// interleave, at kNoisyMinB = 5 CTAs/SM (94 registers, no spills): C4
// sigma=1 step 3.34 -> 3.18 ms; at 8 CTAs/SM the same code spills (3.21 ms)
// and one chain at a time measured 3.34 ms (profiles/k3_variants.sh).  The
// round-1 variants measured slower -- 8-member batches (2.91-2.94 ms at
// sigma=0, 3.69-3.80 with noise), the next batch prefetched under the Philox
// rounds (3.60-3.67 ms, profiles/r01/k3_variants_prefetch.txt), the leaf
// body as a plain Kernel 2 (1.5-5 % below the register form,
// profiles/k2_leaf_sweep.sh) -- and were removed in round 2.
template <typename T, bool NOISY>
__global__ void __launch_bounds__(kLThreads, NOISY ? kNoisyMinB : 8)
    group_mean_step_leaf(LArgs<T> a) {
  using V = typename LVec<T>::V;
  constexpr int kV = LVec<T>::kN;
  __shared__ std::uint32_t sids[32];
  __shared__ std::uint32_t sb[6];
  const T gamma = a.gamma;
  const T cst = (T)a.coord_std;  // noise_component's multiplier
  const std::uint64_t step_no = a.step_no, dim = a.dim;
  const PhiloxKeys& seed = a.pk;
  const std::uint64_t ld_vec = a.ld_vec, nvec = a.nvec, n_tiles = a.n_tiles;
  V* const base = reinterpret_cast<V*>(a.state);
  T chk = T(0);
  double nsq = 0.0;
  const std::uint64_t n_items = (std::uint64_t)a.counts[1] * n_tiles;
  std::uint32_t cached = 0xffffffffu;
  std::uint32_t cnt = 0, nl = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0, b4 = 0;
  for (std::uint64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
    const std::uint32_t g = a.act[w / n_tiles];
    if (g != cached) {  // uniform across the CTA
      __syncthreads();
      const std::uint32_t beg = a.goff[g];
      cnt = a.goff[g + 1] - beg;
      if (threadIdx.x < cnt) sids[threadIdx.x] = a.members[beg + threadIdx.x];
      if (threadIdx.x == 0) sb[5] = leaf_bounds(cnt, sb);
      cached = g;
      __syncthreads();
      nl = sb[5];
      b0 = sb[0];
      b1 = sb[1];
      b2 = sb[2];
      b3 = sb[3];
      b4 = sb[4];
    }
    const std::uint64_t col = (w % n_tiles) * kLThreads + threadIdx.x;
    if (col >= nvec) continue;
    const std::uint64_t j0 = col * kV;
    const bool full = j0 + kV <= dim;
    const V c = __ldg(reinterpret_cast<const V*>(a.curv) + col);
    const V t = __ldg(reinterpret_cast<const V*>(a.tgt) + col);
    V* const colp = base + col;

    // Leaves in a runtime loop (one copy of the 8-member body: the unrolled
    // step + Philox code must stay instruction-cache resident).  Joins:
    // leaves before `r` accumulate into P, the rest into Q, sum = P + Q --
    // L0 | L0+L1 | L0+(L1+L2) | (L0+L1)+(L2+L3) for nl = 1..4.
    const std::uint32_t r = nl == 4 ? 2u : 1u;
    V P = vz<V>(), Q = vz<V>();
    {
      std::uint32_t lb = b0;
#pragma unroll 1
      for (std::uint32_t l = 0; l < nl; ++l) {
        const std::uint32_t le = l == 0 ? b1 : l == 1 ? b2 : l == 2 ? b3 : b4;
        V sl = vz<V>();
#pragma unroll 1
        for (std::uint32_t c0 = lb; c0 < le; c0 += 4) {
          V X[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            X[k] = (c0 + k < le) ? colp[(std::uint64_t)sids[c0 + k] * ld_vec] : vz<V>();
          if (c0 + 4 <= le) {
            // whole batch: the four members' Philox chains are independent
            // and interleave (ILP against the dependent IMAD/LOP3 rounds)
            {
#pragma unroll
              for (int k = 0; k < 4; k += kIlp) {
                float z[kIlp][4] = {};
                if constexpr (NOISY) {
#pragma unroll
                  for (int e = 0; e < kIlp; ++e)
                    philox_normals4(seed, step_no, sids[c0 + k + e], j0 / 4, z[e]);
                }
#pragma unroll
                for (int e = 0; e < kIlp; ++e)
                  step_lanes<T, NOISY>(X[k + e], c, t, gamma, cst, z[e], j0, full, dim, chk,
                                       nsq);
              }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) sl = vsum(sl, X[k]);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (c0 + k < le) {
                step_vec<T, NOISY>(X[k], c, t, gamma, cst, seed, step_no, sids[c0 + k], j0,
                                   full, dim, chk, nsq);
                sl = vsum(sl, X[k]);
              }
            }
          }
        }
        if (l < r) P = l == 0 ? sl : vsum(P, sl);
        else Q = l == r ? sl : vsum(Q, sl);
        lb = le;
      }
    }
    const V sum = nl == 1 ? P : vsum(P, Q);
    const V m = vdivn(sum, cnt);
#pragma unroll 8
    for (std::uint32_t k = 0; k < cnt; ++k) colp[(std::uint64_t)sids[k] * ld_vec] = m;
  }
  // per-CTA sum of n_j^2 (sigma_hat) and the non-finite flag
  if constexpr (NOISY) {
    __shared__ double red[kLThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nsq;
    __syncthreads();
    if (threadIdx.x == 0 && a.noise_partial) {
      double s = 0.0;
      for (int i = 0; i < kLThreads / 32; ++i) s += red[i];
      a.noise_partial[blockIdx.x] = s;
    }
  } else if (threadIdx.x == 0 && a.noise_partial) {
    a.noise_partial[blockIdx.x] = 0.0;
  }
  if (chk != T(0)) atomicOr(a.nonfinite, 1u);
}

template <typename T, bool NOISY>
int leaf_grid() {
  static thread_local int dev_cached = -1, grid = 0;
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  if (dev != dev_cached) {
    int sms = 0, per = 0;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per, group_mean_step_leaf<T, NOISY>, kLThreads, 0));
    grid = sms * (per > 0 ? per : 1);
    dev_cached = dev;
  }
  return grid;
}

template <typename T, bool NOISY>
void launch_leaf(const LArgs<T>& a, cudaStream_t s) {
  group_mean_step_leaf<T, NOISY><<<leaf_grid<T, NOISY>(), kLThreads, 0, s>>>(a);
}

// ---------------------------------------------------------------------------
// Two-round pass for the Moshpit-SGD averaging step (moshpit_average with two
// rounds and no failures, optimizer.hpp:249-284; C4): the local step, round
// 1 and round 2 in ONE read and ONE write of the state.  Coordinates are
// independent and a thread owns one 16-byte column vector of a tile, so it
// can finish both rounds for its column before storing anything:
//   round 1  every group g1 (kernel 3's leaf-streamed tree with the step and
//            the Philox normals): its mean m1[g1] goes to shared memory
//            (this thread's column slot), nothing is written to HBM;
//   round 2  every group g2: the reference tree over its members' values,
//            member k's value being m1[group of k in round 1] (without
//            failures every peer was in an averaged round-1 group, so its
//            row would hold exactly that mean), then the mean is stored to
//            every member row.
// Bit-identical to kernel 3 + kernel 2 (same step, same noise per (step,
// peer, quad), the same trees, the same division); HBM traffic 2 * n * D *
// sizeof(T) per SGD step instead of twice that.  Shared memory: G1 slots of
// 16 bytes per thread (64-thread CTAs: 32 KB at G1 = 32, 7 CTAs per SM).
constexpr int kTwoThreads = 64;
constexpr std::uint32_t kTwoMaxG1 = 96;

template <typename T>
struct TwoArgs {
  T* state;
  std::uint64_t ld_vec, nvec, n_tiles;
  const std::uint32_t* members1;
  const std::uint32_t* goff1;
  const std::uint32_t* counts1;
  const std::uint32_t* members2;
  const std::uint32_t* goff2;
  const std::uint32_t* counts2;
  const std::uint32_t* src1;  // [n] round-1 group of the member at round-2 position pos
  const std::uint32_t* leaf_pos;   // round-1 leaves in order: first position in members1
  const std::uint32_t* leaf_meta;  // len | l << 4 | nl << 6 | cnt << 9 | g << 15
  const std::uint32_t* n_leaves;
  std::uint32_t n, g1_max;
  const T* curv;
  const T* tgt;
  T gamma;
  double coord_std;
  std::uint64_t step_no, dim;
  std::uint32_t* nonfinite;
  double* noise_partial;
  PhiloxKeys pk;
};

// round-2 source table: src1[pos2] = round-1 group of members2[pos2]
// ... and round 1's leaf schedule (group order, <= 4 leaves of <= 8 per group)
__global__ void __launch_bounds__(1024) two_round_src_kernel(
    const std::uint32_t* members1, const std::uint32_t* goff1, const std::uint32_t* counts1,
    const std::uint32_t* members2, std::uint32_t n, std::uint32_t* grp1,
    std::uint32_t* src1, std::uint32_t* leaf_pos, std::uint32_t* leaf_meta,
    std::uint32_t* n_leaves) {
  const std::uint32_t g1n = counts1[0];
  __shared__ std::uint32_t s_first[kTwoMaxG1 + 1];
  if (g1n > kTwoMaxG1) __trap();  // the host's bound (grid lines) broke
  for (std::uint32_t g = threadIdx.x; g < g1n; g += blockDim.x)
    for (std::uint32_t pos = goff1[g]; pos < goff1[g + 1]; ++pos) grp1[members1[pos]] = g;
  if (threadIdx.x == 0) {  // leaves before group g (g1n <= kTwoMaxG1)
    std::uint32_t acc = 0;
    for (std::uint32_t g = 0; g < g1n; ++g) {
      s_first[g] = acc;
      const std::uint32_t cnt = goff1[g + 1] - goff1[g];
      acc += cnt <= 8 ? 1u : cnt <= 16 ? 2u : cnt == 17 ? 3u : 4u;
    }
    s_first[g1n] = acc;
    *n_leaves = acc;
  }
  __syncthreads();
  for (std::uint32_t g = threadIdx.x; g < g1n; g += blockDim.x) {
    const std::uint32_t beg = goff1[g], cnt = goff1[g + 1] - beg;
    std::uint32_t b[5] = {0, 0, 0, 0, 0};
    const std::uint32_t nl = (std::uint32_t)leaf_bounds(cnt, b);
    for (std::uint32_t l = 0; l < nl; ++l) {
      leaf_pos[s_first[g] + l] = beg + b[l];
      leaf_meta[s_first[g] + l] = (b[l + 1] - b[l]) | (l << 4) | (nl << 6) | (cnt << 9) | (g << 15);
    }
  }
  for (std::uint32_t pos = threadIdx.x; pos < n; pos += blockDim.x) src1[pos] = grp1[members2[pos]];
}

template <typename T, bool NOISY>
__global__ void __launch_bounds__(kTwoThreads, 6)
    two_round_step_kernel(TwoArgs<T> a) {
  using V = typename LVec<T>::V;
  constexpr int kV = LVec<T>::kN;
  extern __shared__ uint4 two_smem[];
  V* const m1 = reinterpret_cast<V*>(two_smem);  // [g1_max][kTwoThreads]
  const T gamma = a.gamma;
  const T cst = (T)a.coord_std;
  const std::uint64_t step_no = a.step_no, dim = a.dim, ld_vec = a.ld_vec;
  const PhiloxKeys& seed = a.pk;
  V* const base = reinterpret_cast<V*>(a.state);
  const std::uint32_t G1 = a.counts1[0], G2 = a.counts2[0];
  // round 2's tables in shared memory (its loop is a chain of table look-ups:
  // position -> round-1 slot / member row): packed (src1 << 16 | member) per
  // position, then the group offsets
  std::uint32_t* const s_tab = reinterpret_cast<std::uint32_t*>(m1 + a.g1_max * kTwoThreads);
  std::uint32_t* const s_goff2 = s_tab + a.n;
  for (std::uint32_t q = threadIdx.x; q < a.n; q += kTwoThreads)
    s_tab[q] = (__ldg(a.src1 + q) << 16) | __ldg(a.members2 + q);
  if (G1 > a.g1_max || G2 > a.g1_max) __trap();  // the host's bound (grid lines) broke
  for (std::uint32_t q = threadIdx.x; q <= G2; q += kTwoThreads) s_goff2[q] = __ldg(a.goff2 + q);
  __syncthreads();
  T chk = T(0);
  double nsq = 0.0;
  for (std::uint64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const std::uint64_t col = tile * kTwoThreads + threadIdx.x;
    if (col >= a.nvec) continue;  // no barriers below: each thread owns its column
    const std::uint64_t j0 = col * kV;
    const bool full = j0 + kV <= dim;
    const V c = __ldg(reinterpret_cast<const V*>(a.curv) + col);
    const V t = __ldg(reinterpret_cast<const V*>(a.tgt) + col);
    V* const colp = base + col;
    // round 1: the step + the tree of every group; means to shared memory.
    // Software-pipelined over the flat leaf schedule: the NEXT leaf's member
    // loads (<= 8 rows) are in flight while this leaf's Philox normals, step
    // and sum run (the shared-memory means cap the CTAs per SM, so each
    // thread carries the memory parallelism).
    {
      const std::uint32_t NL = __ldg(a.n_leaves);
      std::uint32_t meta = __ldg(a.leaf_meta), pos = __ldg(a.leaf_pos);
      std::uint32_t id[8];
      V X[8];
      {
        const std::uint32_t len = meta & 15u;
#pragma unroll
        for (int k = 0; k < 8; ++k) id[k] = (k < (int)len) ? __ldg(a.members1 + pos + k) : 0u;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          X[k] = (k < (int)len) ? colp[(std::uint64_t)id[k] * ld_vec] : vz<V>();
      }
      V P = vz<V>(), Q = vz<V>();
#pragma unroll 1
      for (std::uint32_t L = 0; L < NL; ++L) {
        // next leaf's loads first
        std::uint32_t meta_n = 0, id_n[8];
        V X_n[8];
        {
          const bool more = L + 1 < NL;
          const std::uint32_t pos_n = more ? __ldg(a.leaf_pos + L + 1) : 0u;
          meta_n = more ? __ldg(a.leaf_meta + L + 1) : 0u;
          const std::uint32_t len_n = meta_n & 15u;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            id_n[k] = (k < (int)len_n) ? __ldg(a.members1 + pos_n + k) : 0u;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            X_n[k] = (k < (int)len_n) ? colp[(std::uint64_t)id_n[k] * ld_vec] : vz<V>();
        }
        const std::uint32_t len = meta & 15u, l = (meta >> 4) & 3u, nl = (meta >> 6) & 7u;
        const std::uint32_t cnt = (meta >> 9) & 63u, g = meta >> 15;
#pragma unroll
        for (int h = 0; h < 8; h += 4) {
          if ((std::uint32_t)h + 4 <= len) {
            float z[4][4] = {};
            if constexpr (NOISY) {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                philox_normals4(seed, step_no, id[h + e], j0 / 4, z[e]);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
              step_lanes<T, NOISY>(X[h + e], c, t, gamma, cst, z[e], j0, full, dim, chk, nsq);
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if ((std::uint32_t)(h + e) < len)
                step_vec<T, NOISY>(X[h + e], c, t, gamma, cst, seed, step_no, id[h + e], j0,
                                   full, dim, chk, nsq);
          }
        }
        V sl = vz<V>();
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if ((std::uint32_t)k < len) sl = vsum(sl, X[k]);
        // joins: L0 | L0+L1 | L0+(L1+L2) | (L0+L1)+(L2+L3)
        const std::uint32_t r = nl == 4 ? 2u : 1u;
        if (l < r) P = l == 0 ? sl : vsum(P, sl);
        else Q = l == r ? sl : vsum(Q, sl);
        if (l + 1 == nl) m1[g * kTwoThreads + threadIdx.x] = vdivn(nl == 1 ? P : vsum(P, Q), cnt);
        meta = meta_n;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          id[k] = id_n[k];
          X[k] = X_n[k];
        }
      }
    }
    // round 2: member k of group g2 holds m1[src1[pos]]
#pragma unroll 1
    for (std::uint32_t g = 0; g < G2; ++g) {
      const std::uint32_t beg = s_goff2[g];
      const std::uint32_t cnt = s_goff2[g + 1] - beg;
      std::uint32_t b[5] = {0, 0, 0, 0, 0};
      const std::uint32_t nl = (std::uint32_t)leaf_bounds(cnt, b);
      const std::uint32_t b1 = b[1], b2 = b[2], b3 = b[3], b4 = b[4];
      const std::uint32_t r = nl == 4 ? 2u : 1u;
      V P = vz<V>(), Q = vz<V>();
      std::uint32_t lb = 0;
#pragma unroll 1
      for (std::uint32_t l = 0; l < nl; ++l) {
        const std::uint32_t le = l == 0 ? b1 : l == 1 ? b2 : l == 2 ? b3 : b4;
        V sl = vz<V>();
#pragma unroll 4
        for (std::uint32_t k = lb; k < le; ++k)
          sl = vsum(sl, m1[(s_tab[beg + k] >> 16) * kTwoThreads + threadIdx.x]);
        if (l < r) P = l == 0 ? sl : vsum(P, sl);
        else Q = l == r ? sl : vsum(Q, sl);
        lb = le;
      }
      const V m = vdivn(nl == 1 ? P : vsum(P, Q), cnt);
#pragma unroll 4
      for (std::uint32_t k = 0; k < cnt; ++k)
        __stcs(colp + (std::uint64_t)(s_tab[beg + k] & 0xffffu) * ld_vec, m);
    }
  }
  if constexpr (NOISY) {
    __shared__ double red[kTwoThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nsq;
    __syncthreads();
    if (threadIdx.x == 0 && a.noise_partial) {
      double s = 0.0;
      for (int i = 0; i < kTwoThreads / 32; ++i) s += red[i];
      a.noise_partial[blockIdx.x] = s;
    }
  } else if (threadIdx.x == 0 && a.noise_partial) {
    a.noise_partial[blockIdx.x] = 0.0;
  }
  if (chk != T(0)) atomicOr(a.nonfinite, 1u);
}

}  // namespace

template <typename T>
void launch_group_mean_step(T* state, std::uint64_t ld, std::uint64_t dim,
                            const std::uint32_t* members, const std::uint32_t* goff,
                            const std::uint32_t* act, const std::uint32_t* counts,
                            const StepPrologue<T>& sp, cudaStream_t s) {
  if (dim == 0) return;
  constexpr int kV = LVec<T>::kN;
  LArgs<T> a;
  a.state = state;
  a.ld_vec = ld / kV;
  a.nvec = (dim + kV - 1) / kV;
  a.n_tiles = (a.nvec + kLThreads - 1) / kLThreads;
  a.members = members;
  a.goff = goff;
  a.act = act;
  a.counts = counts;
  a.curv = sp.curv;
  a.tgt = sp.tgt;
  a.gamma = sp.gamma;
  a.coord_std = sp.coord_std;
  a.seed = sp.seed;
  a.pk = philox_keys(sp.seed);
  a.step_no = sp.step_no;
  a.dim = sp.dim;
  a.nonfinite = sp.nonfinite;
  a.noise_partial = sp.noise_partial;
  if (sp.philox) launch_leaf<T, true>(a, s);
  else launch_leaf<T, false>(a, s);
  MB_LAUNCH_CHECK();
}

int group_mean_step_grid(bool f64, bool noisy) {
  if (f64) return noisy ? leaf_grid<double, true>() : leaf_grid<double, false>();
  return noisy ? leaf_grid<float, true>() : leaf_grid<float, false>();
}

// Step + two averaging rounds in one pass (see two_round_step_kernel).  The
// caller guarantees: no voided groups (p = 0), groups of <= 32 members, at
// most two_round_max_groups() groups in round 1.  grp1: n u32, src1: n +
// 8 * two_round_max_groups() + 1 u32 (scratch: the round-2 sources, then
// round 1's leaf schedule).  Grid: at most 148 * 16 CTAs (the noise-partial slots).
std::uint32_t two_round_max_groups() { return kTwoMaxG1; }

template <typename T>
void launch_two_round_step(T* state, std::uint64_t ld, std::uint64_t dim, std::uint32_t n,
                           const FusedRound* host_rounds, std::uint32_t g1_max,
                           std::uint32_t* grp1, std::uint32_t* src1, const StepPrologue<T>& sp,
                           cudaStream_t s) {
  if (dim == 0) return;
  if (g1_max > kTwoMaxG1) throw std::invalid_argument("two-round pass: too many round-1 groups");
  constexpr int kV = LVec<T>::kN;
  const FusedRound& r1 = host_rounds[0];
  const FusedRound& r2 = host_rounds[1];
  std::uint32_t* leaf_pos = src1 + n;
  std::uint32_t* leaf_meta = leaf_pos + 4 * kTwoMaxG1;
  std::uint32_t* n_leaves = leaf_meta + 4 * kTwoMaxG1;
  two_round_src_kernel<<<1, 1024, 0, s>>>(r1.members, r1.goff, r1.counts, r2.members, n, grp1,
                                          src1, leaf_pos, leaf_meta, n_leaves);
  MB_LAUNCH_CHECK();
  TwoArgs<T> a;
  a.state = state;
  a.ld_vec = ld / kV;
  a.nvec = (dim + kV - 1) / kV;
  a.n_tiles = (a.nvec + kTwoThreads - 1) / kTwoThreads;
  a.members1 = r1.members;
  a.goff1 = r1.goff;
  a.counts1 = r1.counts;
  a.members2 = r2.members;
  a.goff2 = r2.goff;
  a.counts2 = r2.counts;
  a.src1 = src1;
  a.leaf_pos = leaf_pos;
  a.leaf_meta = leaf_meta;
  a.n_leaves = n_leaves;
  a.n = n;
  a.g1_max = g1_max;
  a.curv = sp.curv;
  a.tgt = sp.tgt;
  a.gamma = sp.gamma;
  a.coord_std = sp.coord_std;
  a.step_no = sp.step_no;
  a.dim = sp.dim;
  a.nonfinite = sp.nonfinite;
  a.noise_partial = sp.noise_partial;
  a.pk = philox_keys(sp.seed);
  if (n > 0xffffu) throw std::invalid_argument("two-round pass: more than 65535 peers");
  // round-1 means + round 2's packed table (n) and group offsets (round 2 has
  // at most as many groups as round 1's bound: both are lines of the grid)
  const std::size_t smem =
      (std::size_t)g1_max * kTwoThreads * 16 + ((std::size_t)n + g1_max + 1) * 4;
  auto run = [&](auto kern) {
    static thread_local int dev_cached = -1;
    static thread_local std::size_t smem_set = 0;
    int dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    if (dev != dev_cached || smem > smem_set) {
      MB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<std::size_t>(smem, 48 * 1024)));
      dev_cached = dev;
      smem_set = std::max<std::size_t>(smem, 48 * 1024);
    }
    int sms = 0, per = 0;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kTwoThreads, smem));
    std::uint64_t grid = (std::uint64_t)sms * std::max(per, 1);
    grid = std::min<std::uint64_t>(grid, std::min<std::uint64_t>(a.n_tiles, 148ull * 16));
    kern<<<(unsigned)grid, kTwoThreads, smem, s>>>(a);
  };
  if (sp.philox) run(two_round_step_kernel<T, true>);
  else run(two_round_step_kernel<T, false>);
  MB_LAUNCH_CHECK();
}

template void launch_two_round_step<float>(float*, std::uint64_t, std::uint64_t, std::uint32_t,
                                           const FusedRound*, std::uint32_t, std::uint32_t*,
                                           std::uint32_t*, const StepPrologue<float>&,
                                           cudaStream_t);
template void launch_two_round_step<double>(double*, std::uint64_t, std::uint64_t, std::uint32_t,
                                            const FusedRound*, std::uint32_t, std::uint32_t*,
                                            std::uint32_t*, const StepPrologue<double>&,
                                            cudaStream_t);

template void launch_group_mean_step<float>(float*, std::uint64_t, std::uint64_t,
                                            const std::uint32_t*, const std::uint32_t*,
                                            const std::uint32_t*, const std::uint32_t*,
                                            const StepPrologue<float>&, cudaStream_t);
template void launch_group_mean_step<double>(double*, std::uint64_t, std::uint64_t,
                                             const std::uint32_t*, const std::uint32_t*,
                                             const std::uint32_t*, const std::uint32_t*,
                                             const StepPrologue<double>&, cudaStream_t);

}  // namespace mb200
