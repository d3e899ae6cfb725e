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
#ifndef MB_K3_PF
#define MB_K3_PF 0
#endif
// Noisy 4-wide form with the next batch's loads issued under this batch's
// Philox rounds: parity-green but measured slower (C4 sigma=1 3.18 -> 3.67 ms
// at 4 CTAs/SM / 127 registers, 3.60 ms at 5 CTAs/SM with spills;
// profiles/r01/k3_variants_prefetch.txt), so off by default.
constexpr bool kPf = MB_K3_PF != 0;

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

// MODE 0: 8-member load batches; 1: 8-member batches with the next leaf
// prefetched; 2 (default): 4-member batches.  Without noise: 64 registers,
// 8 CTAs/SM (warps hide the load latency).  With device noise the batch's
// four Philox chains are computed together (kIlp) so their dependent
// IMAD/LOP3 rounds interleave, at kNoisyMinB = 5 CTAs/SM (94 registers, no
// spills): C4 sigma=1 step 3.34 -> 3.18 ms; at 8 CTAs/SM the same code
// spills (3.21 ms) and one chain at a time measured 3.34 ms
// (profiles/k3_variants.sh).  Same arithmetic in every mode.  MODE 3 / 4
// are the 4- / 8-wide forms WITHOUT the step: a plain Kernel-2 round (used
// for groups of <= 8 members, where the register form's 32-slot body caps
// residency at 3 CTAs/SM).
template <typename T, bool NOISY, int MODE>
__global__ void __launch_bounds__(kLThreads, MODE == 1 ? 4 : (MODE == 2 || MODE == 3) ? (NOISY ? kNoisyMinB : 8) : 6)
    group_mean_step_leaf(LArgs<T> a) {
  constexpr bool PREFETCH = MODE == 1;
  constexpr bool STEP = MODE < 3;
  constexpr bool WIDE4 = MODE == 2 || MODE == 3;
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
    V c = vz<V>(), t = vz<V>();
    if constexpr (STEP) {
      c = __ldg(reinterpret_cast<const V*>(a.curv) + col);
      t = __ldg(reinterpret_cast<const V*>(a.tgt) + col);
    }
    V* const colp = base + col;

    // predicated 8-wide leaf loads (unloaded slots are zero and never used)
    auto load_leaf = [&](V(&buf)[8], std::uint32_t b, std::uint32_t e) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        buf[k] = (b + k < e) ? colp[(std::uint64_t)sids[b + k] * ld_vec] : vz<V>();
    };
    auto sum_leaf = [&](V(&buf)[8], std::uint32_t b, std::uint32_t e) {
      V s = vz<V>();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (b + k < e) {
          if constexpr (STEP)
            step_vec<T, NOISY>(buf[k], c, t, gamma, cst, seed, step_no, sids[b + k], j0,
                               full, dim, chk, nsq);
          s = vsum(s, buf[k]);
        }
      }
      return s;
    };
    // Leaves in a runtime loop (one copy of the 8-member body: the unrolled
    // step + Philox code must stay instruction-cache resident).  Joins:
    // leaves before `r` accumulate into P, the rest into Q, sum = P + Q --
    // L0 | L0+L1 | L0+(L1+L2) | (L0+L1)+(L2+L3) for nl = 1..4.
    const std::uint32_t r = nl == 4 ? 2u : 1u;
    V P = vz<V>(), Q = vz<V>();
    auto load4 = [&](V(&X)[4], std::uint32_t c0, std::uint32_t le) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        X[k] = (c0 + k < le) ? colp[(std::uint64_t)sids[c0 + k] * ld_vec] : vz<V>();
    };
    // One 4-member batch [c0, min(c0+4, le)) stepped and added into sl.
    auto batch4 = [&](V(&X)[4], std::uint32_t c0, std::uint32_t le, V& sl) {
      if (c0 + 4 <= le) {
        // whole batch: the four members' Philox chains are independent
        // and interleave (ILP against the dependent IMAD/LOP3 rounds)
        if constexpr (STEP) {
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
              step_lanes<T, NOISY>(X[k + e], c, t, gamma, cst, z[e], j0, full, dim, chk, nsq);
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) sl = vsum(sl, X[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (c0 + k < le) {
            if constexpr (STEP)
              step_vec<T, NOISY>(X[k], c, t, gamma, cst, seed, step_no, sids[c0 + k], j0,
                                 full, dim, chk, nsq);
            sl = vsum(sl, X[k]);
          }
        }
      }
    };
    if constexpr (WIDE4 && NOISY && kPf) {
      // Same batches, same order, flattened over the leaves so batch i+1's
      // member loads are in flight while batch i runs its Philox rounds.
      auto lend = [&](std::uint32_t l) { return l == 0 ? b1 : l == 1 ? b2 : l == 2 ? b3 : b4; };
      std::uint32_t l = 0, c0 = b0, le = b1;
      V X[4];
      load4(X, c0, le);
      V sl = vz<V>();
#pragma unroll 1
      while (true) {
        std::uint32_t nl2 = l, nc = c0 + 4, ne = le;
        const bool leaf_end = nc >= le;
        if (leaf_end) {
          nl2 = l + 1;
          nc = le;
          ne = nl2 < nl ? lend(nl2) : le;
        }
        const bool more = nl2 < nl;
        V Y[4];
        if (more) load4(Y, nc, ne);
        batch4(X, c0, le, sl);
        if (leaf_end) {
          if (l < r) P = l == 0 ? sl : vsum(P, sl);
          else Q = l == r ? sl : vsum(Q, sl);
          sl = vz<V>();
        }
        if (!more) break;
#pragma unroll
        for (int k = 0; k < 4; ++k) X[k] = Y[k];
        l = nl2;
        c0 = nc;
        le = ne;
      }
    } else if constexpr (WIDE4) {
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
            if constexpr (STEP) {
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
                if constexpr (STEP)
                  step_vec<T, NOISY>(X[k], c, t, gamma, cst, seed, step_no, sids[c0 + k],
                                     j0, full, dim, chk, nsq);
                sl = vsum(sl, X[k]);
              }
            }
          }
        }
        if (l < r) P = l == 0 ? sl : vsum(P, sl);
        else Q = l == r ? sl : vsum(Q, sl);
        lb = le;
      }
    } else {
    V A[8], B[8];
    load_leaf(A, b0, b1);
    std::uint32_t lb = b0, le = b1;
#pragma unroll 1
    for (std::uint32_t l = 0; l < nl; ++l) {
      const std::uint32_t nb = le;
      const std::uint32_t ne = l + 1 == 1 ? b2 : l + 1 == 2 ? b3 : b4;
      const bool more = l + 1 < nl;
      if constexpr (PREFETCH) {
        if (more) load_leaf(B, nb, ne);
      }
      const V sl = sum_leaf(A, lb, le);
      if (l < r) P = l == 0 ? sl : vsum(P, sl);
      else Q = l == r ? sl : vsum(Q, sl);
      if (more) {
        if constexpr (PREFETCH) {
#pragma unroll
          for (int k = 0; k < 8; ++k) A[k] = B[k];
        } else {
          load_leaf(A, nb, ne);
        }
      }
      lb = nb;
      le = ne;
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
  } else if (STEP && threadIdx.x == 0 && a.noise_partial) {
    a.noise_partial[blockIdx.x] = 0.0;
  }
  if (STEP && chk != T(0)) atomicOr(a.nonfinite, 1u);
}

template <typename T, bool NOISY, int MODE>
int leaf_grid() {
  static thread_local int dev_cached = -1, grid = 0;
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  if (dev != dev_cached) {
    int sms = 0, per = 0;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per, group_mean_step_leaf<T, NOISY, MODE>, kLThreads, 0));
    grid = sms * (per > 0 ? per : 1);
    dev_cached = dev;
  }
  return grid;
}

template <typename T, bool NOISY, int MODE>
void launch_leaf(const LArgs<T>& a, cudaStream_t s) {
  group_mean_step_leaf<T, NOISY, MODE><<<leaf_grid<T, NOISY, MODE>(), kLThreads, 0, s>>>(a);
}

}  // namespace

template <typename T>
void launch_group_mean_step(T* state, std::uint64_t ld, std::uint64_t dim,
                            const std::uint32_t* members, const std::uint32_t* goff,
                            const std::uint32_t* act, const std::uint32_t* counts,
                            const StepPrologue<T>& sp, int prefetch, cudaStream_t s) {
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
  // mode < 0: the default, 4-wide batches at 8 CTAs/SM -- measured best on
  // B200 for both sigma = 0 (2.86 vs 2.91 / 2.94 ms per C4 step for modes
  // 1 / 0) and device noise (3.60 vs 3.80 / 3.69 ms)
  const int mode = prefetch >= 0 ? prefetch : 2;
  if (sp.philox) {
    if (mode == 2) launch_leaf<T, true, 2>(a, s);
    else if (mode == 1) launch_leaf<T, true, 1>(a, s);
    else launch_leaf<T, true, 0>(a, s);
  } else {
    if (mode == 2) launch_leaf<T, false, 2>(a, s);
    else if (mode == 1) launch_leaf<T, false, 1>(a, s);
    else launch_leaf<T, false, 0>(a, s);
  }
  MB_LAUNCH_CHECK();
}

// Plain Kernel-2 round through the leaf-streamed body (groups of <= 32).
template <typename T>
void launch_group_mean_leaf(T* state, std::uint64_t ld, std::uint64_t dim,
                            const std::uint32_t* members, const std::uint32_t* goff,
                            const std::uint32_t* act, const std::uint32_t* counts, int wide8,
                            cudaStream_t s) {
  if (dim == 0) return;
  constexpr int kV = LVec<T>::kN;
  LArgs<T> a{};
  a.state = state;
  a.ld_vec = ld / kV;
  a.nvec = (dim + kV - 1) / kV;
  a.n_tiles = (a.nvec + kLThreads - 1) / kLThreads;
  a.members = members;
  a.goff = goff;
  a.act = act;
  a.counts = counts;
  a.dim = dim;
  if (wide8) launch_leaf<T, false, 4>(a, s);
  else launch_leaf<T, false, 3>(a, s);
  MB_LAUNCH_CHECK();
}
template void launch_group_mean_leaf<float>(float*, std::uint64_t, std::uint64_t,
                                            const std::uint32_t*, const std::uint32_t*,
                                            const std::uint32_t*, const std::uint32_t*, int,
                                            cudaStream_t);
template void launch_group_mean_leaf<double>(double*, std::uint64_t, std::uint64_t,
                                             const std::uint32_t*, const std::uint32_t*,
                                             const std::uint32_t*, const std::uint32_t*, int,
                                             cudaStream_t);

int group_mean_step_grid(bool f64, bool noisy, int mode) {
  if (mode < 0) mode = 2;
  if (f64) {
    if (noisy) return mode == 2 ? leaf_grid<double, true, 2>() : mode == 1 ? leaf_grid<double, true, 1>() : leaf_grid<double, true, 0>();
    return mode == 2 ? leaf_grid<double, false, 2>() : mode == 1 ? leaf_grid<double, false, 1>() : leaf_grid<double, false, 0>();
  }
  if (noisy) return mode == 2 ? leaf_grid<float, true, 2>() : mode == 1 ? leaf_grid<float, true, 1>() : leaf_grid<float, true, 0>();
  return mode == 2 ? leaf_grid<float, false, 2>() : mode == 1 ? leaf_grid<float, false, 1>() : leaf_grid<float, false, 0>();
}

template void launch_group_mean_step<float>(float*, std::uint64_t, std::uint64_t,
                                            const std::uint32_t*, const std::uint32_t*,
                                            const std::uint32_t*, const std::uint32_t*,
                                            const StepPrologue<float>&, int, cudaStream_t);
template void launch_group_mean_step<double>(double*, std::uint64_t, std::uint64_t,
                                             const std::uint32_t*, const std::uint32_t*,
                                             const std::uint32_t*, const std::uint32_t*,
                                             const StepPrologue<double>&, int, cudaStream_t);

}  // namespace mb200
