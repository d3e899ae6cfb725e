// diag_kernel.cu -- TrialReport diagnostics and helpers on the GPU.
//
// record_round (protocols.hpp:68-84) needs, after every round:
//   distortion = pairwise_i( sum_j (theta_ij - ref_j)^2 ) / N   (core.hpp:111-126)
//   mean       = mean_of(vectors), pairwise over peers           (core.hpp:128-133)
//   drift      = sqrt(sum_j (mean_j-ref_j)^2) / max(sqrt(sum_j ref_j^2), 1e-300)
// The reference sums over j SEQUENTIALLY.  MOSHPIT_DIAG_EXACT reproduces that
// order (one dependent chain per peer: bit parity, slow at large D);
// MOSHPIT_DIAG_FAST sums fixed chunks in parallel and folds them in a fixed
// order (deterministic, ~1e-15 relative to the sequential sum).  Column means
// use the reference pairwise tree over peers in both modes, in fp64.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "blocktree.cuh"
#include "pairwise.cuh"

namespace mb200 {
namespace {

template <typename Acc>
struct AccOps;
template <>
struct AccOps<double> {
  __device__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ static double div(double a, double b) { return __ddiv_rn(a, b); }
};
template <>
struct AccOps<float> {
  __device__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ static float div(float a, float b) { return __fdiv_rn(a, b); }
};

// One thread per coordinate: pairwise tree over the (selected) rows.
template <typename T, typename Acc>
__global__ void colmean_kernel(const T* __restrict__ x, std::uint64_t n,
                               std::uint64_t ld, std::uint64_t dim,
                               const std::uint32_t* __restrict__ rows,
                               Acc* __restrict__ out) {
  const std::uint64_t j = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (j >= dim) return;
  auto ld_fn = [&](std::uint32_t i) -> Acc {
    const std::uint64_t r = rows ? rows[i] : i;
    return (Acc)x[r * ld + j];
  };
  const Acc s = pairwise_rt<Acc>(ld_fn, (std::uint32_t)n,
                                 [](Acc a, Acc b) { return AccOps<Acc>::add(a, b); },
                                 (Acc)0);
  out[j] = AccOps<Acc>::div(s, (Acc)n);
}

// Column means for peer counts n = 8 * 2^K (the configs' 256, 1024, 4096):
// the reference tree (n <= 8 summed sequentially from +0, else split at
// floor(n/2); core.hpp:72-81) is then a perfect binary tree over n/8
// sequential 8-row blocks, evaluated left to right with a K-level binary
// counter of pending left subtrees (block b merges with the pending sums at
// the levels where b has a 1 bit: left + right, exactly the tree's adds).
// Each thread owns one 16-byte column vector (4 fp32 or 2 fp64 columns) and
// streams its own 16-byte pieces of the block rows into shared memory with
// cp.async, kCmStages blocks ahead: no thread reads another's data, so the
// pipeline needs no barriers, and the registers hold only the K-level stack
// (the previous fully unrolled tree let the compiler hoist every row load:
// 255 registers and a 1.2 KB stack frame, 8 warps/SM, latency-bound).
// rows (optional): element i of the tree is row rows[i] -- the representative
// gather (RepRows): identical values, fewer distinct rows read from HBM.
template <typename T>
struct ColVec;
template <>
struct ColVec<float> {
  using V = float4;
  static constexpr int W = 4;
};
template <>
struct ColVec<double> {
  using V = double2;
  static constexpr int W = 2;
};

constexpr int kCmThreads = 128;
constexpr int kCmStages = 4;
constexpr int kCmMinK = 2, kCmMaxK = 9;  // n = 32 .. 4096 (the configs: 256, 1024, 4096)

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<std::uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One thread's view of the staged tree: its column vector, the row map, its
// 16-byte slots in the ring.  Block b (8 rows) lives in stage b % kCmStages.
// `Leaf` may transform each row's vector as it enters the tree (the fused
// Moshpit-SGD step below); NoLeaf leaves it alone.
struct NoLeaf {
  template <typename V>
  __device__ __forceinline__ void operator()(V&, std::uint32_t) {}
};

template <int K, typename T, typename Leaf = NoLeaf>
struct CmThread {
  using V = typename ColVec<T>::V;
  static constexpr int W = ColVec<T>::W;
  static constexpr int NB = 1 << K;
  const V* col;
  std::uint64_t ldv;
  const std::uint32_t* s_rows;  // null: row i is i
  V* mine;
  bool live;                    // this thread's column vector is inside the row
  Leaf leaf;

  __device__ __forceinline__ void issue(int b, int stage) const {
    if (b < NB && live) {
      V* dst = mine + stage * 8 * kCmThreads;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const std::uint32_t r = s_rows ? s_rows[b * 8 + q] : (std::uint32_t)(b * 8 + q);
        cp_async16(dst + q * kCmThreads, col + (std::uint64_t)r * ldv);
      }
    }
    cp_async_commit();  // empty groups keep the wait count uniform
  }
  // block base + OFF: refill the ring kCmStages - 1 blocks ahead, then the
  // block's sequential sum from +0 (core.hpp:74-77)
  template <int OFF>
  __device__ __forceinline__ void block(int base, double (&o)[W]) {
    issue(base + OFF + kCmStages - 1, (OFF + kCmStages - 1) % kCmStages);
    cp_async_wait<kCmStages - 1>();
    const V* src = mine + (OFF % kCmStages) * 8 * kCmThreads;
#pragma unroll
    for (int w = 0; w < W; ++w) o[w] = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      V e = src[q * kCmThreads];
      leaf(e, (std::uint32_t)((base + OFF) * 8 + q));
      const T* pe = reinterpret_cast<const T*>(&e);
#pragma unroll
      for (int w = 0; w < W; ++w) o[w] = __dadd_rn(o[w], (double)pe[w]);
    }
  }
};

// the subtree over 2^L blocks starting at block base + OFF, at compile time
template <int L, int OFF, class C>
__device__ __forceinline__ void cm_subtree(C& c, int base, double (&o)[C::W]) {
  constexpr int W = C::W;
  if constexpr (L == 0) {
    c.template block<OFF>(base, o);
  } else {
    double l[W], r[W];
    cm_subtree<L - 1, OFF>(c, base, l);
    cm_subtree<L - 1, OFF + (1 << (L - 1))>(c, base, r);
#pragma unroll
    for (int w = 0; w < W; ++w) o[w] = __dadd_rn(l[w], r[w]);
  }
}

// The whole tree for one thread: compile-time subtrees of 2^KS blocks, the
// top K - KS levels with a binary counter of pending left subtrees.
template <int K, class C>
__device__ __forceinline__ void cm_tree(C& c, double (&v)[C::W]) {
  constexpr int W = C::W;
  constexpr int KS = K < 3 ? K : 3, KT = K - KS, NS = 1 << KT;
  static_assert(KS >= 2 || KT == 0, "stage offsets need subtree bases % kCmStages == 0");
#pragma unroll
  for (int b = 0; b < kCmStages - 1; ++b) c.issue(b, b);
  double stk[KT > 0 ? KT : 1][W];
#pragma unroll 1
  for (int t = 0; t < NS; ++t) {
    cm_subtree<KS, 0>(c, t << KS, v);
    bool placed = false;
#pragma unroll
    for (int l = 0; l < KT; ++l) {
      if (!placed) {
        if ((t >> l) & 1) {
#pragma unroll
          for (int w = 0; w < W; ++w) v[w] = __dadd_rn(stk[l][w], v[w]);
        } else {
#pragma unroll
          for (int w = 0; w < W; ++w) stk[l][w] = v[w];
          placed = true;
        }
      }
    }
  }
  // after subtree NS - 1 (all bits set) v holds the whole tree
}

template <int K, typename T>
__global__ void __launch_bounds__(kCmThreads)
    colmean_staged(const T* __restrict__ x, std::uint64_t ld, std::uint64_t dim,
                   const std::uint32_t* __restrict__ rows, double* __restrict__ out) {
  using V = typename ColVec<T>::V;
  constexpr int W = ColVec<T>::W;
  constexpr int N = 8 << K;
  extern __shared__ __align__(16) unsigned char cm_smem[];
  V* const ring = reinterpret_cast<V*>(cm_smem);  // [stage][8 rows][kCmThreads]
  std::uint32_t* const s_rows =
      reinterpret_cast<std::uint32_t*>(ring + kCmStages * 8 * kCmThreads);
  if (rows) {
    for (int i = threadIdx.x; i < N; i += kCmThreads) s_rows[i] = rows[i];
    __syncthreads();
  }
  const std::uint64_t cv = blockIdx.x * (std::uint64_t)kCmThreads + threadIdx.x;
  if (cv * W >= dim) return;
  CmThread<K, T> c{reinterpret_cast<const V*>(x) + cv, ld / W, rows ? s_rows : nullptr,
                   ring + threadIdx.x, true, NoLeaf{}};
  double v[W];
  cm_tree<K>(c, v);
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (cv * W + w < dim) out[cv * W + w] = __ddiv_rn(v[w], (double)N);
}

// ---------------------------------------------------------------------------
// Noise-free Moshpit-SGD local step fused into hat theta = mean_of(post-step
// vectors) (optimizer.hpp:356-376): every row of the tree is stepped as it
// enters it -- g = c (theta - t), theta' = theta - gamma g, separately
// rounded, the standalone step kernel's arithmetic -- and written back; the
// tree then sums the post values.  One read and one write of the state
// instead of the step's read + write and the mean's read.
// ---------------------------------------------------------------------------
template <typename T>
struct StepLeafOp {
  using V = typename ColVec<T>::V;
  static constexpr int W = ColVec<T>::W;
  V c, t;
  T gamma;
  std::uint64_t cv, dim;
  V* out;  // this thread's column vector of row 0
  std::uint64_t ldv;
  bool live;
  T chk;

  __device__ __forceinline__ void operator()(V& e, std::uint32_t row) {
    if (!live) return;
    T* pe = reinterpret_cast<T*>(&e);
    const T* pc = reinterpret_cast<const T*>(&c);
    const T* pt = reinterpret_cast<const T*>(&t);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      if (cv * W + w >= dim) break;
      const T g = mul_rn(pc[w], sub_rn(pe[w], pt[w]));
      chk = add_rn(chk, mul_rn(g, T(0)));  // stays 0 unless some g is inf / NaN
      pe[w] = sub_rn(pe[w], mul_rn(gamma, g));
    }
    out[(std::uint64_t)row * ldv] = e;
  }
  __device__ static float sub_rn(float a, float b) { return __fsub_rn(a, b); }
  __device__ static float mul_rn(float a, float b) { return __fmul_rn(a, b); }
  __device__ static float add_rn(float a, float b) { return __fadd_rn(a, b); }
  __device__ static double sub_rn(double a, double b) { return __dsub_rn(a, b); }
  __device__ static double mul_rn(double a, double b) { return __dmul_rn(a, b); }
  __device__ static double add_rn(double a, double b) { return __dadd_rn(a, b); }
};

template <int K, typename T>
__global__ void __launch_bounds__(kCmThreads)
    step_colmean_staged(T* __restrict__ x, std::uint64_t ld, std::uint64_t dim,
                        double* __restrict__ hat, const T* __restrict__ curv,
                        const T* __restrict__ tgt, T gamma, std::uint32_t* nonfinite) {
  using V = typename ColVec<T>::V;
  constexpr int W = ColVec<T>::W;
  constexpr int N = 8 << K;
  extern __shared__ __align__(16) unsigned char cm_smem[];
  V* const ring = reinterpret_cast<V*>(cm_smem);
  const std::uint64_t cv = blockIdx.x * (std::uint64_t)kCmThreads + threadIdx.x;
  if (cv * W >= dim) return;
  const std::uint64_t ldv = ld / W;
  StepLeafOp<T> op;
  if (cv * W + W <= dim) {
    op.c = __ldg(reinterpret_cast<const V*>(curv) + cv);
    op.t = __ldg(reinterpret_cast<const V*>(tgt) + cv);
  } else {
    T* pc = reinterpret_cast<T*>(&op.c);
    T* pt = reinterpret_cast<T*>(&op.t);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      pc[w] = cv * W + w < dim ? curv[cv * W + w] : T(0);
      pt[w] = cv * W + w < dim ? tgt[cv * W + w] : T(0);
    }
  }
  op.gamma = gamma;
  op.cv = cv;
  op.dim = dim;
  op.out = reinterpret_cast<V*>(x) + cv;
  op.ldv = ldv;
  op.live = true;
  op.chk = T(0);
  CmThread<K, T, StepLeafOp<T>> c{reinterpret_cast<const V*>(x) + cv, ldv, nullptr,
                                  ring + threadIdx.x, true, op};
  double v[W];
  cm_tree<K>(c, v);
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (cv * W + w < dim) hat[cv * W + w] = __ddiv_rn(v[w], (double)N);
  if (c.leaf.chk != T(0)) atomicOr(nonfinite, 1u);
}

template <int K, typename T>
void launch_colmean_staged(const T* x, std::uint64_t ld, std::uint64_t dim,
                           const std::uint32_t* rows, double* out, cudaStream_t s) {
  constexpr int W = ColVec<T>::W;
  constexpr std::size_t smem =
      (std::size_t)kCmStages * 8 * kCmThreads * 16 + ((std::size_t)8 << K) * 4;
  static thread_local int attr_dev = -1;
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    MB_CUDA(cudaFuncSetAttribute(colmean_staged<K, T>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_dev = dev;
  }
  const std::uint64_t nv = (dim + W - 1) / W;
  colmean_staged<K, T><<<(unsigned)((nv + kCmThreads - 1) / kCmThreads), kCmThreads, smem, s>>>(
      x, ld, dim, rows, out);
}

// fp64 state, n = 256 / 1024: the tree fully unrolled at compile time, one
// 16-byte column vector (2 columns) per thread, no shared memory.  Measured
// against the staged form at C2 (1024 x 4 Mi fp64): 1.9-2.2 vs 2.6 ms with the
// representative gather, and beside the EXACT distortion on the other stream
// it leaves that kernel's CTAs room (the staged form's 68 KB of shared memory
// per CTA cost the EXACT record 2.6 ms per round).  The same unrolled form
// for fp32 state hoists every row load (255 registers, 1.2 KB of stack).
template <int N, typename T, typename Acc>
__device__ __forceinline__ void ctree(const typename ColVec<T>::V* __restrict__ col,
                                      std::uint64_t ldv, int base, const std::uint32_t* rows,
                                      Acc (&out)[ColVec<T>::W]) {
  constexpr int W = ColVec<T>::W;
  if constexpr (N <= 8) {
    typename ColVec<T>::V v[N];
#pragma unroll
    for (int q = 0; q < N; ++q)
      v[q] = __ldg(col + (std::uint64_t)(rows ? rows[base + q] : (std::uint32_t)(base + q)) * ldv);
#pragma unroll
    for (int w = 0; w < W; ++w) out[w] = Acc(0);
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const T* e = reinterpret_cast<const T*>(&v[q]);
#pragma unroll
      for (int w = 0; w < W; ++w) out[w] = AccOps<Acc>::add(out[w], (Acc)e[w]);
    }
  } else {
    Acc a[W], b[W];
    ctree<N / 2, T, Acc>(col, ldv, base, rows, a);
    ctree<N - N / 2, T, Acc>(col, ldv, base + N / 2, rows, b);
#pragma unroll
    for (int w = 0; w < W; ++w) out[w] = AccOps<Acc>::add(a[w], b[w]);
  }
}

// rows (optional): element i of the tree is row rows[i] -- the representative
// gather (RepRows): identical values, fewer distinct rows read from HBM.
template <int N, typename T, typename Acc>
__global__ void __launch_bounds__(128)
    colmean_unrolled(const T* __restrict__ x, std::uint64_t ld, std::uint64_t dim,
                     const std::uint32_t* __restrict__ rows, Acc* __restrict__ out) {
  using V = typename ColVec<T>::V;
  constexpr int W = ColVec<T>::W;
  __shared__ std::uint32_t s_rows[N];
  if (rows) {
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_rows[i] = rows[i];
    __syncthreads();
  }
  const std::uint64_t cv = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (cv * W >= dim) return;
  Acc s[W];
  ctree<N, T, Acc>(reinterpret_cast<const V*>(x) + cv, ld / W, 0, rows ? s_rows : nullptr, s);
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (cv * W + w < dim) out[cv * W + w] = AccOps<Acc>::div(s[w], (Acc)N);
}

template <typename T>
bool try_colmean_staged(const T* x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                        const std::uint32_t* rows, double* out, cudaStream_t s) {
  constexpr int W = ColVec<T>::W;
  if (ld % W != 0 || reinterpret_cast<std::uintptr_t>(x) % 16 != 0) return false;
  if (n < (8u << kCmMinK) || (n & (n - 1)) != 0 || n > (8u << kCmMaxK)) return false;
  switch (__builtin_ctzll(n) - 3) {
    case 2: launch_colmean_staged<2, T>(x, ld, dim, rows, out, s); break;
    case 3: launch_colmean_staged<3, T>(x, ld, dim, rows, out, s); break;
    case 4: launch_colmean_staged<4, T>(x, ld, dim, rows, out, s); break;
    case 5: launch_colmean_staged<5, T>(x, ld, dim, rows, out, s); break;
    case 6: launch_colmean_staged<6, T>(x, ld, dim, rows, out, s); break;
    case 7: launch_colmean_staged<7, T>(x, ld, dim, rows, out, s); break;
    case 8: launch_colmean_staged<8, T>(x, ld, dim, rows, out, s); break;
    case 9: launch_colmean_staged<9, T>(x, ld, dim, rows, out, s); break;
    default: return false;
  }
  MB_LAUNCH_CHECK();
  return true;
}

// EXACT: per peer, sequential over j exactly as core.hpp:118-122.  The only
// serial part of the reference order is the add chain of each peer; the
// squared differences are independent.  A CTA owns P peers: warps 1..7 stage
// (x_ij - ref_j)^2 for a tile of kExK columns of its P rows into shared memory
// (coalesced row segments, computed with the reference's separate rounding),
// while lanes 0..P-1 of warp 0 run the P add chains over the previous tile.
// Cost ~ D x (DADD + LDS issue) per chain instead of D dependent global loads.
constexpr int kExThreads = 256;
constexpr int kExProducers = kExThreads - 32;
constexpr int kExK = 512;

template <int P>
constexpr std::size_t exact_smem() {
  return 2ull * P * (kExK + 1) * sizeof(double);
}

// acc[i] (in/out when `accumulate`, else written): the running j-sum of peer i.
template <typename T, int P>
__global__ void __launch_bounds__(kExThreads)
    dist_exact_tiled(const T* __restrict__ x, std::uint64_t n, std::uint64_t ld,
                     std::uint64_t dim, const double* __restrict__ ref,
                     double* __restrict__ acc, int accumulate,
                     const std::uint32_t* __restrict__ list,
                     const std::uint32_t* __restrict__ list_count) {
  extern __shared__ double sm_ex[];
  // chains of rows list[p0 .. p0+P) (or rows p0 .. p0+P): acc is by row id
  const std::uint64_t rows = list ? *list_count : n;
  const std::uint64_t p0 = (std::uint64_t)blockIdx.x * P;
  if (p0 >= rows) return;  // uniform across the CTA
  n = rows;
  auto row_of = [&](std::uint64_t q) -> std::uint64_t { return list ? list[q] : q; };
  const int tid = threadIdx.x;
  double a = 0.0;
  if (tid < P && p0 + tid < n && accumulate) a = acc[row_of(p0 + tid)];
  const std::uint64_t ntiles = (dim + kExK - 1) / kExK;
  // all of a producer thread's loads for a tile are issued before any use
  // (the latency of one batch per tile, hidden behind the chains' tile)
  auto produce = [&](std::uint64_t t, int buf) {
    const std::uint64_t j0 = t * kExK;
    constexpr int kE = P * kExK;
    constexpr int kIt = (kE + kExProducers - 1) / kExProducers;
    double xv[kIt], rv[kIt];
#pragma unroll
    for (int u = 0; u < kIt; ++u) {
      const int e = tid - 32 + u * kExProducers;
      const int q = e / kExK, k = e % kExK;
      const std::uint64_t j = j0 + k, i = p0 + q;
      const bool ok = e < kE && j < dim && i < n;
      // padding: (0 - 0)^2 = +0.0 added to a sum of squares is bit-neutral
      xv[u] = ok ? (double)x[row_of(i) * ld + j] : 0.0;
      rv[u] = ok ? ref[j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kIt; ++u) {
      const int e = tid - 32 + u * kExProducers;
      if (e < kE) {
        const int q = e / kExK, k = e % kExK;
        const double diff = __dsub_rn(xv[u], rv[u]);
        sm_ex[(buf * P + q) * (kExK + 1) + k] = __dmul_rn(diff, diff);
      }
    }
  };
  if (tid >= 32 && ntiles) produce(0, 0);
  __syncthreads();
  for (std::uint64_t t = 0; t < ntiles; ++t) {
    const int buf = (int)(t & 1);
    if (tid >= 32) {
      if (t + 1 < ntiles) produce(t + 1, buf ^ 1);
    } else if (tid < P) {
      const double* row = sm_ex + (buf * P + tid) * (kExK + 1);
#pragma unroll 16
      for (int k = 0; k < kExK; ++k) a = __dadd_rn(a, row[k]);
    }
    __syncthreads();
  }
  if (tid < P && p0 + tid < n) acc[row_of(p0 + tid)] = a;
}

template <typename T, int P>
void launch_dist_exact_p(const T* x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                         const double* ref, double* acc, int accumulate, cudaStream_t s,
                         const std::uint32_t* list, const std::uint32_t* count) {
  static bool attr = false;
  if (!attr) {
    MB_CUDA(cudaFuncSetAttribute(dist_exact_tiled<T, P>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)exact_smem<P>()));
    attr = true;
  }
  const unsigned blocks = (unsigned)((n + P - 1) / P);
  dist_exact_tiled<T, P><<<blocks, kExThreads, exact_smem<P>(), s>>>(x, n, ld, dim, ref, acc,
                                                                   accumulate, list, count);
}

// list / count: chains only for the representative rows (RepRows); acc by row.
template <typename T>
void launch_dist_exact(const T* x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                       const double* ref, double* acc, int accumulate, cudaStream_t s,
                       const std::uint32_t* list = nullptr, const std::uint32_t* count = nullptr) {
  // rows per CTA: enough CTAs to spread the chains over the SMs
  const int P = n >= 2048 ? 8 : n >= 1024 ? 4 : n >= 512 ? 2 : 1;
  switch (P) {
    case 1: launch_dist_exact_p<T, 1>(x, n, ld, dim, ref, acc, accumulate, s, list, count); break;
    case 2: launch_dist_exact_p<T, 2>(x, n, ld, dim, ref, acc, accumulate, s, list, count); break;
    case 4: launch_dist_exact_p<T, 4>(x, n, ld, dim, ref, acc, accumulate, s, list, count); break;
    default: launch_dist_exact_p<T, 8>(x, n, ld, dim, ref, acc, accumulate, s, list, count);
  }
  MB_LAUNCH_CHECK();
}

// drift, EXACT (protocols.hpp:75-81 in order): the two j-chains
// (mean_j - ref_j)^2 and ref_j^2 on lanes 0 and 1 of warp 0, the squares
// staged by warps 1..7.  acc2[0..1] running sums (in/out when `accumulate`).
__global__ void __launch_bounds__(kExThreads)
    drift_exact_tiled(const double* __restrict__ mean, const double* __restrict__ ref,
                      std::uint64_t dim, double* __restrict__ acc2, int accumulate) {
  extern __shared__ double sm_ex[];
  const int tid = threadIdx.x;
  double a = 0.0;
  if (tid < 2 && accumulate) a = acc2[tid];
  const std::uint64_t ntiles = (dim + kExK - 1) / kExK;
  auto produce = [&](std::uint64_t t, int buf) {
    const std::uint64_t j0 = t * kExK;
    constexpr int kIt = (kExK + kExProducers - 1) / kExProducers;
    double mv[kIt], rv[kIt];
#pragma unroll
    for (int u = 0; u < kIt; ++u) {
      const int k = tid - 32 + u * kExProducers;
      const std::uint64_t j = j0 + k;
      const bool ok = k < kExK && j < dim;
      mv[u] = ok ? mean[j] : 0.0;
      rv[u] = ok ? ref[j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kIt; ++u) {
      const int k = tid - 32 + u * kExProducers;
      if (k < kExK) {
        const double dm = __dsub_rn(mv[u], rv[u]);
        sm_ex[(buf * 2 + 0) * (kExK + 1) + k] = __dmul_rn(dm, dm);
        sm_ex[(buf * 2 + 1) * (kExK + 1) + k] = __dmul_rn(rv[u], rv[u]);
      }
    }
  };
  if (tid >= 32 && ntiles) produce(0, 0);
  __syncthreads();
  for (std::uint64_t t = 0; t < ntiles; ++t) {
    const int buf = (int)(t & 1);
    if (tid >= 32) {
      if (t + 1 < ntiles) produce(t + 1, buf ^ 1);
    } else if (tid < 2) {
      const double* row = sm_ex + (buf * 2 + tid) * (kExK + 1);
#pragma unroll 16
      for (int k = 0; k < kExK; ++k) a = __dadd_rn(a, row[k]);
    }
    __syncthreads();
  }
  if (tid < 2) acc2[tid] = a;
}

void launch_drift_exact(const double* mean, const double* ref, std::uint64_t dim, double* acc2,
                        int accumulate, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    MB_CUDA(cudaFuncSetAttribute(drift_exact_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)exact_smem<2>()));
    attr = true;
  }
  drift_exact_tiled<<<1, kExThreads, exact_smem<2>(), s>>>(mean, ref, dim, acc2, accumulate);
  MB_LAUNCH_CHECK();
}

constexpr int kRedThreads = 256;
// FAST partial chunk: the distortion's per-row j-sum is taken over chunks of
// kChunk columns (one CTA of the one-pass kernel each), folded in chunk order.
constexpr std::uint64_t kChunk = 1 << 12;

__device__ double block_sum_fixed(double v) {
  __shared__ double buf[kRedThreads];
  buf[threadIdx.x] = v;
  __syncthreads();
  for (int s = kRedThreads / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) buf[threadIdx.x] = __dadd_rn(buf[threadIdx.x], buf[threadIdx.x + s]);
    __syncthreads();
  }
  const double r = buf[0];
  __syncthreads();
  return r;
}

__global__ void fold_rows(const double* __restrict__ partial, std::uint64_t n,
                          std::uint64_t nch, double* __restrict__ sq,
                          const std::uint32_t* __restrict__ rep) {
  const std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const std::uint64_t r = rep ? rep[i] : i;  // identical rows share their partials
  double acc = 0.0;
  for (std::uint64_t c = 0; c < nch; ++c) acc = __dadd_rn(acc, partial[r * nch + c]);
  sq[i] = acc;
}

// Representatives of a round (RepRows, common.cuh): one thread per group.
__global__ void build_reps_kernel(const std::uint32_t* __restrict__ members,
                                  const std::uint32_t* __restrict__ goff,
                                  const std::uint8_t* __restrict__ gvoid,
                                  const std::uint32_t* __restrict__ counts,
                                  std::uint32_t* __restrict__ rep, std::uint32_t* __restrict__ list,
                                  std::uint32_t* __restrict__ count, int list_voided) {
  const std::uint32_t ng = counts[0];
  for (std::uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < ng;
       g += gridDim.x * blockDim.x) {
    const std::uint32_t b = goff[g], e = goff[g + 1];
    if (!gvoid[g]) {  // averaged: every member now equals the first member's row
      const std::uint32_t first = members[b];
      for (std::uint32_t k = b; k < e; ++k) rep[members[k]] = first;
      list[atomicAdd(count, 1u)] = first;
    } else {  // voided: the members keep their own rows
      for (std::uint32_t k = b; k < e; ++k) {
        rep[members[k]] = members[k];
        if (list_voided) list[atomicAdd(count, 1u)] = members[k];
      }
    }
  }
}

// FAST row partials of every member of an averaged group from its
// representative's (the rows are identical): afterwards every row's slot
// holds its own partials, so a later record can skip the rows it knows are
// unchanged (the voided rows of the next round).
__global__ void scatter_rep_partials(double* __restrict__ partial,
                                     const std::uint32_t* __restrict__ rep, std::uint64_t n,
                                     std::uint64_t nch) {
  const std::uint64_t total = n * nch;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t i = e / nch, c = e % nch;
    const std::uint32_t r = rep[i];
    if (r != i) partial[i * nch + c] = partial[(std::uint64_t)r * nch + c];
  }
}

// in-place expansion sq[i] = sq[rep[i]] (representatives are their own rep)
__global__ void expand_reps(double* __restrict__ sq, const std::uint32_t* __restrict__ rep,
                            std::uint64_t n) {
  const std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (i < n && rep[i] != i) sq[i] = sq[rep[i]];
}

// pairwise over peers, / n  (core.hpp:125): the reference tree evaluated by
// one CTA (blocktree.cuh, bit-identical to the sequential evaluation) for
// n <= 8192, one thread above that.
constexpr int kFinThreads = 256;
__global__ void __launch_bounds__(kFinThreads)
    finish_distortion(const double* __restrict__ sq, std::uint64_t n, double* __restrict__ out) {
  __shared__ double lvl[2 * kBlockTreeMaxNodes];
  if (n == 0) {
    if (threadIdx.x == 0) *out = 0.0;
    return;
  }
  if (n <= 8192) {
    auto ld_fn = [&](std::uint32_t i) { return sq[i]; };
    const double s = pairwise_block(ld_fn, (std::uint32_t)n, lvl);
    if (threadIdx.x == 0) *out = __ddiv_rn(s, (double)n);
    return;
  }
  if (threadIdx.x != 0) return;
  auto ld_fn = [&](std::uint32_t i) { return sq[i]; };
  const double s = pairwise_rt<double>(ld_fn, (std::uint32_t)n,
                                       [](double a, double b) { return __dadd_rn(a, b); }, 0.0);
  *out = __ddiv_rn(s, (double)n);
}

__global__ void drift_fast_partial(const double* __restrict__ mean,
                                   const double* __restrict__ ref,
                                   std::uint64_t dim, double* __restrict__ partial) {
  const std::uint64_t c = blockIdx.x;
  const std::uint64_t lo = c * kChunk, hi = lo + kChunk < dim ? lo + kChunk : dim;
  double a = 0.0, b = 0.0;
  for (std::uint64_t j = lo + threadIdx.x; j < hi; j += kRedThreads) {
    const double dm = __dsub_rn(mean[j], ref[j]);
    a = __dadd_rn(a, __dmul_rn(dm, dm));
    b = __dadd_rn(b, __dmul_rn(ref[j], ref[j]));
  }
  const double sa = block_sum_fixed(a);
  const double sb = block_sum_fixed(b);
  if (threadIdx.x == 0) {
    partial[2 * c] = sa;
    partial[2 * c + 1] = sb;
  }
}

// The two chunk folds in chunk order by one thread, the partials staged in
// shared memory by the whole CTA first (a lone thread's global loads were
// ~80 us of latency per record on the drift stream, its critical path).
constexpr int kDriftFinThreads = 256, kDriftFinBatch = 1024;
__global__ void __launch_bounds__(kDriftFinThreads)
    drift_fast_finish(const double* __restrict__ partial, std::uint64_t nch,
                      double* __restrict__ out) {
  __shared__ double buf[2 * kDriftFinBatch];
  double a = 0.0, b = 0.0;
  for (std::uint64_t c0 = 0; c0 < nch; c0 += kDriftFinBatch) {
    const std::uint64_t m = nch - c0 < (std::uint64_t)kDriftFinBatch ? nch - c0 : kDriftFinBatch;
    for (std::uint64_t q = threadIdx.x; q < 2 * m; q += kDriftFinThreads)
      buf[q] = partial[2 * c0 + q];
    __syncthreads();
    if (threadIdx.x == 0) {
      for (std::uint64_t c = 0; c < m; ++c) {
        a = __dadd_rn(a, buf[2 * c]);
        b = __dadd_rn(b, buf[2 * c + 1]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = __ddiv_rn(__dsqrt_rn(a), fmax(__dsqrt_rn(b), 1e-300));
}

__device__ __forceinline__ std::uint64_t splitmix64_dev(std::uint64_t s) {
  std::uint64_t z = s + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_synthetic_kernel(T* __restrict__ x, std::uint64_t n,
                                      std::uint64_t dim, std::uint64_t ld,
                                      std::uint64_t seed, std::uint64_t col0) {
  const std::uint64_t total = n * dim;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
       e < total; e += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t i = e / dim, j = e % dim;
    const std::uint64_t z = splitmix64_dev(seed ^ (i << 32) ^ (col0 + j));
    x[i * ld + j] = (T)((double)(z >> 40) * 0x1.0p-24);
  }
}

template <typename T>
__global__ void broadcast_rows_kernel(T* __restrict__ dst, std::uint64_t ld,
                                      const T* __restrict__ row, std::uint64_t n,
                                      std::uint64_t dim) {
  const std::uint64_t total = n * dim;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
       e < total; e += (std::uint64_t)gridDim.x * blockDim.x)
    dst[(e / dim) * ld + e % dim] = row[e % dim];
}

// ---- slab-streamed variants: the j-sums continue across D-slabs --------
// FAST: block (c, y) sums chunk c of kFastRows rows in a fixed order (chunk
// offset c0 in the row's partials, so the slab-streamed and resident paths
// agree): each thread takes 16-byte vectors (4 fp32 / 2 fp64 coordinates)
// 256 vectors apart and sums its elements sequentially, one chain per row,
// then the block tree of block_sum_fixed per row.  The rows of a block share
// every reference load (the fp64 reference is twice the bytes of an fp32
// row: one row per block read 12 bytes per fp32 coordinate through L2).
#ifndef MB_FAST_ROWS
#define MB_FAST_ROWS 4
#endif
constexpr int kFastRows = MB_FAST_ROWS;  // rows per block (bits do not depend on it;
// C2 round + FAST record 6.97 ms at 4, 7.60 at 16, 8.24 at 8: profiles/r02/diag/fast_rows.txt)

template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    dist_rows_fast_off(const T* __restrict__ x, std::uint64_t ld, std::uint64_t dim,
                       const double* __restrict__ ref, std::uint64_t nch_total,
                       std::uint64_t c0, double* __restrict__ partial, std::uint64_t n,
                       const std::uint32_t* __restrict__ list,
                       const std::uint32_t* __restrict__ list_count) {
  using V = typename ColVec<T>::V;
  constexpr int W = ColVec<T>::W;
  __shared__ double buf[kFastRows][kRedThreads];
  const std::uint64_t rows = list ? *list_count : n;
  const std::uint64_t c = blockIdx.x;
  const std::uint64_t lo = c * kChunk, hi = lo + kChunk < dim ? lo + kChunk : dim;
  const bool vec = (ld % W == 0) && (reinterpret_cast<std::uintptr_t>(x) % 16 == 0);
  for (std::uint64_t y0 = (std::uint64_t)blockIdx.y * kFastRows; y0 < rows;
       y0 += (std::uint64_t)gridDim.y * kFastRows) {
    const T* rp[kFastRows];
    std::uint64_t ri[kFastRows];
#pragma unroll
    for (int r = 0; r < kFastRows; ++r) {
      const std::uint64_t y = y0 + r < rows ? y0 + r : y0;  // short tail: repeat, not stored
      ri[r] = list ? list[y] : y;
      rp[r] = x + ri[r] * ld;
    }
    double acc[kFastRows];
#pragma unroll
    for (int r = 0; r < kFastRows; ++r) acc[r] = 0.0;
#pragma unroll 2
    for (std::uint64_t j = lo + (std::uint64_t)threadIdx.x * W; j < hi; j += kRedThreads * W) {
      const bool whole = vec && j + W <= hi;
      double rf[W];
      if (j + W <= hi) {  // ref: a cudaMalloc'd fp64 vector, j a multiple of W
#pragma unroll
        for (int w = 0; w < W; w += 2) {
          const double2 r2 = __ldg(reinterpret_cast<const double2*>(ref + j + w));
          rf[w] = r2.x;
          rf[w + 1] = r2.y;
        }
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) rf[w] = j + w < hi ? __ldg(ref + j + w) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < kFastRows; ++r) {
        T e[W];
        if (whole) {
          const V v = __ldg(reinterpret_cast<const V*>(rp[r] + j));
#pragma unroll
          for (int w = 0; w < W; ++w) e[w] = reinterpret_cast<const T*>(&v)[w];
        } else {
#pragma unroll
          for (int w = 0; w < W; ++w) e[w] = j + w < hi ? rp[r][j + w] : T(0);
        }
#pragma unroll
        for (int w = 0; w < W; ++w) {
          if (j + w >= hi) break;
          const double diff = __dsub_rn((double)e[w], rf[w]);
          acc[r] = __dadd_rn(acc[r], __dmul_rn(diff, diff));
        }
      }
    }
    // block_sum_fixed's tree, all rows at once
#pragma unroll
    for (int r = 0; r < kFastRows; ++r) buf[r][threadIdx.x] = acc[r];
    __syncthreads();
    for (int st = kRedThreads / 2; st > 0; st >>= 1) {
      if ((int)threadIdx.x < st) {
#pragma unroll
        for (int r = 0; r < kFastRows; ++r)
          buf[r][threadIdx.x] = __dadd_rn(buf[r][threadIdx.x], buf[r][threadIdx.x + st]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < kFastRows; ++r)
      if ((int)threadIdx.x == r && y0 + r < rows) partial[ri[r] * nch_total + c0 + c] = buf[r][0];
    __syncthreads();
  }
}

__global__ void drift_fast_partial_off(const double* __restrict__ mean,
                                       const double* __restrict__ ref, std::uint64_t dim,
                                       std::uint64_t c0, double* __restrict__ partial) {
  const std::uint64_t c = blockIdx.x;
  const std::uint64_t lo = c * kChunk, hi = lo + kChunk < dim ? lo + kChunk : dim;
  double a = 0.0, b = 0.0;
  for (std::uint64_t j = lo + threadIdx.x; j < hi; j += kRedThreads) {
    const double dm = __dsub_rn(mean[j], ref[j]);
    a = __dadd_rn(a, __dmul_rn(dm, dm));
    b = __dadd_rn(b, __dmul_rn(ref[j], ref[j]));
  }
  const double sa = block_sum_fixed(a);
  const double sb = block_sum_fixed(b);
  if (threadIdx.x == 0) {
    partial[2 * (c0 + c)] = sa;
    partial[2 * (c0 + c) + 1] = sb;
  }
}

__global__ void drift_finish_acc(const double* __restrict__ acc2, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  *out = __ddiv_rn(__dsqrt_rn(acc2[0]), fmax(__dsqrt_rn(acc2[1]), 1e-300));
}

unsigned grid_for(std::uint64_t work, unsigned threads) {
  std::uint64_t b = (work + threads - 1) / threads;
  if (b > 148ull * 64) b = 148ull * 64;
  return (unsigned)(b ? b : 1);
}

}  // namespace

std::uint64_t diag_chunk() { return kChunk; }

// grid rows (groups of kFastRows rows) for the FAST partials: every group
// of the n rows, or, over a representative list (its length is on the
// device), ~2 waves of CTAs looping over the groups (1, 4 and 16 waves
// measured the same)
unsigned fast_rows_grid(std::uint64_t n, std::uint64_t nch, bool listed) {
  const std::uint64_t groups = (n + kFastRows - 1) / kFastRows;
  if (!listed) return (unsigned)groups;
  static const std::uint64_t waves = [] {
    const char* e = std::getenv("MOSHPIT_FAST_ROW_WAVES");
    return (std::uint64_t)(e ? std::max(1, std::atoi(e)) : 2);
  }();
  const std::uint64_t y = std::max<std::uint64_t>(1, waves * 2368 / std::max<std::uint64_t>(nch, 1));
  return (unsigned)std::min<std::uint64_t>(groups, y);
}

template <typename T>
void launch_dist_slab(const T* x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                      const double* ref, int exact, double* acc, double* partial,
                      std::uint64_t nch_total, std::uint64_t c0, cudaStream_t s,
                      const RepRows* reps) {
  if (n == 0 || dim == 0) return;
  const std::uint32_t* list = reps ? reps->list : nullptr;
  const std::uint32_t* count = reps ? reps->count : nullptr;
  if (exact) {
    launch_dist_exact<T>(x, n, ld, dim, ref, acc, 1, s, list, count);
    return;
  } else {
    const std::uint64_t nch = (dim + kChunk - 1) / kChunk;
    const unsigned gy = fast_rows_grid(n, nch, list != nullptr);
    dist_rows_fast_off<T><<<dim3((unsigned)nch, gy), kRedThreads, 0, s>>>(
        x, ld, dim, ref, nch_total, c0, partial, n, list, count);
  }
  MB_LAUNCH_CHECK();
}

void launch_build_reps(const std::uint32_t* members, const std::uint32_t* goff,
                       const std::uint8_t* gvoid, const std::uint32_t* counts, std::uint64_t n,
                       std::uint32_t* rep, std::uint32_t* list, std::uint32_t* count,
                       cudaStream_t s, int list_voided) {
  MB_CUDA(cudaMemsetAsync(count, 0, 4, s));
  build_reps_kernel<<<(unsigned)std::max<std::uint64_t>(1, (n + 255) / 256), 256, 0, s>>>(
      members, goff, gvoid, counts, rep, list, count, list_voided);
  MB_LAUNCH_CHECK();
}

void launch_drift_slab(const double* mean, const double* ref, std::uint64_t dim, int exact,
                       double* acc2, double* partial, std::uint64_t c0, cudaStream_t s) {
  if (dim == 0) return;
  if (exact) {
    launch_drift_exact(mean, ref, dim, acc2, 1, s);
    return;
  } else {
    const std::uint64_t nch = (dim + kChunk - 1) / kChunk;
    drift_fast_partial_off<<<(unsigned)nch, kRedThreads, 0, s>>>(mean, ref, dim, c0, partial);
  }
  MB_LAUNCH_CHECK();
}

// Final reductions of the slab-streamed diagnostics.
void launch_diag_finish(std::uint64_t n, std::uint64_t nch_total, int exact, double* acc,
                        double* row_partial, double* acc2, double* drift_partial,
                        double* dist_out, double* drift_out, cudaStream_t s,
                        const std::uint32_t* rep) {
  if (!exact) {
    fold_rows<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(row_partial, n, nch_total, acc, rep);
    MB_LAUNCH_CHECK();
  } else if (rep) {
    expand_reps<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(acc, rep, n);
    MB_LAUNCH_CHECK();
  }
  finish_distortion<<<1, kFinThreads, 0, s>>>(acc, n, dist_out);
  MB_LAUNCH_CHECK();
  if (drift_out) {
    if (exact)
      drift_finish_acc<<<1, 1, 0, s>>>(acc2, drift_out);
    else
      drift_fast_finish<<<1, kDriftFinThreads, 0, s>>>(drift_partial, nch_total, drift_out);
    MB_LAUNCH_CHECK();
  }
}

template void launch_dist_slab<float>(const float*, std::uint64_t, std::uint64_t, std::uint64_t,
                                      const double*, int, double*, double*, std::uint64_t,
                                      std::uint64_t, cudaStream_t, const RepRows*);
template void launch_dist_slab<double>(const double*, std::uint64_t, std::uint64_t,
                                       std::uint64_t, const double*, int, double*, double*,
                                       std::uint64_t, std::uint64_t, cudaStream_t,
                                       const RepRows*);

std::size_t diag_partial_elems(std::uint64_t n, std::uint64_t dim) {
  const std::uint64_t nch = (dim + kChunk - 1) / kChunk;
  const std::uint64_t a = n * (nch ? nch : 1), b = 2 * (nch ? nch : 1);
  return a > b ? a : b;
}

namespace {

template <int K, typename T>
void launch_step_colmean_k(T* x, std::uint64_t ld, std::uint64_t dim, double* hat,
                           const T* curv, const T* tgt, T gamma, std::uint32_t* nonfinite,
                           unsigned grid, cudaStream_t s) {
  constexpr std::size_t smem = (std::size_t)kCmStages * 8 * kCmThreads * 16;
  static thread_local int attr_dev = -1;
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    MB_CUDA(cudaFuncSetAttribute(step_colmean_staged<K, T>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_dev = dev;
  }
  step_colmean_staged<K, T><<<grid, kCmThreads, smem, s>>>(x, ld, dim, hat, curv, tgt, gamma,
                                                           nonfinite);
}

}  // namespace

template <typename T>
bool launch_step_colmean(T* x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                         const T* curv, const T* tgt, T gamma, double coord_std, int philox,
                         std::uint64_t seed, std::uint64_t step_no, std::uint32_t* nonfinite,
                         double* noise_partial, std::uint64_t partial_slots, double* hat,
                         cudaStream_t s) {
  constexpr int W = ColVec<T>::W;
  (void)coord_std, (void)seed, (void)step_no, (void)noise_partial, (void)partial_slots;
  // noise-free steps only: with the Philox rounds the fused kernel (its tree
  // stack plus the generator at 12 warps/SM) measured 3.6 ms at C4 against
  // 1.9 + 0.6 ms for the vectorised step kernel + the staged mean
  // (profiles/r02/c4diag_launches_*)
  if (philox || dim == 0) return false;
  if (ld % W != 0 || reinterpret_cast<std::uintptr_t>(x) % 16 != 0) return false;
  if (reinterpret_cast<std::uintptr_t>(curv) % 16 != 0 ||
      reinterpret_cast<std::uintptr_t>(tgt) % 16 != 0)
    return false;
  if (n < (8u << kCmMinK) || (n & (n - 1)) != 0 || n > (8u << kCmMaxK)) return false;
  const unsigned grid = (unsigned)(((dim + W - 1) / W + kCmThreads - 1) / kCmThreads);
  switch (__builtin_ctzll(n) - 3) {
    case 2: launch_step_colmean_k<2, T>(x, ld, dim, hat, curv, tgt, gamma, nonfinite, grid, s); break;
    case 3: launch_step_colmean_k<3, T>(x, ld, dim, hat, curv, tgt, gamma, nonfinite, grid, s); break;
    case 4: launch_step_colmean_k<4, T>(x, ld, dim, hat, curv, tgt, gamma, nonfinite, grid, s); break;
    case 5: launch_step_colmean_k<5, T>(x, ld, dim, hat, curv, tgt, gamma, nonfinite, grid, s); break;
    case 6: launch_step_colmean_k<6, T>(x, ld, dim, hat, curv, tgt, gamma, nonfinite, grid, s); break;
    case 7: launch_step_colmean_k<7, T>(x, ld, dim, hat, curv, tgt, gamma, nonfinite, grid, s); break;
    case 8: launch_step_colmean_k<8, T>(x, ld, dim, hat, curv, tgt, gamma, nonfinite, grid, s); break;
    default: launch_step_colmean_k<9, T>(x, ld, dim, hat, curv, tgt, gamma, nonfinite, grid, s); break;
  }
  MB_LAUNCH_CHECK();
  return true;
}

template bool launch_step_colmean<float>(float*, std::uint64_t, std::uint64_t, std::uint64_t,
                                         const float*, const float*, float, double, int,
                                         std::uint64_t, std::uint64_t, std::uint32_t*, double*,
                                         std::uint64_t, double*, cudaStream_t);
template bool launch_step_colmean<double>(double*, std::uint64_t, std::uint64_t,
                                          std::uint64_t, const double*, const double*, double,
                                          double, int, std::uint64_t, std::uint64_t,
                                          std::uint32_t*, double*, std::uint64_t, double*,
                                          cudaStream_t);

template <typename T, typename Acc>
void launch_colmean(const T* x, std::uint64_t n, std::uint64_t ld,
                    std::uint64_t dim, const std::uint32_t* rows, Acc* out,
                    cudaStream_t s, bool rows_optional) {
  if (dim == 0 || n == 0) return;
  // fp64 accumulation (the diagnostics) for n = 8 * 2^K: the staged tree
  if constexpr (std::is_same<Acc, double>::value) {
    // the representative gather: the fp32 column means read every row of
    // the tree either way; the gather trades HBM bytes for L2 hits
    // (MOSHPIT_REP_GATHER_F32=0 reads the rows themselves)
    static const bool gather32 = [] {
      const char* e = std::getenv("MOSHPIT_REP_GATHER_F32");
      return !e || std::atoi(e) != 0;
    }();
    const std::uint32_t* g =
        (rows_optional && !std::is_same<T, double>::value && !gather32) ? nullptr : rows;
    if constexpr (std::is_same<T, double>::value) {
      if (ld % 2 == 0 && reinterpret_cast<std::uintptr_t>(x) % 16 == 0 && (n == 256 || n == 1024)) {
        const unsigned blocks = (unsigned)(((dim + 1) / 2 + 127) / 128);
        if (n == 256) colmean_unrolled<256, T, Acc><<<blocks, 128, 0, s>>>(x, ld, dim, g, out);
        else colmean_unrolled<1024, T, Acc><<<blocks, 128, 0, s>>>(x, ld, dim, g, out);
        MB_LAUNCH_CHECK();
        return;
      }
    }
    if (try_colmean_staged<T>(x, n, ld, dim, g, out, s)) return;
  }
  const unsigned threads = 128;
  colmean_kernel<T, Acc><<<(unsigned)((dim + threads - 1) / threads), threads, 0, s>>>(
      x, n, ld, dim, rows, out);
  MB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// fp32 column means over the representative map by EXACT sums.  The tree's
// leaves are fp32 values widened to fp64; every partial sum of them (any
// subset, any order) is an integer multiple of 2^lo (lo: the smallest ulp
// exponent among the column's nonzero values) bounded by n * 2^hi (hi: the
// largest |value| < 2^hi), so when hi + ceil(log2 n) - lo <= 53 every add of
// the reference tree (core.hpp:72-81) is exact and the tree's result equals
// the exact sum -- which the sum over the DISTINCT rows with their
// multiplicities (count * value is exact in fp64) also computes.  Same bits,
// but each distinct row is read once (C2 after a round: ~300 of 1024) instead
// of a tree leaf per row.  Columns that fail the bound (or hold Inf/NaN) are
// listed and run the tree itself.
// ---------------------------------------------------------------------------
namespace {

__global__ void cs_mult(const std::uint32_t* __restrict__ rep, std::uint64_t n,
                        std::uint32_t* __restrict__ mult) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (std::uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&mult[rep[i]], 1u);
}
__global__ void cs_compact(const std::uint32_t* __restrict__ mult, std::uint64_t n,
                           std::uint32_t* __restrict__ dl, std::uint32_t* __restrict__ dm,
                           std::uint32_t* __restrict__ cnt) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (std::uint64_t)gridDim.x * blockDim.x)
    if (mult[i]) {
      const std::uint32_t k = atomicAdd(cnt, 1u);
      dl[k] = (std::uint32_t)i;
      dm[k] = mult[i];
    }
}
__device__ __forceinline__ void cs_range(float f, int& lo, int& hi, bool& bad) {
  const std::uint32_t u = __float_as_uint(f);
  const int E = (int)((u >> 23) & 0xffu);
  if (E == 255) bad = true;
  else if (E != 0) { lo = min(lo, E - 150); hi = max(hi, E - 126); }
  else if (u & 0x7fffffu) { lo = min(lo, -149); hi = max(hi, -126); }
}
__global__ void __launch_bounds__(256)
    cs_sum(const float4* __restrict__ x, std::uint64_t ldv, std::uint64_t nv, std::uint64_t dim,
           std::uint64_t n, int lgn, const std::uint32_t* __restrict__ dl,
           const std::uint32_t* __restrict__ dm, const std::uint32_t* __restrict__ cnt,
           double* __restrict__ out, std::uint32_t* __restrict__ flagged,
           std::uint32_t* __restrict__ fcnt) {
  const std::uint64_t cv = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (cv >= nv) return;
  const std::uint32_t L = *cnt;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int lo = 1 << 20, hi = -(1 << 20);
  bool bad = false;
#pragma unroll 8
  for (std::uint32_t k = 0; k < L; ++k) {
    const float4 v = __ldg(x + (std::uint64_t)dl[k] * ldv + cv);
    const double m = (double)dm[k];
    cs_range(v.x, lo, hi, bad);
    cs_range(v.y, lo, hi, bad);
    cs_range(v.z, lo, hi, bad);
    cs_range(v.w, lo, hi, bad);
    a0 = __dadd_rn(a0, __dmul_rn(m, (double)v.x));
    a1 = __dadd_rn(a1, __dmul_rn(m, (double)v.y));
    a2 = __dadd_rn(a2, __dmul_rn(m, (double)v.z));
    a3 = __dadd_rn(a3, __dmul_rn(m, (double)v.w));
  }
  if (bad || hi + lgn - lo > 53) {
    flagged[atomicAdd(fcnt, 1u)] = (std::uint32_t)cv;
    return;
  }
  const double a[4] = {a0, a1, a2, a3};
#pragma unroll
  for (int w = 0; w < 4; ++w)
    if (cv * 4 + w < dim) out[cv * 4 + w] = __ddiv_rn(a[w], (double)n);
}
// the listed column vectors: the reference tree over the rows (colmean_kernel's)
__global__ void cs_fix(const float* __restrict__ x, std::uint64_t n, std::uint64_t ld,
                       std::uint64_t dim, const std::uint32_t* __restrict__ rep,
                       const std::uint32_t* __restrict__ flagged,
                       const std::uint32_t* __restrict__ fcnt, double* __restrict__ out) {
  const std::uint64_t items = (std::uint64_t)*fcnt * 4;
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < items;
       i += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t j = (std::uint64_t)flagged[i / 4] * 4 + i % 4;
    if (j >= dim) continue;
    auto ld_fn = [&](std::uint32_t r) -> double { return (double)x[(std::uint64_t)rep[r] * ld + j]; };
    const double t = pairwise_rt<double>(ld_fn, (std::uint32_t)n,
                                         [](double a, double b) { return __dadd_rn(a, b); }, 0.0);
    out[j] = __ddiv_rn(t, (double)n);
  }
}

// n = 8 * 2^K >= 256: a warp per listed column -- lane l evaluates the
// aligned subtree over rows [l n/32, (l+1) n/32) (the reference tree splits
// at n/2 down to 8-row blocks, so these are its subtrees), then five xor
// shuffle levels join them pairwise: the tree's own adds, 32 lanes deep.
__global__ void cs_fix_warp(const float* __restrict__ x, std::uint64_t n, std::uint64_t ld,
                            std::uint64_t dim, const std::uint32_t* __restrict__ rep,
                            const std::uint32_t* __restrict__ flagged,
                            const std::uint32_t* __restrict__ fcnt, double* __restrict__ out) {
  const std::uint64_t items = (std::uint64_t)*fcnt * 4;
  const std::uint32_t lane = threadIdx.x & 31u, c = (std::uint32_t)(n / 32);
  const std::uint64_t warps = (std::uint64_t)gridDim.x * (blockDim.x / 32);
  for (std::uint64_t i = (blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x) / 32; i < items;
       i += warps) {
    const std::uint64_t j = (std::uint64_t)flagged[i / 4] * 4 + i % 4;
    if (j >= dim) continue;  // warp-uniform
    const std::uint32_t base = lane * c;
    auto ld_fn = [&](std::uint32_t r) -> double {
      return (double)x[(std::uint64_t)rep[base + r] * ld + j];
    };
    double v = pairwise_rt<double>(ld_fn, c, [](double a, double b) { return __dadd_rn(a, b); },
                                   0.0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) out[j] = __ddiv_rn(v, (double)n);
  }
}

}  // namespace

std::size_t colsum_scratch_bytes(std::uint64_t n, std::uint64_t dim) {
  return (3 * n + 4 + (dim + 3) / 4) * 4 + 64;
}

bool launch_colmean_exactsum(const float* x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                             const std::uint32_t* rep, double* out, void* scratch,
                             cudaStream_t s) {
  static const bool on = [] {
    const char* e = std::getenv("MOSHPIT_COLSUM_EXACT");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || !rep || !scratch || n == 0 || dim == 0 || ld % 4 != 0 ||
      reinterpret_cast<std::uintptr_t>(x) % 16 != 0 || n > (1u << 24))
    return false;
  int lgn = 0;
  while ((1ull << lgn) < n) ++lgn;
  auto* u = static_cast<std::uint32_t*>(scratch);
  std::uint32_t *mult = u, *dl = u + n, *dm = u + 2 * n, *cnt = u + 3 * n, *fcnt = cnt + 1,
                *flagged = cnt + 4;
  MB_CUDA(cudaMemsetAsync(mult, 0, n * 4, s));
  MB_CUDA(cudaMemsetAsync(cnt, 0, 16, s));
  const unsigned gb = (unsigned)std::min<std::uint64_t>((n + 255) / 256, 1184);
  cs_mult<<<gb, 256, 0, s>>>(rep, n, mult);
  cs_compact<<<gb, 256, 0, s>>>(mult, n, dl, dm, cnt);
  const std::uint64_t nv = (dim + 3) / 4;
  cs_sum<<<(unsigned)((nv + 255) / 256), 256, 0, s>>>(reinterpret_cast<const float4*>(x), ld / 4,
                                                     nv, dim, n, lgn, dl, dm, cnt, out, flagged,
                                                     fcnt);
  if (n >= 256 && n % 8 == 0 && (((n / 8) & (n / 8 - 1)) == 0))
    cs_fix_warp<<<1184, 128, 0, s>>>(x, n, ld, dim, rep, flagged, fcnt, out);
  else
    cs_fix<<<1184, 128, 0, s>>>(x, n, ld, dim, rep, flagged, fcnt, out);
  MB_LAUNCH_CHECK();
  return true;
}

template <typename T>
void launch_distortion(const T* x, std::uint64_t n, std::uint64_t ld,
                       std::uint64_t dim, const double* ref, double* sq,
                       double* partial, double* out, int exact, cudaStream_t s,
                       const RepRows* reps) {
  if (n == 0) {
    finish_distortion<<<1, kFinThreads, 0, s>>>(sq, 0, out);
    MB_LAUNCH_CHECK();
    return;
  }
  const std::uint32_t* list = reps ? reps->list : nullptr;
  const std::uint32_t* count = reps ? reps->count : nullptr;
  const std::uint32_t* rep = reps ? reps->rep : nullptr;
  if (exact || dim == 0) {
    launch_dist_exact<T>(x, n, ld, dim, ref, sq, 0, s, list, count);
    if (rep) {
      expand_reps<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sq, rep, n);
      MB_LAUNCH_CHECK();
    }
  } else {
    const std::uint64_t nch = (dim + kChunk - 1) / kChunk;
    const unsigned gy = fast_rows_grid(n, nch, list != nullptr);
    dist_rows_fast_off<T><<<dim3((unsigned)nch, gy), kRedThreads, 0, s>>>(
        x, ld, dim, ref, nch, 0, partial, n, list, count);
    MB_LAUNCH_CHECK();
    fold_rows<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(partial, n, nch, sq, rep);
  }
  MB_LAUNCH_CHECK();
  finish_distortion<<<1, kFinThreads, 0, s>>>(sq, n, out);
  MB_LAUNCH_CHECK();
}

// FAST distortion after a round from the representative rows listed in
// `reps` -- every row when the caller's partial cache is cold, only the
// averaged groups' representatives when every other row is known to be
// unchanged since the previous call (its partials are still in its slot) --
// then the representatives' partials scattered into their members' slots.
// The per-row partials and their fold are the uncached path's: bit-identical.
template <typename T>
void launch_distortion_fast_cached(const T* x, std::uint64_t n, std::uint64_t ld,
                                   std::uint64_t dim, const double* ref, double* sq,
                                   double* partial, double* out, cudaStream_t s,
                                   const RepRows& reps) {
  if (n == 0 || dim == 0) {
    launch_distortion<T>(x, n, ld, dim, ref, sq, partial, out, 0, s, &reps);
    return;
  }
  const std::uint64_t nch = (dim + kChunk - 1) / kChunk;
  const unsigned gy = fast_rows_grid(n, nch, true);
  dist_rows_fast_off<T><<<dim3((unsigned)nch, gy), kRedThreads, 0, s>>>(
      x, ld, dim, ref, nch, 0, partial, n, reps.list, reps.count);
  MB_LAUNCH_CHECK();
  fold_rows<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(partial, n, nch, sq, reps.rep);
  MB_LAUNCH_CHECK();
  scatter_rep_partials<<<grid_for(n * nch, 256), 256, 0, s>>>(partial, reps.rep, n, nch);
  MB_LAUNCH_CHECK();
  finish_distortion<<<1, kFinThreads, 0, s>>>(sq, n, out);
  MB_LAUNCH_CHECK();
}
template void launch_distortion_fast_cached<float>(const float*, std::uint64_t, std::uint64_t,
                                                   std::uint64_t, const double*, double*,
                                                   double*, double*, cudaStream_t,
                                                   const RepRows&);
template void launch_distortion_fast_cached<double>(const double*, std::uint64_t, std::uint64_t,
                                                    std::uint64_t, const double*, double*,
                                                    double*, double*, cudaStream_t,
                                                    const RepRows&);

void launch_drift(const double* mean, const double* ref, std::uint64_t dim,
                  double* partial, double* out, int exact, cudaStream_t s) {
  if (exact || dim == 0) {
    launch_drift_exact(mean, ref, dim, partial, 0, s);  // partial[0..1] = the two j-sums
    drift_finish_acc<<<1, 1, 0, s>>>(partial, out);
  } else {
    const std::uint64_t nch = (dim + kChunk - 1) / kChunk;
    drift_fast_partial<<<(unsigned)nch, kRedThreads, 0, s>>>(mean, ref, dim, partial);
    MB_LAUNCH_CHECK();
    drift_fast_finish<<<1, kDriftFinThreads, 0, s>>>(partial, nch, out);
  }
  MB_LAUNCH_CHECK();
}

template <typename T>
void launch_fill_synthetic(T* x, std::uint64_t n, std::uint64_t dim,
                           std::uint64_t ld, std::uint64_t seed,
                           std::uint64_t col0, cudaStream_t s) {
  if (n == 0 || dim == 0) return;
  fill_synthetic_kernel<T><<<grid_for(n * dim, 256), 256, 0, s>>>(x, n, dim, ld, seed, col0);
  MB_LAUNCH_CHECK();
}

template <typename T>
void launch_broadcast_rows(T* dst, std::uint64_t ld, const T* row,
                           std::uint64_t n, std::uint64_t dim, cudaStream_t s) {
  if (n == 0 || dim == 0) return;
  broadcast_rows_kernel<T><<<grid_for(n * dim, 256), 256, 0, s>>>(dst, ld, row, n, dim);
  MB_LAUNCH_CHECK();
}

#define MB_INST(T)                                                                      \
  template void launch_colmean<T, double>(const T*, std::uint64_t, std::uint64_t,       \
                                          std::uint64_t, const std::uint32_t*, double*, \
                                          cudaStream_t, bool);                          \
  template void launch_distortion<T>(const T*, std::uint64_t, std::uint64_t,            \
                                     std::uint64_t, const double*, double*, double*,    \
                                     double*, int, cudaStream_t, const RepRows*);       \
  template void launch_fill_synthetic<T>(T*, std::uint64_t, std::uint64_t,              \
                                         std::uint64_t, std::uint64_t, std::uint64_t,   \
                                         cudaStream_t);                                 \
  template void launch_broadcast_rows<T>(T*, std::uint64_t, const T*, std::uint64_t,    \
                                         std::uint64_t, cudaStream_t);
MB_INST(float)
MB_INST(double)
template void launch_colmean<float, float>(const float*, std::uint64_t, std::uint64_t,
                                          std::uint64_t, const std::uint32_t*, float*,
                                          cudaStream_t, bool);
#undef MB_INST

}  // namespace mb200
