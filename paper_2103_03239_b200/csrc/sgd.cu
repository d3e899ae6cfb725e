// sgd.cu -- Moshpit SGD on the Quadratic objective (SURVEY 8a rows a17/a18,
// 8f rank 1): optimizer::local_step (optimizer.hpp:231-242) and
// optimizer::run_moshpit_sgd (optimizer.hpp:297-439) on the GPU.
//
// Per step: membership events (leavers truncate, joiners copy a donor row:
// device memcpy), the local step theta <- theta - gamma*(c*(theta - t) + noise)
// as one elementwise kernel (no FMA: the reference rounds the product and the
// difference separately), the averaging pass (kernels 1 + 2 on the shared
// "averaging" stream, cells redrawn each sync exactly as
// optimizer.hpp:254-268), and the diagnostics as fp64 device reductions
// (EXACT: the reference's sequential order; FAST: fixed-order blocks).
// Noise: the reference's own sequential polar stream drawn on the host
// (bit-exact; O(N*D) host draws per step) or a counter-based Philox4x32-10
// normal on the device (statistical parity; the performance path).
#include <cmath>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <memory>

#include "philox.cuh"
#include "plane.cuh"

namespace mb200 {
namespace {

template <typename T>
struct SOps;
template <>
struct SOps<float> {
  __device__ static float sub(float a, float b) { return __fsub_rn(a, b); }
  __device__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ static float add(float a, float b) { return __fadd_rn(a, b); }
};
template <>
struct SOps<double> {
  __device__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ static double add(double a, double b) { return __dadd_rn(a, b); }
};

constexpr int kStepThreads = 256;

// theta <- theta - gamma * (c * (theta - t) + nj)   (optimizer.hpp:356-373)
template <typename T>
__global__ void __launch_bounds__(kStepThreads)
    sgd_step_kernel(T* __restrict__ x, std::uint64_t n, std::uint64_t dim, std::uint64_t ld,
                    const T* __restrict__ curv, const T* __restrict__ tgt, T gamma,
                    const T* __restrict__ noise, double coord_std, int philox_mode,
                    std::uint64_t seed, std::uint64_t step, std::uint32_t* nonfinite,
                    double* noise_partial) {
  using O = SOps<T>;
  __shared__ double red[kStepThreads];
  double nsq = 0.0;
  const std::uint64_t quads = (dim + 3) / 4;
  const std::uint64_t total = n * quads;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t i = e / quads, q = e % quads;
    float z[4] = {0, 0, 0, 0};
    if (philox_mode) philox_normals4(seed, step, i, q, z);
    T nq = T(0);  // per-quad n_j^2 partial (the fused kernel's terms)
    for (int u = 0; u < 4; ++u) {
      const std::uint64_t j = q * 4 + u;
      if (j >= dim) break;
      T* p = x + i * ld + j;
      T g = O::mul(curv[j], O::sub(*p, tgt[j]));
      if (noise) {
        g = O::add(g, noise[i * dim + j]);
      } else if (philox_mode) {
        const T nj = noise_component(z[u], coord_std, (T*)nullptr);
        nsq_add(nq, nj);
        g = O::add(g, nj);
      }
      if (!isfinite(g)) atomicOr(nonfinite, 1u);
      *p = O::sub(*p, O::mul(gamma, g));
    }
    nsq += (double)nq;
  }
  if (philox_mode) {
    red[threadIdx.x] = nsq;
    __syncthreads();
    for (int s = kStepThreads / 2; s > 0; s >>= 1) {
      if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) noise_partial[blockIdx.x] = red[0];
  }
}

// The same step on 16-byte vectors (4 fp32 / 2 fp64 coordinates of one row)
// for 16-byte-aligned rows: one thread per vector, grid-stride, curvature and
// target read as vectors, the quad's Philox normals once per vector (fp64:
// the vector's half of the quad).  Identical per-coordinate arithmetic; the
// n_j^2 partials are per vector (fp32: per quad, as above).
template <typename T>
struct SVec;
template <>
struct SVec<float> {
  using V = float4;
  static constexpr int W = 4;
};
template <>
struct SVec<double> {
  using V = double2;
  static constexpr int W = 2;
};

template <typename T>
__global__ void __launch_bounds__(kStepThreads)
    sgd_step_vec(T* __restrict__ x, std::uint64_t n, std::uint64_t dim, std::uint64_t ld,
                 const T* __restrict__ curv, const T* __restrict__ tgt, T gamma,
                 const T* __restrict__ noise, double coord_std, int philox_mode,
                 const __grid_constant__ PhiloxKeys pk, std::uint64_t step,
                 std::uint32_t* nonfinite, double* noise_partial) {
  using O = SOps<T>;
  using V = typename SVec<T>::V;
  constexpr int W = SVec<T>::W;
  __shared__ double red[kStepThreads / 32];
  double nsq = 0.0;
  T chk = T(0);
  const std::uint64_t nv = (dim + W - 1) / W, ldv = ld / W;
  const std::uint64_t total = n * nv;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t i = e / nv, cv = e % nv, j0 = cv * W;
    V* p = reinterpret_cast<V*>(x) + i * ldv + cv;
    V v = *p, c, t;
    T* pv = reinterpret_cast<T*>(&v);
    T* pc = reinterpret_cast<T*>(&c);
    T* pt = reinterpret_cast<T*>(&t);
    if (j0 + W <= dim) {
      c = __ldg(reinterpret_cast<const V*>(curv) + cv);
      t = __ldg(reinterpret_cast<const V*>(tgt) + cv);
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        pc[w] = j0 + w < dim ? curv[j0 + w] : T(0);
        pt[w] = j0 + w < dim ? tgt[j0 + w] : T(0);
      }
    }
    float z[4] = {0, 0, 0, 0};
    const int zo = W == 4 ? 0 : (int)(cv & 1) * 2;
    if (philox_mode && !noise) philox_normals4(pk, step, i, W == 4 ? cv : cv >> 1, z);
    T nq = T(0);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const std::uint64_t j = j0 + w;
      if (j >= dim) break;
      T g = O::mul(pc[w], O::sub(pv[w], pt[w]));
      if (noise) {
        g = O::add(g, noise[i * dim + j]);
      } else if (philox_mode) {
        const T nj = noise_component(z[zo + w], coord_std, (T*)nullptr);
        nsq_add(nq, nj);
        g = O::add(g, nj);
      }
      chk = O::add(chk, O::mul(g, T(0)));
      pv[w] = O::sub(pv[w], O::mul(gamma, g));
    }
    *p = v;
    nsq += (double)nq;
  }
  if (chk != T(0)) atomicOr(nonfinite, 1u);
  if (philox_mode && !noise) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nsq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int k = 0; k < kStepThreads / 32; ++k) t += red[k];
      noise_partial[blockIdx.x] = t;
    }
  }
}

// Sequential D-vector diagnostics (EXACT, one thread, optimizer.hpp:386-418):
// out[0] pv inner product, [1] f(mean), [2] |grad f(mean)|^2, [3] f(weighted);
// wsum[j] += w_k * mean[j] in place.
__global__ void sgd_vec_exact(const double* __restrict__ mean, const double* __restrict__ hat,
                              const double* __restrict__ c, const double* __restrict__ t,
                              double* __restrict__ wsum, double w_k, double weight_total,
                              std::uint64_t dim, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double ip = 0.0, f = 0.0, gn = 0.0, fw = 0.0;
  for (std::uint64_t j = 0; j < dim; ++j) {
    const double mj = mean[j];
    ip = __dadd_rn(ip, __dmul_rn(__dsub_rn(mj, hat[j]), __dadd_rn(mj, hat[j])));
    const double dd = __dsub_rn(mj, t[j]);
    f = __dadd_rn(f, __dmul_rn(__dmul_rn(__dmul_rn(0.5, c[j]), dd), dd));
    const double g = __dmul_rn(c[j], dd);
    gn = __dadd_rn(gn, __dmul_rn(g, g));
    const double ws = __dadd_rn(wsum[j], __dmul_rn(w_k, mj));
    wsum[j] = ws;
    const double wd = __dsub_rn(__ddiv_rn(ws, weight_total), t[j]);
    fw = __dadd_rn(fw, __dmul_rn(__dmul_rn(__dmul_rn(0.5, c[j]), wd), wd));
  }
  out[0] = ip;
  out[1] = f;
  out[2] = gn;
  out[3] = fw;
}

constexpr int kRed = 256;
// FAST chunk: 4096 coordinates per CTA (256 CTAs at D = 2^20; 16 at 2^16
// left the per-step vector sums latency-bound)
constexpr std::uint64_t kChunk = 1 << 12;

__device__ double blk_sum(double v, double* buf) {
  buf[threadIdx.x] = v;
  __syncthreads();
  for (int s = kRed / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) buf[threadIdx.x] = __dadd_rn(buf[threadIdx.x], buf[threadIdx.x + s]);
    __syncthreads();
  }
  const double r = buf[0];
  __syncthreads();
  return r;
}

// FAST variant: fixed-order chunk partials, folded by sgd_vec_fold.
__global__ void sgd_vec_fast(const double* __restrict__ mean, const double* __restrict__ hat,
                             const double* __restrict__ c, const double* __restrict__ t,
                             double* __restrict__ wsum, double w_k, double weight_total,
                             std::uint64_t dim, double* __restrict__ partial) {
  __shared__ double buf[kRed];
  const std::uint64_t lo = blockIdx.x * kChunk, hi = lo + kChunk < dim ? lo + kChunk : dim;
  double a[4] = {0, 0, 0, 0};
  for (std::uint64_t j = lo + threadIdx.x; j < hi; j += kRed) {
    const double mj = mean[j];
    a[0] = __dadd_rn(a[0], __dmul_rn(__dsub_rn(mj, hat[j]), __dadd_rn(mj, hat[j])));
    const double dd = __dsub_rn(mj, t[j]);
    a[1] = __dadd_rn(a[1], __dmul_rn(__dmul_rn(__dmul_rn(0.5, c[j]), dd), dd));
    const double g = __dmul_rn(c[j], dd);
    a[2] = __dadd_rn(a[2], __dmul_rn(g, g));
    const double ws = __dadd_rn(wsum[j], __dmul_rn(w_k, mj));
    wsum[j] = ws;
    const double wd = __dsub_rn(__ddiv_rn(ws, weight_total), t[j]);
    a[3] = __dadd_rn(a[3], __dmul_rn(__dmul_rn(__dmul_rn(0.5, c[j]), wd), wd));
  }
  for (int q = 0; q < 4; ++q) {
    const double s = blk_sum(a[q], buf);
    if (threadIdx.x == 0) partial[blockIdx.x * 4 + q] = s;
  }
}

__global__ void sgd_vec_fold(const double* __restrict__ partial, std::uint64_t nch,
                             double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s[4] = {0, 0, 0, 0};
  for (std::uint64_t c = 0; c < nch; ++c)
    for (int q = 0; q < 4; ++q) s[q] = __dadd_rn(s[q], partial[c * 4 + q]);
  for (int q = 0; q < 4; ++q) out[q] = s[q];
}

// V_k = sum_i sum_j (theta_ij - mean_j)^2 / n, EXACT: one running sum over
// (i, j) in row-major order (optimizer.hpp:394-401).
template <typename T>
__global__ void dispersion_exact(const T* __restrict__ x, std::uint64_t n, std::uint64_t ld,
                                 std::uint64_t dim, const double* __restrict__ mean,
                                 double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double v = 0.0;
  for (std::uint64_t i = 0; i < n; ++i)
    for (std::uint64_t j = 0; j < dim; ++j) {
      const double dd = __dsub_rn((double)x[i * ld + j], mean[j]);
      v = __dadd_rn(v, __dmul_rn(dd, dd));
    }
  *out = __ddiv_rn(v, (double)n);
}

// FAST: block (chunk, row) partials, then per-row sums in chunk order
// (row_sums) and one fold over the rows in row order.
template <typename T>
__global__ void dispersion_fast(const T* __restrict__ x, std::uint64_t ld, std::uint64_t dim,
                                const double* __restrict__ mean, std::uint64_t nch,
                                double* __restrict__ partial) {
  __shared__ double buf[kRed];
  const std::uint64_t c = blockIdx.x, i = blockIdx.y;
  const std::uint64_t lo = c * kChunk, hi = lo + kChunk < dim ? lo + kChunk : dim;
  double a = 0.0;
  for (std::uint64_t j = lo + threadIdx.x; j < hi; j += kRed) {
    const double dd = __dsub_rn((double)x[i * ld + j], mean[j]);
    a = __dadd_rn(a, __dmul_rn(dd, dd));
  }
  const double s = blk_sum(a, buf);
  if (threadIdx.x == 0) partial[i * nch + c] = s;
}

// The same partials for the representative rows only (list / count on the
// device; after an averaging pass every member of a non-voided group holds
// the identical row), grid-y looping over the list.
template <typename T>
__global__ void dispersion_fast_list(const T* __restrict__ x, std::uint64_t ld,
                                     std::uint64_t dim, const double* __restrict__ mean,
                                     std::uint64_t nch, double* __restrict__ partial,
                                     const std::uint32_t* __restrict__ list,
                                     const std::uint32_t* __restrict__ count) {
  __shared__ double buf[kRed];
  const std::uint64_t c = blockIdx.x;
  const std::uint64_t lo = c * kChunk, hi = lo + kChunk < dim ? lo + kChunk : dim;
  for (std::uint64_t y = blockIdx.y; y < *count; y += gridDim.y) {
    const std::uint64_t i = list[y];
    double a = 0.0;
    for (std::uint64_t j = lo + threadIdx.x; j < hi; j += kRed) {
      const double dd = __dsub_rn((double)x[i * ld + j], mean[j]);
      a = __dadd_rn(a, __dmul_rn(dd, dd));
    }
    const double s = blk_sum(a, buf);
    if (threadIdx.x == 0) partial[i * nch + c] = s;
  }
}

// V_k's FAST fold, part 1: each row's chunk partials in chunk order (row i's
// read from rep[i] when given: identical rows share their partials), one
// thread per row; part 2 is fold_all over the row sums in row order.
__global__ void row_sums(const double* __restrict__ partial, std::uint64_t n, std::uint64_t nch,
                         const std::uint32_t* __restrict__ rep, double* __restrict__ out) {
  const std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* p = partial + (std::uint64_t)(rep ? rep[i] : i) * nch;
  double s = 0.0;
  for (std::uint64_t c = 0; c < nch; ++c) s = __dadd_rn(s, p[c]);
  out[i] = s;
}

__global__ void fold_all(const double* __restrict__ partial, std::uint64_t count, double div,
                         double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (std::uint64_t k = 0; k < count; ++k) s = __dadd_rn(s, partial[k]);
  *out = __ddiv_rn(s, div);
}

template <typename T>
__global__ void cast_kernel(const double* __restrict__ in, T* __restrict__ out,
                            std::uint64_t n) {
  const std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (T)in[i];
}

template <typename T>
__global__ void broadcast_theta0(T* __restrict__ x, std::uint64_t n, std::uint64_t ld,
                                 std::uint64_t dim, const double* __restrict__ th0) {
  const std::uint64_t total = n * dim;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (std::uint64_t)gridDim.x * blockDim.x)
    x[(e / dim) * ld + e % dim] = (T)th0[e % dim];
}

unsigned grid_for(std::uint64_t work, unsigned threads) {
  std::uint64_t b = (work + threads - 1) / threads;
  if (b > 148ull * 16) b = 148ull * 16;
  return (unsigned)(b ? b : 1);
}

// ---- LogisticRegression (optimizer.hpp:75-146) ------------------------------
// coeff[i][s] = -y_s / (1 + exp(y_s * margin)), margin = sum_j x_sj * theta_ij
// in j order (optimizer.hpp:124-128); ymargin[i][s] = value()'s softplus term.
// CUDA's exp/log1p need not round like glibc's in the last bit, so logistic
// parity is a tolerance; the summation orders are the reference's.
template <typename T>
__global__ void logit_coeff(const T* __restrict__ x, std::uint64_t ld, std::uint64_t dim,
                            const double* __restrict__ xs, const double* __restrict__ ys,
                            std::uint64_t S, double* __restrict__ coeff,
                            double* __restrict__ ymargin) {
  const std::uint64_t sidx = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  const std::uint64_t i = blockIdx.y;
  if (sidx >= S) return;
  const T* th = x + i * ld;
  const double* xr = xs + sidx * dim;
  double margin = 0.0;
  for (std::uint64_t j = 0; j < dim; ++j) margin = __dadd_rn(margin, __dmul_rn(xr[j], (double)th[j]));
  const double y = ys[sidx];
  if (coeff) coeff[i * S + sidx] = __ddiv_rn(-y, __dadd_rn(1.0, exp(__dmul_rn(y, margin))));
  if (ymargin) {  // the value() term log(1 + exp(-m)), m = margin * y, both tails
    const double m = __dmul_rn(margin, y);
    ymargin[i * S + sidx] = m > 0.0 ? log1p(exp(-m)) : __dadd_rn(-m, log1p(exp(m)));
  }
}

// g_ij = (sum_s coeff_is * x_sj) / m + l2 * theta_ij  (optimizer.hpp:129-135), then
// optionally the SGD update theta -= gamma (g + n_j) (optimizer.hpp:356-373).
template <typename T>
__global__ void logit_grad(T* __restrict__ x, std::uint64_t ld, std::uint64_t dim,
                           const double* __restrict__ xs, std::uint64_t S,
                           const double* __restrict__ coeff, double l2, int update, T gamma,
                           const T* __restrict__ noise, double coord_std, int philox_mode,
                           std::uint64_t seed, std::uint64_t step, std::uint32_t* nonfinite,
                           double* nsq_out, double* __restrict__ g_out, std::uint64_t i0) {
  const std::uint64_t j = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  const std::uint64_t i = blockIdx.y;
  if (j >= dim) return;
  const double* c = coeff + i * S;
  double g = 0.0;
  for (std::uint64_t sidx = 0; sidx < S; ++sidx) g = __dadd_rn(g, __dmul_rn(c[sidx], xs[sidx * dim + j]));
  T* p = x + i * ld + j;
  g = __dadd_rn(__ddiv_rn(g, (double)S), __dmul_rn(l2, (double)*p));
  if (!update) {
    g_out[j] = g;
    return;
  }
  using O = SOps<T>;
  T gt = (T)g;
  if (noise) {
    gt = O::add(gt, noise[i * dim + j]);
  } else if (philox_mode) {
    float z[4];
    philox_normals4(seed, step, i0 + i, j / 4, z);
    const T nj = noise_component(z[j % 4], coord_std, (T*)nullptr);
    atomicAdd(nsq_out, (double)nj * (double)nj);
    gt = O::add(gt, nj);
  }
  if (!isfinite(gt)) atomicOr(nonfinite, 1u);
  *p = O::sub(*p, O::mul(gamma, gt));
}

// Tiled forms of the two kernels above for the per-peer step: both are
// GEMM-shaped (margins = Theta . X^T, gradient = C . X) but every output must
// be summed sequentially in k from 0.0 with separately rounded products (the
// reference's order), so they run on the fp64 SIMT pipes (DMUL + DADD, no
// tensor cores, no FMA): 64x64 output tiles per 256-thread CTA, 4x4 outputs
// per thread, k staged through double-buffered shared memory 16 at a time
// (the next tile's global loads in flight while the current one is used).
// Each output's k-loop is still the plain sequential chain.
constexpr int kLT = 64, kLK = 16;

template <typename T>
__global__ void __launch_bounds__(256)
    logit_coeff_tiled(const T* __restrict__ x, std::uint64_t n, std::uint64_t ld,
                      std::uint64_t dim, const double* __restrict__ xs,
                      const double* __restrict__ ys, std::uint64_t S,
                      double* __restrict__ coeff) {
  // double-buffered k-tiles; the next tile's global loads are in flight
  // (registers) while the current one is multiplied
  __shared__ double As[2][kLK][kLT + 1];  // theta[i][k] -> As[.][k][i - i0]
  __shared__ double Bs[2][kLK][kLT + 1];  // xs[s][k]    -> Bs[.][k][s - s0]
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const std::uint64_t i0 = (std::uint64_t)blockIdx.y * kLT, s0 = (std::uint64_t)blockIdx.x * kLT;
  constexpr int kPer = kLT * kLK / 256;  // elements of each tile loaded per thread
  double ra[kPer], rb[kPer];
  auto fetch = [&](std::uint64_t k0) {
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int e = threadIdx.x + 256 * q;
      const int r = e / kLK, kk = e % kLK;
      const std::uint64_t k = k0 + kk, i = i0 + r, sm = s0 + r;
      ra[q] = (i < n && k < dim) ? (double)x[i * ld + k] : 0.0;
      rb[q] = (sm < S && k < dim) ? xs[sm * dim + k] : 0.0;
    }
  };
  auto stash = [&](int b) {
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int e = threadIdx.x + 256 * q;
      const int r = e / kLK, kk = e % kLK;
      As[b][kk][r] = ra[q];
      Bs[b][kk][r] = rb[q];
    }
  };
  double acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
  fetch(0);
  stash(0);
  __syncthreads();
  int cur = 0;
  for (std::uint64_t k0 = 0; k0 < dim; k0 += kLK) {
    const bool more = k0 + kLK < dim;
    if (more) fetch(k0 + kLK);
    const int kn = dim - k0 < (std::uint64_t)kLK ? (int)(dim - k0) : kLK;
    if (kn == kLK) {
#pragma unroll
      for (int kk = 0; kk < kLK; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = As[cur][kk][ty + 16 * r];
#pragma unroll
        for (int c = 0; c < 4; ++c) b[c] = Bs[cur][kk][tx + 16 * c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = __dadd_rn(acc[r][c], __dmul_rn(b[c], a[r]));
      }
    } else {
      for (int kk = 0; kk < kn; ++kk) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            acc[r][c] = __dadd_rn(acc[r][c],
                                  __dmul_rn(Bs[cur][kk][tx + 16 * c], As[cur][kk][ty + 16 * r]));
      }
    }
    if (more) stash(cur ^ 1);
    __syncthreads();
    cur ^= 1;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const std::uint64_t i = i0 + ty + 16 * r;
    if (i >= n) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const std::uint64_t sm = s0 + tx + 16 * c;
      if (sm >= S) continue;
      const double y = ys[sm];
      coeff[i * S + sm] = __ddiv_rn(-y, __dadd_rn(1.0, exp(__dmul_rn(y, acc[r][c]))));
    }
  }
}

// Gradient tiles are TM x TN (4 x 4 outputs per thread, TM*TN/16 threads).
// 64 x 64 is used: at N = dim = 1024 its 256 tiles leave 108 SMs with two
// and 40 with one (fp64 pipe 57 % vs 73 % for the 1024-tile margins), but
// 32 x 32 tiles (1024, balanced) measured slower still (0.88 vs 0.83 ms):
// half the operand reuse per shared-memory load.
template <typename T, int TM, int TN>
__global__ void __launch_bounds__(TM * TN / 16)
    logit_grad_tiled(T* __restrict__ x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                     const double* __restrict__ xs, std::uint64_t S,
                     const double* __restrict__ coeff, double l2, T gamma,
                     const T* __restrict__ noise, double coord_std, int philox_mode,
                     std::uint64_t seed, std::uint64_t step, std::uint32_t* nonfinite,
                     double* nsq_out) {
  constexpr int NT = TM * TN / 16, CW = TN / 4, RS = TM / 4;
  __shared__ double As[2][kLK][TM + 1];            // coeff[i][s] -> As[.][s - k0][i - i0]
  __shared__ __align__(16) double Bs[2][kLK][TN];  // xs[s][j]    -> Bs[.][s - k0][j - j0]
  const int tx = threadIdx.x % CW, ty = threadIdx.x / CW;
  const std::uint64_t i0 = (std::uint64_t)blockIdx.y * TM, j0 = (std::uint64_t)blockIdx.x * TN;
  constexpr int kPa = TM * kLK / NT, kPb = TN * kLK / NT;
  double ra[kPa], rb[kPb];
  auto fetch = [&](std::uint64_t k0) {
#pragma unroll
    for (int q = 0; q < kPa; ++q) {
      const int e = threadIdx.x + NT * q;
      const int r = e / kLK, kk = e % kLK;
      const std::uint64_t i = i0 + r, k = k0 + kk;
      ra[q] = (i < n && k < S) ? coeff[i * S + k] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kPb; ++q) {
      const int e = threadIdx.x + NT * q;
      const int kk = e / TN, cc = e % TN;
      const std::uint64_t k = k0 + kk, j = j0 + cc;
      rb[q] = (k < S && j < dim) ? xs[k * dim + j] : 0.0;
    }
  };
  auto stash = [&](int b) {
#pragma unroll
    for (int q = 0; q < kPa; ++q) {
      const int e = threadIdx.x + NT * q;
      As[b][e % kLK][e / kLK] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < kPb; ++q) {
      const int e = threadIdx.x + NT * q;
      Bs[b][e / TN][e % TN] = rb[q];
    }
  };
  double acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
  fetch(0);
  stash(0);
  __syncthreads();
  int cur = 0;
  for (std::uint64_t k0 = 0; k0 < S; k0 += kLK) {
    const bool more = k0 + kLK < S;
    if (more) fetch(k0 + kLK);
    const int kn = S - k0 < (std::uint64_t)kLK ? (int)(S - k0) : kLK;
    if (kn == kLK) {
#pragma unroll
      for (int kk = 0; kk < kLK; ++kk) {
        double a[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = As[cur][kk][ty + RS * r];
        const double2 b01 = *reinterpret_cast<const double2*>(&Bs[cur][kk][tx * 4]);
        const double2 b23 = *reinterpret_cast<const double2*>(&Bs[cur][kk][tx * 4 + 2]);
        const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = __dadd_rn(acc[r][c], __dmul_rn(a[r], b[c]));
      }
    } else {
      for (int kk = 0; kk < kn; ++kk) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            acc[r][c] = __dadd_rn(acc[r][c],
                                  __dmul_rn(As[cur][kk][ty + RS * r], Bs[cur][kk][tx * 4 + c]));
      }
    }
    if (more) stash(cur ^ 1);
    __syncthreads();
    cur ^= 1;
  }
  using O = SOps<T>;
  double nsq = 0.0;
  bool bad = false;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const std::uint64_t i = i0 + ty + RS * r;
    if (i >= n) continue;
    float z[4] = {0.f, 0.f, 0.f, 0.f};
    if (philox_mode) philox_normals4(seed, step, i, (j0 >> 2) + tx, z);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const std::uint64_t j = j0 + tx * 4 + c;
      if (j >= dim) continue;
      T* p = x + i * ld + j;
      const double g = __dadd_rn(__ddiv_rn(acc[r][c], (double)S), __dmul_rn(l2, (double)*p));
      T gt = (T)g;
      if (noise) {
        gt = O::add(gt, noise[i * dim + j]);
      } else if (philox_mode) {
        const T nj = noise_component(z[c], coord_std, (T*)nullptr);
        nsq += (double)nj * (double)nj;
        gt = O::add(gt, nj);
      }
      if (!isfinite(gt)) bad = true;
      *p = O::sub(*p, O::mul(gamma, gt));
    }
  }
  if (bad) atomicOr(nonfinite, 1u);
  if (philox_mode) {
    for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(nsq_out, nsq);
  }
}

// value(theta) = sum_s softplus(-y m) / m + sum_j 0.5 l2 t^2, in order
// (optimizer.hpp:106-120), from the per-sample terms logit_coeff wrote.
__global__ void logit_value_finish(const double* __restrict__ ym, std::uint64_t S,
                                   const double* __restrict__ th, std::uint64_t dim, double l2,
                                   double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double f = 0.0;
  for (std::uint64_t sidx = 0; sidx < S; ++sidx) f = __dadd_rn(f, ym[sidx]);
  f = __ddiv_rn(f, (double)S);
  for (std::uint64_t j = 0; j < dim; ++j)
    f = __dadd_rn(f, __dmul_rn(__dmul_rn(__dmul_rn(0.5, l2), th[j]), th[j]));
  *out = f;
}

// pv inner product (optimizer.hpp:386-391), the weighted iterate
// (:411-417) and |g|^2 (:408), sequential in j.
__global__ void logit_vec_diag(const double* __restrict__ mean, const double* __restrict__ hat,
                               double* __restrict__ wsum, double w_k, double weight_total,
                               std::uint64_t dim, double* __restrict__ wtd,
                               double* __restrict__ pv_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double ip = 0.0;
  for (std::uint64_t j = 0; j < dim; ++j) {
    ip = __dadd_rn(ip, __dmul_rn(__dsub_rn(mean[j], hat[j]), __dadd_rn(mean[j], hat[j])));
    const double ws = __dadd_rn(wsum[j], __dmul_rn(w_k, mean[j]));
    wsum[j] = ws;
    wtd[j] = __ddiv_rn(ws, weight_total);
  }
  *pv_out = ip;
}

__global__ void sumsq_exact(const double* __restrict__ g, std::uint64_t dim,
                            double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (std::uint64_t j = 0; j < dim; ++j) s = __dadd_rn(s, __dmul_rn(g[j], g[j]));
  *out = s;
}

}  // namespace

// optimizer.hpp:39-44
std::vector<double> quad_curvature(std::uint64_t dim, double L, double mu) {
  std::vector<double> c(dim ? dim : 1);
  for (std::uint64_t j = 0; j < dim; ++j) {
    const double t = dim > 1 ? static_cast<double>(j) / static_cast<double>(dim - 1) : 0.0;
    c[j] = mu + (L - mu) * t;
  }
  if (dim == 1) c[0] = L;
  return c;
}

struct SgdRun {
  int dtype;
  std::size_t es;
  std::uint64_t dim, ld;
  cudaStream_t s;
  DeviceBuffer c64, t64, cT, tT, noise_dev, flag, npart, hat, mean, wsum, vpart, vout, dpart;
  DeviceBuffer rep, rlist, rcount;  // representatives after an averaging pass
  RoundTables tables;               // the fused averaging pass's round tables
  double noise_sq_host = 0.0;
  // LogisticRegression(xs, ys, l2): samples S, rows of xs are dim doubles.
  bool logit = false;
  std::uint64_t S = 0;
  double l2 = 0.0;
  DeviceBuffer lxs, lys, coeff, ym, gm, wtd;
  // fp32 tensor-core path (tc_logit.cu): tf32 hi/lo splits of X and X^T, and
  // per-step scratch for Theta's split and the split coefficients
  bool tc = false;
  DeviceBuffer x_hi, x_lo, xt_hi, xt_lo, th_hi, th_lo, c_hi, c_lo;

  void logit_upload(const double* xs, const double* ys, std::uint64_t samples, double l2_,
                    std::uint64_t n_max) {
    logit = true;
    S = samples;
    l2 = l2_;
    tc = dtype == MOSHPIT_F32 && logit_tc_enabled(dim, S);
    lxs.resize(S * dim * 8 + 16);
    lys.resize(S * 8 + 16);
    coeff.resize(n_max * S * 8 + 16);
    ym.resize(S * 8 + 16);
    gm.resize((dim ? dim : 1) * 8 + 16);
    wtd.resize((dim ? dim : 1) * 8 + 16);
    if (dim) MB_CUDA(cudaMemcpyAsync(lxs.ptr, xs, S * dim * 8, cudaMemcpyHostToDevice, s));
    MB_CUDA(cudaMemcpyAsync(lys.ptr, ys, S * 8, cudaMemcpyHostToDevice, s));
    if (tc) {
      for (DeviceBuffer* b : {&x_hi, &x_lo, &xt_hi, &xt_lo}) b->resize(S * dim * 4 + 16);
      for (DeviceBuffer* b : {&th_hi, &th_lo}) b->resize(n_max * dim * 4 + 16);
      for (DeviceBuffer* b : {&c_hi, &c_lo}) b->resize(n_max * S * 4 + 16);
      logit_tc_prepare(lxs.as<double>(), S, dim, x_hi.as<float>(), x_lo.as<float>(),
                       xt_hi.as<float>(), xt_lo.as<float>(), s);
    }
  }

  // optimizer.hpp:356-373 with LogisticRegression::gradient: margins/coefficients
  // for every (peer, sample), then gradient + update for every (peer, j).
  template <typename T>
  void lstep(void* x, std::uint64_t n, double gamma, double coord_std, int philox,
             std::uint64_t seed, std::uint64_t k, const T* noise_host_rows) {
    const T* nz = nullptr;
    if (noise_host_rows) {
      noise_dev.resize(n * dim * sizeof(T) + 16);
      MB_CUDA(cudaMemcpyAsync(noise_dev.ptr, noise_host_rows, n * dim * sizeof(T),
                              cudaMemcpyHostToDevice, s));
      nz = noise_dev.as<T>();
    }
    if (dim == 0) return;
    if constexpr (std::is_same_v<T, float>) {
      if (tc) {  // fp32 state: both GEMMs on the tensor cores (3xTF32)
        logit_tc_step(static_cast<float*>(x), n, ld, dim, S, x_hi.as<float>(), x_lo.as<float>(),
                      xt_hi.as<float>(), xt_lo.as<float>(), lys.as<double>(), l2, (float)gamma,
                      nz, coord_std, philox, seed, k, flag.as<std::uint32_t>(),
                      npart.as<double>() + k * 148 * 16, th_hi.as<float>(), th_lo.as<float>(),
                      c_hi.as<float>(), c_lo.as<float>(), s);
        return;
      }
    }
    const unsigned ty = (unsigned)((n + kLT - 1) / kLT);
    logit_coeff_tiled<T><<<dim3((unsigned)((S + kLT - 1) / kLT), ty), 256, 0, s>>>(
        static_cast<const T*>(x), n, ld, dim, lxs.as<double>(), lys.as<double>(), S,
        coeff.as<double>());
    // gradient tile TM x TN (see logit_grad_tiled); MOSHPIT_LOGIT_GTILE=64x32|64x16
    // are measurement knobs
    static const int gt = [] {
      const char* e = std::getenv("MOSHPIT_LOGIT_GTILE");
      if (!e) return 0;
      const std::string v(e);
      return v == "64x32" ? 1 : v == "64x16" ? 2 : 0;
    }();
    auto grad = [&](auto tm, auto tn) {
      constexpr int TM = decltype(tm)::value, TN = decltype(tn)::value;
      logit_grad_tiled<T, TM, TN><<<dim3((unsigned)((dim + TN - 1) / TN),
                                         (unsigned)((n + TM - 1) / TM)), TM * TN / 16, 0, s>>>(
          static_cast<T*>(x), n, ld, dim, lxs.as<double>(), S, coeff.as<double>(), l2, (T)gamma,
          nz, coord_std, philox, seed, k, flag.as<std::uint32_t>(),
          npart.as<double>() + k * 148 * 16);
    };
    using I64 = std::integral_constant<int, 64>;
    if (gt == 1) grad(I64{}, std::integral_constant<int, 32>{});
    else if (gt == 2) grad(I64{}, std::integral_constant<int, 16>{});
    else grad(I64{}, I64{});
    MB_LAUNCH_CHECK();
  }

  // f(mean), |grad f(mean)|^2, f(weighted) and the pv product into o[0..3]
  // (optimizer.hpp:383-417), each in the reference's summation order.
  void logit_diag(double w_k, double weight_total, double* o) {
    logit_vec_diag<<<1, 1, 0, s>>>(mean.as<double>(), hat.as<double>(), wsum.as<double>(), w_k,
                                   weight_total, dim, wtd.as<double>(), o);
    const unsigned sb = (unsigned)((S + 127) / 128);
    logit_coeff<double><<<dim3(sb, 1), 128, 0, s>>>(mean.as<double>(), dim, dim,
                                                   lxs.as<double>(), lys.as<double>(), S,
                                                   coeff.as<double>(), ym.as<double>());
    logit_value_finish<<<1, 1, 0, s>>>(ym.as<double>(), S, mean.as<double>(), dim, l2, o + 1);
    if (dim)
      logit_grad<double><<<dim3((unsigned)((dim + 127) / 128), 1), 128, 0, s>>>(
          mean.as<double>(), dim, dim, lxs.as<double>(), S, coeff.as<double>(), l2, 0, 0.0,
          nullptr, 0.0, 0, 0, 0, flag.as<std::uint32_t>(), nullptr, gm.as<double>(), 0);
    sumsq_exact<<<1, 1, 0, s>>>(gm.as<double>(), dim, o + 2);
    logit_coeff<double><<<dim3(sb, 1), 128, 0, s>>>(wtd.as<double>(), dim, dim,
                                                   lxs.as<double>(), lys.as<double>(), S,
                                                   nullptr, ym.as<double>());
    logit_value_finish<<<1, 1, 0, s>>>(ym.as<double>(), S, wtd.as<double>(), dim, l2, o + 3);
    MB_LAUNCH_CHECK();
  }

  template <typename T>
  void step(void* x, std::uint64_t n, double gamma, double coord_std, int philox,
            std::uint64_t seed, std::uint64_t k, const T* noise_host_rows) {
    const T* nz = nullptr;
    if (noise_host_rows) {
      noise_dev.resize(n * dim * sizeof(T) + 16);
      MB_CUDA(cudaMemcpyAsync(noise_dev.ptr, noise_host_rows, n * dim * sizeof(T),
                              cudaMemcpyHostToDevice, s));
      nz = noise_dev.as<T>();
    }
    constexpr int W = SVec<T>::W;
    if (ld % W == 0 && reinterpret_cast<std::uintptr_t>(x) % 16 == 0) {
      const unsigned grid = grid_for(n * ((dim + W - 1) / W), kStepThreads);
      sgd_step_vec<T><<<grid, kStepThreads, 0, s>>>(
          static_cast<T*>(x), n, dim, ld, cT.as<T>(), tT.as<T>(), (T)gamma, nz, coord_std,
          philox, philox_keys(seed), k, flag.as<std::uint32_t>(),
          npart.as<double>() + k * 148 * 16);
    } else {
      const unsigned grid = grid_for(n * ((dim + 3) / 4), kStepThreads);
      sgd_step_kernel<T><<<grid, kStepThreads, 0, s>>>(
          static_cast<T*>(x), n, dim, ld, cT.as<T>(), tT.as<T>(), (T)gamma, nz, coord_std,
          philox, seed, k, flag.as<std::uint32_t>(), npart.as<double>() + k * 148 * 16);
    }
    MB_LAUNCH_CHECK();
  }
};

}  // namespace mb200

using namespace mb200;

extern "C" {

// optimizer.hpp:231-242 local_step with Quadratic(dim, L, mu, target); the
// noise is drawn from *noise (the caller's RngStream), as the reference does.
int moshpit_local_step_quadratic(int dtype, void* theta, std::uint64_t dim, double L, double mu,
                                 const double* target, double gamma, double sigma,
                                 moshpit_rng_state* noise) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    if (L < mu || mu < 0.0) throw std::invalid_argument("Quadratic: need L >= mu >= 0");
    if (dim == 0) return;
    require_device();
    Xoshiro st;
    std::memcpy(st.s, noise->s, sizeof(st.s));
    st.have_spare = noise->have_spare != 0;
    st.spare = noise->spare;
    const double coord_std = sigma > 0.0 ? sigma / std::sqrt(static_cast<double>(dim)) : 0.0;
    std::vector<double> nz;
    if (coord_std > 0.0) {
      nz.resize(dim);
      for (auto& v : nz) v = coord_std * st.normal();
    }
    StreamHolder h;
    SgdRun r{dtype, es, dim, dim, h.s};
    const auto c = quad_curvature(dim, L, mu);
    r.cT.resize(dim * es);
    r.tT.resize(dim * es);
    r.flag.resize(16);
    r.npart.resize(148 * 16 * 8 + 16);
    DeviceBuffer x(dim * es + 16), tmp(dim * 8 + 16);
    MB_CUDA(cudaMemsetAsync(r.flag.ptr, 0, 16, h.s));
    MB_CUDA(cudaMemcpyAsync(x.ptr, theta, dim * es, cudaMemcpyHostToDevice, h.s));
    DeviceBuffer c64(dim * 8), t64(dim * 8);
    MB_CUDA(cudaMemcpyAsync(c64.ptr, c.data(), dim * 8, cudaMemcpyHostToDevice, h.s));
    MB_CUDA(cudaMemcpyAsync(t64.ptr, target, dim * 8, cudaMemcpyHostToDevice, h.s));
    const unsigned b = (unsigned)((dim + 255) / 256);
    if (dtype == MOSHPIT_F32) {
      cast_kernel<float><<<b, 256, 0, h.s>>>(c64.as<double>(), r.cT.as<float>(), dim);
      cast_kernel<float><<<b, 256, 0, h.s>>>(t64.as<double>(), r.tT.as<float>(), dim);
      std::vector<float> nzf(nz.begin(), nz.end());
      r.step<float>(x.ptr, 1, gamma, coord_std, 0, 0, 0, nz.empty() ? nullptr : nzf.data());
      MB_CUDA(cudaStreamSynchronize(h.s));
    } else {
      cast_kernel<double><<<b, 256, 0, h.s>>>(c64.as<double>(), r.cT.as<double>(), dim);
      cast_kernel<double><<<b, 256, 0, h.s>>>(t64.as<double>(), r.tT.as<double>(), dim);
      r.step<double>(x.ptr, 1, gamma, coord_std, 0, 0, 0, nz.empty() ? nullptr : nz.data());
      MB_CUDA(cudaStreamSynchronize(h.s));
    }
    std::uint32_t bad = 0;
    MB_CUDA(cudaMemcpy(&bad, r.flag.ptr, 4, cudaMemcpyDeviceToHost));
    if (bad) throw std::runtime_error("local_step: non-finite gradient");
    MB_CUDA(cudaMemcpy(theta, x.ptr, dim * es, cudaMemcpyDeviceToHost));
    std::memcpy(noise->s, st.s, sizeof(st.s));
    noise->have_spare = st.have_spare ? 1 : 0;
    noise->spare = st.spare;
  });
}

// The shared driver; lxs != nullptr selects LogisticRegression(lxs, lys, l2)
// (mu = l2, optimizer.hpp:141), else Quadratic(dim, L, mu, target).
static int run_sgd(
    int dtype, std::uint32_t M, std::uint32_t d, std::uint32_t T, std::uint32_t n_peers,
    std::uint64_t dim, double L, double mu, const double* target, const double* lxs,
    const double* lys, std::uint64_t samples, double l2, const double* theta0,
    double gamma, std::uint32_t tau, std::uint32_t steps, double sigma,
    std::uint32_t inner_rounds, std::uint64_t seed, const std::uint32_t* ev_step,
    const std::int32_t* ev_delta, std::uint64_t n_events, int diag, int noise_mode,
    double* f_gap, double* grad_norm_sq, double* f_gap_weighted, double* dispersion,
    double* final_mean, double* diag6, void* final_thetas, double* loop_ms) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    const bool logit = lxs != nullptr;
    if (logit) {
      if (samples == 0 || !lys) throw std::invalid_argument("LogisticRegression: bad dataset");
      mu = l2;
    } else if (L < mu || mu < 0.0) {
      throw std::invalid_argument("Quadratic: need L >= mu >= 0");
    }
    // OptimizerConfig::validate (optimizer.hpp:195-202)
    if (gamma <= 0.0) throw std::invalid_argument("OptimizerConfig: gamma > 0");
    if (tau < 1) throw std::invalid_argument("OptimizerConfig: tau >= 1");
    if (sigma < 0.0) throw std::invalid_argument("OptimizerConfig: sigma >= 0");
    if (M < 1 || d < 1 || T < 1)
      throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
    const std::uint64_t cap = moshpit_grid_capacity(M, d);
    if (n_peers < 1 || n_peers > cap) throw std::invalid_argument("OptimizerConfig: 1 <= N <= M^d");
    for (std::uint64_t e = 0; e < n_events; ++e)
      if (ev_delta[e] < 0 && static_cast<std::uint32_t>(-ev_delta[e]) >= n_peers)
        throw std::invalid_argument("run_moshpit_sgd: schedule kills everyone");
    if (diag < MOSHPIT_DIAG_NONE || diag > MOSHPIT_DIAG_EXACT)
      throw std::invalid_argument("run_moshpit_sgd: unknown diagnostics mode");
    if (noise_mode != 0 && noise_mode != 1)
      throw std::invalid_argument("run_moshpit_sgd: noise_mode must be 0 or 1");
    require_device();
    int dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    const std::uint32_t inner = inner_rounds == 0 ? d : inner_rounds;
    std::uint64_t n_max = n_peers;
    for (std::uint64_t e = 0; e < n_events; ++e)
      if (ev_delta[e] > 0) n_max += static_cast<std::uint64_t>(ev_delta[e]);
    StreamHolder h;
    SgdRun r{dtype, es, dim, padded_ld(dim, es), h.s};
    const std::uint64_t D = dim ? dim : 1;
    DeviceBuffer x(n_max * r.ld * es + 16), th0(D * 8);
    r.c64.resize(D * 8);
    r.t64.resize(D * 8);
    r.cT.resize(D * es);
    r.tT.resize(D * es);
    r.flag.resize(16);
    r.npart.resize((std::uint64_t)(steps + 1) * 148 * 16 * 8 + 16);
    r.hat.resize(D * 8);
    r.mean.resize(D * 8);
    r.wsum.resize(D * 8);
    const std::uint64_t nch = (dim + kChunk - 1) / kChunk;
    r.vpart.resize((nch + 1) * 4 * 8 + 64);
    r.dpart.resize(n_max * ((nch ? nch : 1) + 1) * 8 + 16);
    DeviceBuffer out((std::uint64_t)(steps + 1) * 8 * 8);
    MB_CUDA(cudaMemsetAsync(r.flag.ptr, 0, 16, h.s));
    MB_CUDA(cudaMemsetAsync(r.wsum.ptr, 0, D * 8, h.s));
    MB_CUDA(cudaMemsetAsync(r.npart.ptr, 0, r.npart.bytes, h.s));
    if (logit) {
      r.logit_upload(lxs, lys, samples, l2, n_max);
    } else {
      const auto c = quad_curvature(dim, L, mu);
      MB_CUDA(cudaMemcpyAsync(r.c64.ptr, c.data(), dim * 8, cudaMemcpyHostToDevice, h.s));
      MB_CUDA(cudaMemcpyAsync(r.t64.ptr, target, dim * 8, cudaMemcpyHostToDevice, h.s));
    }
    MB_CUDA(cudaMemcpyAsync(th0.ptr, theta0, dim * 8, cudaMemcpyHostToDevice, h.s));
    const unsigned b = (unsigned)((D + 255) / 256);
    if (dtype == MOSHPIT_F32) {
      cast_kernel<float><<<b, 256, 0, h.s>>>(r.c64.as<double>(), r.cT.as<float>(), dim);
      cast_kernel<float><<<b, 256, 0, h.s>>>(r.t64.as<double>(), r.tT.as<float>(), dim);
      broadcast_theta0<float><<<grid_for(n_peers * D, 256), 256, 0, h.s>>>(
          x.as<float>(), n_peers, r.ld, dim, th0.as<double>());
    } else {
      cast_kernel<double><<<b, 256, 0, h.s>>>(r.c64.as<double>(), r.cT.as<double>(), dim);
      cast_kernel<double><<<b, 256, 0, h.s>>>(r.t64.as<double>(), r.tT.as<double>(), dim);
      broadcast_theta0<double><<<grid_for(n_peers * D, 256), 256, 0, h.s>>>(
          x.as<double>(), n_peers, r.ld, dim, th0.as<double>());
    }
    MB_LAUNCH_CHECK();

    Xoshiro noise = Xoshiro::named(seed, "noise");
    Xoshiro avg = Xoshiro::named(seed, "averaging");
    Xoshiro join = Xoshiro::named(seed, "join");
    std::unique_ptr<Plane> plane;
    std::uint64_t n = n_peers;
    std::uint32_t n_min = n_peers;
    double noise_sq_sum = 0.0, weight_total = 0.0, w_k = 1.0;
    std::uint64_t noise_count = 0;
    const double w_growth = mu > 0.0 ? 1.0 / (1.0 - gamma * mu) : 1.0;
    const double coord_std = sigma > 0.0 ? sigma / std::sqrt(static_cast<double>(dim)) : 0.0;
    const int exact = diag == MOSHPIT_DIAG_EXACT;
    // DIAG_NONE: kernel 3 -- the local step rides in the first averaging
    // round's loads (one read + one write of the state for step + round 1).
    const bool fused =
        !logit && diag == MOSHPIT_DIAG_NONE && !(coord_std > 0.0 && noise_mode == 0);
    // MOSHPIT_SGD_FUSED_ROUNDS=1: the step plus every inner round in one pass
    // (temporal blocking, fused_rounds.cu; bit-identical).  Opt-in: at C4 it
    // measured 3.96 / 4.60 ms per step (sigma 0 / 1) against 2.87 / 3.07 for
    // kernel 3 + kernel 2 -- the shared-memory rounds are latency-bound
    // (profiles/r02/fused_rounds.md)
    const bool fused_rounds = [] {
      const char* e = std::getenv("MOSHPIT_SGD_FUSED_ROUNDS");
      return e && std::atoi(e) != 0;
    }();
    // Two averaging rounds per sync (d = 2, C4): the step and both rounds in
    // one pass (two_round_step_kernel, step_kernel.cu; bit-identical to kernel
    // 3 + kernel 2, half the HBM traffic).  Needs groups of <= 32 (M <= 32)
    // and at most two_round_max_groups() round-1 groups (<= M^(d-1) lines).
    // MOSHPIT_SGD_TWO_ROUND=0: kernel 3 + kernel 2.
    std::uint64_t g1_bound = 1;
    for (std::uint32_t q = 1; q < d && g1_bound <= two_round_max_groups(); ++q) g1_bound *= M;
    const bool two_round = [&] {
      const char* e = std::getenv("MOSHPIT_SGD_TWO_ROUND");
      if (e && std::atoi(e) == 0) return false;
      return inner == 2 && M <= 32 && g1_bound <= two_round_max_groups();
    }();
    // no per-step diagnostics: fused quadratic runs and logistic DIAG_NONE
    const bool skip_diag = fused || (logit && diag == MOSHPIT_DIAG_NONE);
    DeviceBuffer cpad, tpad;
    if (fused) {  // curvature / target padded to the row stride (zeros)
      cpad.resize(r.ld * es + 16);
      tpad.resize(r.ld * es + 16);
      MB_CUDA(cudaMemsetAsync(cpad.ptr, 0, r.ld * es, h.s));
      MB_CUDA(cudaMemsetAsync(tpad.ptr, 0, r.ld * es, h.s));
      MB_CUDA(cudaMemcpyAsync(cpad.ptr, r.cT.ptr, dim * es, cudaMemcpyDeviceToDevice, h.s));
      MB_CUDA(cudaMemcpyAsync(tpad.ptr, r.tT.ptr, dim * es, cudaMemcpyDeviceToDevice, h.s));
    }
    std::vector<double> nz64;
    std::vector<float> nz32;
    PinnedBuffer nz_pin;
    std::vector<double> wt_hist(steps);
    // the averaging plane of the initial population is built before the timed
    // loop (allocations are not part of a step); membership changes rebuild it
    if (n_peers > 1 && n_peers <= cap && steps >= tau)
      plane = std::make_unique<Plane>(M, d, n_peers, dev);
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (loop_ms) {
      MB_CUDA(cudaEventCreate(&ev0));
      MB_CUDA(cudaEventCreate(&ev1));
      MB_CUDA(cudaEventRecord(ev0, h.s));
    }
    for (std::uint32_t k = 0; k < steps; ++k) {
      for (std::uint64_t e = 0; e < n_events; ++e) {  // optimizer.hpp:337-350
        if (ev_step[e] != k) continue;
        if (ev_delta[e] < 0) {
          const std::uint64_t leave = static_cast<std::uint64_t>(-ev_delta[e]);
          if (leave >= n) throw std::runtime_error("run_moshpit_sgd: all peers vanished");
          n -= leave;
        } else {
          for (std::int32_t q = 0; q < ev_delta[e]; ++q) {
            const std::uint64_t donor = join.below(n);
            MB_CUDA(cudaMemcpyAsync(static_cast<char*>(x.ptr) + n * r.ld * es,
                                    static_cast<char*>(x.ptr) + donor * r.ld * es, r.ld * es,
                                    cudaMemcpyDeviceToDevice, h.s));
            ++n;
          }
        }
      }
      n_min = std::min<std::uint32_t>(n_min, static_cast<std::uint32_t>(n));
      // local step (optimizer.hpp:356-375)
      const void* host_noise = nullptr;
      if (coord_std > 0.0 && noise_mode == 0) {
        nz_pin.resize(n * dim * es + 16);
        MB_CUDA(cudaStreamSynchronize(h.s));  // the pinned buffer is reused per step
        for (std::uint64_t i = 0; i < n * dim; ++i) {
          const double nj = coord_std * noise.normal();
          noise_sq_sum += nj * nj;
          if (dtype == MOSHPIT_F32)
            nz_pin.as<float>()[i] = static_cast<float>(nj);
          else
            nz_pin.as<double>()[i] = nj;
        }
        host_noise = nz_pin.ptr;
      }
      noise_count += n;
      const int philox = (coord_std > 0.0 && noise_mode == 1) ? 1 : 0;
      const bool sync = (k + 1) % tau == 0 && n > 1;
      if (fused) {
        if (sync) {
          if (n > cap) throw std::invalid_argument("moshpit_average: N exceeds grid capacity M^d");
          if (!plane || plane->n != n) plane = std::make_unique<Plane>(M, d, n, dev);
          plane->init_cells(avg, h.s);
          StepPrologue<float> sf;
          StepPrologue<double> sd;
          double* np_slot = r.npart.as<double>() + (std::uint64_t)k * 148 * 16;
          sf = StepPrologue<float>{cpad.as<float>(), tpad.as<float>(), (float)gamma, coord_std,
                                   philox, seed, k, dim, r.flag.as<std::uint32_t>(), np_slot};
          sd = StepPrologue<double>{cpad.as<double>(), tpad.as<double>(), gamma, coord_std,
                                    philox, seed, k, dim, r.flag.as<std::uint32_t>(), np_slot};
          if (two_round) {
            r.tables.form(*plane, 2, nullptr, 0.0, avg, h.s);
            r.tables.scratch.resize(((std::uint64_t)n * 2 + 8 * two_round_max_groups() + 4) * 4);
            auto* g1 = r.tables.scratch.as<std::uint32_t>();
            const auto g1n = (std::uint32_t)std::min<std::uint64_t>(g1_bound, n);
            if (dtype == MOSHPIT_F32)
              launch_two_round_step<float>(x.as<float>(), r.ld, dim, (std::uint32_t)n,
                                           r.tables.host.data(), g1n, g1, g1 + n, sf, h.s);
            else
              launch_two_round_step<double>(x.as<double>(), r.ld, dim, (std::uint32_t)n,
                                            r.tables.host.data(), g1n, g1, g1 + n, sd, h.s);
            plane->mark_done(h.s);
          } else if (fused_rounds &&
                     inner <= fused_rounds_max(n, std::min<std::uint64_t>(plane->grid.lines(), n))) {
            const auto gcap = (std::uint32_t)std::min<std::uint64_t>(plane->grid.lines(), n);
            // the step and all `inner` rounds in one pass over the state
            // (temporal blocking): bit-identical to kernel 3 + kernel 2
            r.tables.form(*plane, inner, nullptr, 0.0, avg, h.s);
            if (dtype == MOSHPIT_F32)
              launch_rounds_fused<float>(x.as<float>(), r.ld, dim, (std::uint32_t)n, gcap,
                                         r.tables.dev(), inner, &sf, h.s);
            else
              launch_rounds_fused<double>(x.as<double>(), r.ld, dim, (std::uint32_t)n, gcap,
                                          r.tables.dev(), inner, &sd, h.s);
            plane->mark_done(h.s);
          } else {
            if (dtype == MOSHPIT_F32)
              plane->round(nullptr, 0.0, avg, dtype, x.ptr, dim, r.ld, h.s, MOSHPIT_KERNEL_AUTO,
                           &sf);
            else
              plane->round(nullptr, 0.0, avg, dtype, x.ptr, dim, r.ld, h.s, MOSHPIT_KERNEL_AUTO,
                           nullptr, &sd);
            for (std::uint32_t q = 1; q < inner; ++q)
              plane->round(nullptr, 0.0, avg, dtype, x.ptr, dim, r.ld, h.s, MOSHPIT_KERNEL_AUTO);
          }
        } else if (dtype == MOSHPIT_F32) {
          r.step<float>(x.ptr, n, gamma, coord_std, philox, seed, k, nullptr);
        } else {
          r.step<double>(x.ptr, n, gamma, coord_std, philox, seed, k, nullptr);
        }
        continue;
      }
      if (logit) {
        if (dtype == MOSHPIT_F32)
          r.lstep<float>(x.ptr, n, gamma, coord_std, philox, seed, k,
                         static_cast<const float*>(host_noise));
        else
          r.lstep<double>(x.ptr, n, gamma, coord_std, philox, seed, k,
                          static_cast<const double*>(host_noise));
      }
      // the noise-free step fused into hat theta = mean_of(post) for
      // n = 8 * 2^K: one pass over the state instead of the step's read +
      // write and the mean's read
      auto fused_hat = [&](auto* xs, auto* cs, auto* ts, auto g) {
        return !logit && !host_noise &&
               launch_step_colmean(xs, n, r.ld, dim, cs, ts, g, coord_std, philox, seed, k,
                                   r.flag.as<std::uint32_t>(),
                                   r.npart.as<double>() + (std::uint64_t)k * 148 * 16, 148 * 16,
                                   r.hat.as<double>(), h.s);
      };
      if (skip_diag) {
      } else if (dtype == MOSHPIT_F32) {
        if (!fused_hat(x.as<float>(), r.cT.as<float>(), r.tT.as<float>(), (float)gamma)) {
          if (!logit)
            r.step<float>(x.ptr, n, gamma, coord_std, philox, seed, k,
                          static_cast<const float*>(host_noise));
          launch_colmean<float, double>(x.as<float>(), n, r.ld, dim, nullptr,
                                        r.hat.as<double>(), h.s);
        }
      } else {
        if (!fused_hat(x.as<double>(), r.cT.as<double>(), r.tT.as<double>(), gamma)) {
          if (!logit)
            r.step<double>(x.ptr, n, gamma, coord_std, philox, seed, k,
                           static_cast<const double*>(host_noise));
          launch_colmean<double, double>(x.as<double>(), n, r.ld, dim, nullptr,
                                         r.hat.as<double>(), h.s);
        }
      }
      // averaging pass (optimizer.hpp:379-381, 249-284)
      if ((k + 1) % tau == 0 && n > 1) {
        if (n > cap) throw std::invalid_argument("moshpit_average: N exceeds grid capacity M^d");
        if (!plane || plane->n != n) plane = std::make_unique<Plane>(M, d, n, dev);
        plane->init_cells(avg, h.s);
        for (std::uint32_t q = 0; q < inner; ++q)
          plane->round(nullptr, 0.0, avg, dtype, x.ptr, dim, r.ld, h.s, MOSHPIT_KERNEL_AUTO);
      }
      if (skip_diag) continue;
      // after an averaging pass the diagnostics read one row per averaged
      // group of its last round (identical rows: bit-identical results)
      const bool synced = (k + 1) % tau == 0 && n > 1 && inner > 0;
      if (synced) {
        r.rep.resize(n * 4 + 16);
        r.rlist.resize(n * 4 + 16);
        r.rcount.resize(16);
        launch_build_reps(plane->members.as<std::uint32_t>(), plane->goff.as<std::uint32_t>(),
                          plane->gvoid.as<std::uint8_t>(), plane->counts.as<std::uint32_t>(), n,
                          r.rep.as<std::uint32_t>(), r.rlist.as<std::uint32_t>(),
                          r.rcount.as<std::uint32_t>(), h.s);
      }
      const std::uint32_t* rep_map = synced ? r.rep.as<std::uint32_t>() : nullptr;
      double* o = out.as<double>() + (std::uint64_t)k * 8;
      if (dtype == MOSHPIT_F32)
        launch_colmean<float, double>(x.as<float>(), n, r.ld, dim, rep_map, r.mean.as<double>(),
                                      h.s, true);
      else
        launch_colmean<double, double>(x.as<double>(), n, r.ld, dim, rep_map,
                                       r.mean.as<double>(), h.s, true);
      // V_k, FAST: (row, chunk) partials folded in (row, chunk) order; after an
      // averaging pass only the representatives' partials are computed
      auto dispersion_fast_any = [&](double* dst) {
        const std::uint64_t ch = nch ? nch : 1;
        double* rowsum = r.dpart.as<double>() + n_max * ch;  // the spare column
        if (rep_map) {
          const unsigned gy = (unsigned)std::min<std::uint64_t>(
              n, std::max<std::uint64_t>(1, 2 * 2368 / ch));
          if (dtype == MOSHPIT_F32)
            dispersion_fast_list<float><<<dim3((unsigned)ch, gy), kRed, 0, h.s>>>(
                x.as<float>(), r.ld, dim, r.mean.as<double>(), ch, r.dpart.as<double>(),
                r.rlist.as<std::uint32_t>(), r.rcount.as<std::uint32_t>());
          else
            dispersion_fast_list<double><<<dim3((unsigned)ch, gy), kRed, 0, h.s>>>(
                x.as<double>(), r.ld, dim, r.mean.as<double>(), ch, r.dpart.as<double>(),
                r.rlist.as<std::uint32_t>(), r.rcount.as<std::uint32_t>());
          row_sums<<<(unsigned)((n + 255) / 256), 256, 0, h.s>>>(r.dpart.as<double>(), n, ch,
                                                                  rep_map, rowsum);
          fold_all<<<1, 1, 0, h.s>>>(rowsum, n, (double)n, dst);
          return;
        }
        if (dtype == MOSHPIT_F32)
          dispersion_fast<float><<<dim3((unsigned)ch, (unsigned)n), kRed, 0, h.s>>>(
              x.as<float>(), r.ld, dim, r.mean.as<double>(), ch, r.dpart.as<double>());
        else
          dispersion_fast<double><<<dim3((unsigned)ch, (unsigned)n), kRed, 0, h.s>>>(
              x.as<double>(), r.ld, dim, r.mean.as<double>(), ch, r.dpart.as<double>());
        row_sums<<<(unsigned)((n + 255) / 256), 256, 0, h.s>>>(r.dpart.as<double>(), n, ch,
                                                                nullptr, rowsum);
        fold_all<<<1, 1, 0, h.s>>>(rowsum, n, (double)n, dst);
      };
      w_k *= w_growth;
      weight_total += w_k;
      wt_hist[k] = weight_total;
      if (logit) {
        r.logit_diag(w_k, weight_total, o);
        if (exact) {
          if (dtype == MOSHPIT_F32)
            dispersion_exact<float><<<1, 1, 0, h.s>>>(x.as<float>(), n, r.ld, dim,
                                                      r.mean.as<double>(), o + 4);
          else
            dispersion_exact<double><<<1, 1, 0, h.s>>>(x.as<double>(), n, r.ld, dim,
                                                       r.mean.as<double>(), o + 4);
        } else {
          dispersion_fast_any(o + 4);
        }
      } else if (exact) {
        sgd_vec_exact<<<1, 1, 0, h.s>>>(r.mean.as<double>(), r.hat.as<double>(),
                                        r.c64.as<double>(), r.t64.as<double>(),
                                        r.wsum.as<double>(), w_k, weight_total, dim, o);
        if (dtype == MOSHPIT_F32)
          dispersion_exact<float><<<1, 1, 0, h.s>>>(x.as<float>(), n, r.ld, dim,
                                                    r.mean.as<double>(), o + 4);
        else
          dispersion_exact<double><<<1, 1, 0, h.s>>>(x.as<double>(), n, r.ld, dim,
                                                     r.mean.as<double>(), o + 4);
      } else {
        const std::uint64_t ch = nch ? nch : 1;
        sgd_vec_fast<<<(unsigned)ch, kRed, 0, h.s>>>(r.mean.as<double>(), r.hat.as<double>(),
                                                    r.c64.as<double>(), r.t64.as<double>(),
                                                    r.wsum.as<double>(), w_k, weight_total, dim,
                                                    r.vpart.as<double>());
        sgd_vec_fold<<<1, 1, 0, h.s>>>(r.vpart.as<double>(), ch, o);
        dispersion_fast_any(o + 4);
      }
      MB_LAUNCH_CHECK();
    }
    if (loop_ms) MB_CUDA(cudaEventRecord(ev1, h.s));
    if (skip_diag) {
      if (dtype == MOSHPIT_F32)
        launch_colmean<float, double>(x.as<float>(), n, r.ld, dim, nullptr, r.mean.as<double>(),
                                      h.s);
      else
        launch_colmean<double, double>(x.as<double>(), n, r.ld, dim, nullptr,
                                       r.mean.as<double>(), h.s);
      const double nan = std::nan("");
      std::vector<double> fill((std::uint64_t)steps * 8 + 8, nan);
      MB_CUDA(cudaMemcpyAsync(out.ptr, fill.data(), (std::uint64_t)steps * 64,
                              cudaMemcpyHostToDevice, h.s));
    }
    std::vector<double> hout((std::uint64_t)steps * 8 + 8);
    MB_CUDA(cudaMemcpyAsync(hout.data(), out.ptr, (std::uint64_t)steps * 64, cudaMemcpyDeviceToHost,
                            h.s));
    std::vector<double> hnp;
    if (noise_mode == 1 && coord_std > 0.0) {
      hnp.resize((std::uint64_t)steps * 148 * 16);
      MB_CUDA(cudaMemcpyAsync(hnp.data(), r.npart.ptr, hnp.size() * 8, cudaMemcpyDeviceToHost, h.s));
    }
    if (final_mean)
      MB_CUDA(cudaMemcpyAsync(final_mean, r.mean.ptr, dim * 8, cudaMemcpyDeviceToHost, h.s));
    if (final_thetas)
      MB_CUDA(cudaMemcpy2DAsync(final_thetas, dim * es, x.ptr, r.ld * es, dim * es, n,
                                cudaMemcpyDeviceToHost, h.s));
    MB_CUDA(cudaStreamSynchronize(h.s));
    if (loop_ms) {
      float ms = 0.f;
      MB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
      *loop_ms = ms;
      cudaEventDestroy(ev0);
      cudaEventDestroy(ev1);
    }
    std::uint32_t bad = 0;
    MB_CUDA(cudaMemcpy(&bad, r.flag.ptr, 4, cudaMemcpyDeviceToHost));
    if (bad) throw std::runtime_error("run_moshpit_sgd: non-finite gradient");
    for (double v : hnp) noise_sq_sum += v;
    double pv_max = skip_diag ? std::nan("") : 0.0;
    for (std::uint32_t k = 0; k < steps && !skip_diag; ++k) {
      const double* o = hout.data() + (std::uint64_t)k * 8;
      pv_max = std::max(pv_max, o[0]);
      f_gap[k] = o[1] - 0.0;
      grad_norm_sq[k] = o[2];
      f_gap_weighted[k] = o[3] - 0.0;
      dispersion[k] = o[4];
    }
    if (skip_diag)
      for (std::uint32_t k = 0; k < steps; ++k)
        f_gap[k] = grad_norm_sq[k] = f_gap_weighted[k] = dispersion[k] = std::nan("");
    double v_sync_max = skip_diag ? std::nan("") : 0.0;
    for (std::uint32_t k = tau - 1; k < steps && !skip_diag; k += tau)
      v_sync_max = std::max(v_sync_max, dispersion[k]);
    diag6[0] = std::sqrt(v_sync_max) / gamma;
    diag6[1] = noise_count > 0 && sigma > 0.0
                   ? std::sqrt(noise_sq_sum / static_cast<double>(noise_count))
                   : 0.0;
    diag6[2] = 0.0;
    diag6[3] = std::sqrt(std::max(0.0, pv_max)) / gamma;
    diag6[4] = n_min;
    diag6[5] = static_cast<double>(n);
  });
}

// optimizer.hpp:297-439 run_moshpit_sgd with Quadratic(dim, L, mu, target).
// noise_mode 0: the reference "noise" stream (host draws, bit-exact);
// noise_mode 1: device Philox normals (statistical parity).
// diag: MOSHPIT_DIAG_EXACT or MOSHPIT_DIAG_FAST.  diag6 = {delta_aq_hat,
// sigma_hat, delta_pv1_hat, delta_pv2_hat, n_min, n_final}.
int moshpit_run_moshpit_sgd_quadratic(
    int dtype, std::uint32_t M, std::uint32_t d, std::uint32_t T, std::uint32_t n_peers,
    std::uint64_t dim, double L, double mu, const double* target, const double* theta0,
    double gamma, std::uint32_t tau, std::uint32_t steps, double sigma,
    std::uint32_t inner_rounds, std::uint64_t seed, const std::uint32_t* ev_step,
    const std::int32_t* ev_delta, std::uint64_t n_events, int diag, int noise_mode,
    double* f_gap, double* grad_norm_sq, double* f_gap_weighted, double* dispersion,
    double* final_mean, double* diag6, void* final_thetas, double* loop_ms) {
  return run_sgd(dtype, M, d, T, n_peers, dim, L, mu, target, nullptr, nullptr, 0, 0.0, theta0,
                 gamma, tau, steps, sigma, inner_rounds, seed, ev_step, ev_delta, n_events, diag,
                 noise_mode, f_gap, grad_norm_sq, f_gap_weighted, dispersion, final_mean, diag6,
                 final_thetas, loop_ms);
}

// optimizer.hpp:297-439 run_moshpit_sgd with LogisticRegression(xs, ys, l2)
// (optimizer.hpp:75-146): xs is samples x dim row-major fp64, ys in {-1,+1}.
// Diagnostics are always the reference's sequential orders (the objective's
// own evaluation dominates them); diag only selects NONE vs. computed.
int moshpit_run_moshpit_sgd_logistic(
    int dtype, std::uint32_t M, std::uint32_t d, std::uint32_t T, std::uint32_t n_peers,
    std::uint64_t dim, const double* xs, const double* ys, std::uint64_t samples, double l2,
    const double* theta0, double gamma, std::uint32_t tau, std::uint32_t steps, double sigma,
    std::uint32_t inner_rounds, std::uint64_t seed, const std::uint32_t* ev_step,
    const std::int32_t* ev_delta, std::uint64_t n_events, int diag, int noise_mode,
    double* f_gap, double* grad_norm_sq, double* f_gap_weighted, double* dispersion,
    double* final_mean, double* diag6, void* final_thetas, double* loop_ms) {
  if (!xs) return guarded([] { throw std::invalid_argument("LogisticRegression: bad dataset"); });
  return run_sgd(dtype, M, d, T, n_peers, dim, 0.0, 0.0, nullptr, xs, ys, samples, l2, theta0,
                 gamma, tau, steps, sigma, inner_rounds, seed, ev_step, ev_delta, n_events, diag,
                 noise_mode, f_gap, grad_norm_sq, f_gap_weighted, dispersion, final_mean, diag6,
                 final_thetas, loop_ms);
}

// LogisticRegression::synthetic (optimizer.hpp:89-104): the dataset is drawn
// on the host from the caller's stream (it is setup, not the hot path).
int moshpit_logistic_synthetic(std::uint64_t dim, std::uint64_t samples,
                               moshpit_rng_state* stream, double* xs, double* ys) {
  return guarded([&] {
    Xoshiro st;
    std::memcpy(st.s, stream->s, sizeof(st.s));
    st.have_spare = stream->have_spare != 0;
    st.spare = stream->spare;
    std::vector<double> truth(dim);
    for (auto& t : truth) t = st.normal();
    for (std::uint64_t i = 0; i < samples; ++i) {
      double dot = 0.0;
      for (std::uint64_t j = 0; j < dim; ++j) {
        xs[i * dim + j] = st.normal();
        dot += xs[i * dim + j] * truth[j];
      }
      ys[i] = dot + 0.1 * st.normal() > 0.0 ? 1.0 : -1.0;
    }
    std::memcpy(stream->s, st.s, sizeof(st.s));
    stream->have_spare = st.have_spare ? 1 : 0;
    stream->spare = st.spare;
  });
}

// value / gradient (GPU) and smoothness (the constructor's trace bound,
// optimizer.hpp:82-86) of LogisticRegression(xs, ys, l2) at theta.
int moshpit_logistic_eval(const double* xs, const double* ys, std::uint64_t samples,
                          std::uint64_t dim, double l2, const double* theta, double* value,
                          double* grad, double* smoothness) {
  return guarded([&] {
    if (!xs || !ys || samples == 0) throw std::invalid_argument("LogisticRegression: bad dataset");
    if (smoothness) {
      double trace = 0.0;
      for (std::uint64_t i = 0; i < samples * dim; ++i) trace += xs[i] * xs[i];
      *smoothness = trace / (4.0 * static_cast<double>(samples)) + l2;
    }
    if (!value && !grad) return;
    require_device();
    StreamHolder h;
    SgdRun r{MOSHPIT_F64, 8, dim, dim, h.s};
    r.flag.resize(16);
    r.logit_upload(xs, ys, samples, l2, 1);
    DeviceBuffer th((dim ? dim : 1) * 8 + 16), o(64);
    if (dim) MB_CUDA(cudaMemcpyAsync(th.ptr, theta, dim * 8, cudaMemcpyHostToDevice, h.s));
    MB_CUDA(cudaMemsetAsync(r.gm.ptr, 0, (dim ? dim : 1) * 8, h.s));
    logit_coeff<double><<<dim3((unsigned)((samples + 127) / 128), 1), 128, 0, h.s>>>(
        th.as<double>(), dim, dim, r.lxs.as<double>(), r.lys.as<double>(), samples,
        r.coeff.as<double>(), r.ym.as<double>());
    logit_value_finish<<<1, 1, 0, h.s>>>(r.ym.as<double>(), samples, th.as<double>(), dim, l2,
                                         o.as<double>());
    if (dim)
      logit_grad<double><<<dim3((unsigned)((dim + 127) / 128), 1), 128, 0, h.s>>>(
          th.as<double>(), dim, dim, r.lxs.as<double>(), samples, r.coeff.as<double>(), l2, 0,
          0.0, nullptr, 0.0, 0, 0, 0, r.flag.as<std::uint32_t>(), nullptr, r.gm.as<double>(), 0);
    MB_LAUNCH_CHECK();
    if (value) MB_CUDA(cudaMemcpyAsync(value, o.ptr, 8, cudaMemcpyDeviceToHost, h.s));
    if (grad && dim)
      MB_CUDA(cudaMemcpyAsync(grad, r.gm.ptr, dim * 8, cudaMemcpyDeviceToHost, h.s));
    MB_CUDA(cudaStreamSynchronize(h.s));
  });
}

// optimizer.hpp:231-242 local_step with LogisticRegression(xs, ys, l2).
int moshpit_local_step_logistic(int dtype, void* theta, std::uint64_t dim, const double* xs,
                                const double* ys, std::uint64_t samples, double l2,
                                double gamma, double sigma, moshpit_rng_state* noise) {
  return guarded([&] {
    const std::size_t es = elem_size(dtype);
    if (!xs || !ys || samples == 0) throw std::invalid_argument("LogisticRegression: bad dataset");
    if (dim == 0) return;
    require_device();
    Xoshiro st;
    std::memcpy(st.s, noise->s, sizeof(st.s));
    st.have_spare = noise->have_spare != 0;
    st.spare = noise->spare;
    const double coord_std = sigma > 0.0 ? sigma / std::sqrt(static_cast<double>(dim)) : 0.0;
    std::vector<double> nz;
    if (coord_std > 0.0) {
      nz.resize(dim);
      for (auto& v : nz) v = coord_std * st.normal();
    }
    StreamHolder h;
    SgdRun r{dtype, es, dim, dim, h.s};
    r.flag.resize(16);
    r.npart.resize(148 * 16 * 8 + 16);
    MB_CUDA(cudaMemsetAsync(r.flag.ptr, 0, 16, h.s));
    r.logit_upload(xs, ys, samples, l2, 1);
    DeviceBuffer x(dim * es + 16);
    MB_CUDA(cudaMemcpyAsync(x.ptr, theta, dim * es, cudaMemcpyHostToDevice, h.s));
    if (dtype == MOSHPIT_F32) {
      std::vector<float> nzf(nz.begin(), nz.end());
      r.lstep<float>(x.ptr, 1, gamma, coord_std, 0, 0, 0, nz.empty() ? nullptr : nzf.data());
      MB_CUDA(cudaStreamSynchronize(h.s));
    } else {
      r.lstep<double>(x.ptr, 1, gamma, coord_std, 0, 0, 0, nz.empty() ? nullptr : nz.data());
      MB_CUDA(cudaStreamSynchronize(h.s));
    }
    std::uint32_t bad = 0;
    MB_CUDA(cudaMemcpy(&bad, r.flag.ptr, 4, cudaMemcpyDeviceToHost));
    if (bad) throw std::runtime_error("local_step: non-finite gradient");
    MB_CUDA(cudaMemcpy(theta, x.ptr, dim * es, cudaMemcpyDeviceToHost));
    std::memcpy(noise->s, st.s, sizeof(st.s));
    noise->have_spare = st.have_spare ? 1 : 0;
    noise->spare = st.spare;
  });
}

}  // extern "C"
