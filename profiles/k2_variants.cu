// k2_variants.cu -- design-space probe for Kernel 2 (segmented group mean) on
// C2's shape: 1024 rows x 4 Mi fp32, 32 groups of 32 members in random order.
// Every variant evaluates the same reference tree (bit-identical results are
// checked against variant A); only memory hints / occupancy / work split
// differ.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false
//                 -o k2v profiles/k2_variants.cu ; run: ./k2v
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                           \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 div4(float4 a, float n) {
  return make_float4(__fdiv_rn(a.x, n), __fdiv_rn(a.y, n), __fdiv_rn(a.z, n), __fdiv_rn(a.w, n));
}
template <int N, int B>
__device__ __forceinline__ float4 tree(const float4 (&x)[32]) {
  if constexpr (N <= 8) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < N; ++i) s = add4(s, x[B + i]);
    return s;
  } else {
    return add4(tree<N / 2, B>(x), tree<N - N / 2, B + N / 2>(x));
  }
}
template <int N, int B>
__device__ __forceinline__ float4 tree16(const float4 (&x)[16]) {
  if constexpr (N <= 8) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < N; ++i) s = add4(s, x[B + i]);
    return s;
  } else {
    return add4(tree16<N / 2, B>(x), tree16<N - N / 2, B + N / 2>(x));
  }
}

enum { LD_CS = 0, LD_NC = 1, LD_DEF = 2 };
enum { ST_CS = 0, ST_WB = 1 };

template <int LD>
__device__ __forceinline__ float4 ld(const float4* p) {
  if constexpr (LD == LD_CS) return __ldcs(p);
  if constexpr (LD == LD_NC) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
  }
  return *p;
}
template <int ST>
__device__ __forceinline__ void st(float4* p, float4 v) {
  if constexpr (ST == ST_CS) __stcs(p, v);
  else *p = v;
}

// A-E: thread = one float4 column, all 32 members in registers.
template <int LD, int ST, int MINB, int TH = 128>
__global__ void __launch_bounds__(TH, MINB)
    k_full(float4* base, std::uint64_t ldv, std::uint64_t nvec, const std::uint32_t* members,
           std::uint32_t ngroups) {
  __shared__ std::uint32_t ids[32];
  const std::uint64_t ntiles = (nvec + TH - 1) / TH, nitems = ngroups * ntiles;
  std::uint32_t cached = ~0u;
  for (std::uint64_t w = blockIdx.x; w < nitems; w += gridDim.x) {
    const std::uint32_t g = (std::uint32_t)(w / ntiles);
    if (g != cached) {
      __syncthreads();
      if (threadIdx.x < 32) ids[threadIdx.x] = members[g * 32 + threadIdx.x];
      cached = g;
      __syncthreads();
    }
    const std::uint64_t col = (w % ntiles) * TH + threadIdx.x;
    if (col >= nvec) continue;
    float4 x[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = ld<LD>(base + ids[k] * ldv + col);
    const float4 m = div4(tree<32, 0>(x), 32.f);
#pragma unroll
    for (int k = 0; k < 32; ++k) st<ST>(base + ids[k] * ldv + col, m);
  }
}

// G: two sequential halves of 16 members per thread (64 value registers).
template <int MINB>
__global__ void __launch_bounds__(128, MINB)
    k_halves(float4* base, std::uint64_t ldv, std::uint64_t nvec, const std::uint32_t* members,
             std::uint32_t ngroups) {
  __shared__ std::uint32_t ids[32];
  const std::uint64_t ntiles = (nvec + 127) / 128, nitems = ngroups * ntiles;
  std::uint32_t cached = ~0u;
  for (std::uint64_t w = blockIdx.x; w < nitems; w += gridDim.x) {
    const std::uint32_t g = (std::uint32_t)(w / ntiles);
    if (g != cached) {
      __syncthreads();
      if (threadIdx.x < 32) ids[threadIdx.x] = members[g * 32 + threadIdx.x];
      cached = g;
      __syncthreads();
    }
    const std::uint64_t col = (w % ntiles) * 128 + threadIdx.x;
    if (col >= nvec) continue;
    float4 x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = __ldcs(base + ids[k] * ldv + col);
    const float4 lo = tree16<16, 0>(x);
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = __ldcs(base + ids[16 + k] * ldv + col);
    const float4 m = div4(add4(lo, tree16<16, 0>(x)), 32.f);
#pragma unroll
    for (int k = 0; k < 32; ++k) __stcs(base + ids[k] * ldv + col, m);
  }
}

// H: half-warp split -- lanes 0-15 hold members 0-15, lanes 16-31 members
// 16-31 of the same 16 columns; one shuffle joins the halves (the top split of
// the reference tree for n = 32), each half stores its 16 rows.
template <int MINB>
__global__ void __launch_bounds__(128, MINB)
    k_split(float4* base, std::uint64_t ldv, std::uint64_t nvec, const std::uint32_t* members,
            std::uint32_t ngroups) {
  __shared__ std::uint32_t ids[32];
  const std::uint64_t ntiles = (nvec + 63) / 64, nitems = ngroups * ntiles;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = lane >> 4;
  std::uint32_t cached = ~0u;
  for (std::uint64_t w = blockIdx.x; w < nitems; w += gridDim.x) {
    const std::uint32_t g = (std::uint32_t)(w / ntiles);
    if (g != cached) {
      __syncthreads();
      if (threadIdx.x < 32) ids[threadIdx.x] = members[g * 32 + threadIdx.x];
      cached = g;
      __syncthreads();
    }
    const std::uint64_t col = (w % ntiles) * 64 + warp * 16 + (lane & 15);
    const bool ok = col < nvec;
    float4 x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      x[k] = ok ? __ldcs(base + ids[half * 16 + k] * ldv + col) : make_float4(0, 0, 0, 0);
    const float4 mine = tree16<16, 0>(x);
    float4 other;
    other.x = __shfl_xor_sync(0xffffffffu, mine.x, 16);
    other.y = __shfl_xor_sync(0xffffffffu, mine.y, 16);
    other.z = __shfl_xor_sync(0xffffffffu, mine.z, 16);
    other.w = __shfl_xor_sync(0xffffffffu, mine.w, 16);
    const float4 s = half ? add4(other, mine) : add4(mine, other);  // S(0..15) + S(16..31)
    const float4 m = div4(s, 32.f);
    if (ok) {
#pragma unroll
      for (int k = 0; k < 16; ++k) __stcs(base + ids[half * 16 + k] * ldv + col, m);
    }
  }
}

__global__ void fill(float* x, std::uint64_t n) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (std::uint64_t)gridDim.x * blockDim.x) {
    std::uint64_t z = i * 0x9E3779B97F4A7C15ULL;
    z ^= z >> 31;
    x[i] = (float)((z >> 40) & 0xffffff) * 0x1.0p-24f;
  }
}

int main() {
  const std::uint64_t rows = 1024, D = 1ull << 22, nvec = D / 4;
  const std::uint32_t ngroups = 32;
  float* x;
  float* x0;
  std::uint32_t* members;
  CK(cudaMalloc(&x, rows * D * 4));
  CK(cudaMalloc(&x0, rows * D * 4));
  CK(cudaMalloc(&members, rows * 4));
  std::vector<std::uint32_t> perm(rows);
  std::iota(perm.begin(), perm.end(), 0u);
  std::mt19937 rng(7);
  std::shuffle(perm.begin(), perm.end(), rng);
  CK(cudaMemcpy(members, perm.data(), rows * 4, cudaMemcpyHostToDevice));
  fill<<<148 * 16, 256>>>(x0, rows * D);
  CK(cudaDeviceSynchronize());
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ref;
  auto run = [&](const char* name, auto kern, int grid, int th = 128) -> int {
    CK(cudaMemcpy(x, x0, rows * D * 4, cudaMemcpyDeviceToDevice));
    kern<<<grid, th>>>((float4*)x, nvec, nvec, members, ngroups);  // one round for the check
    CK(cudaDeviceSynchronize());
    std::vector<float> h(8192);
    CK(cudaMemcpy(h.data(), x + 123 * D + 4096, 8192 * 4, cudaMemcpyDeviceToHost));
    const bool same = ref.empty() || std::equal(h.begin(), h.end(), ref.begin());
    if (ref.empty()) ref = h;
    const int iters = 20;
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) kern<<<grid, th>>>((float4*)x, nvec, nvec, members, ngroups);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = 2.0 * rows * D * 4 * iters / (ms / 1e3) / 1e9;
    printf("%-44s grid %5d  %7.3f ms/round  %7.1f GB/s  %s\n", name, grid, ms / iters, gbs,
           same ? "bit-identical" : "MISMATCH");
    return 0;
  };
  int per = 0;
  auto occ = [&](auto k) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 128, 0);
    return sms * per;
  };
  run("A full32 ldcs/stcs minB3 (current)", k_full<LD_CS, ST_CS, 3>, occ(k_full<LD_CS, ST_CS, 3>));
  run("E2 ldcs/stcs 128thr grid=1/SM", k_full<LD_CS, ST_CS, 1>, sms);
  run("E3 default 128thr grid=1/SM", k_full<LD_DEF, ST_WB, 1>, sms);
  run("E4 ldcs/stcs 256thr grid=1/SM", k_full<LD_CS, ST_CS, 1, 256>, sms, 256);
  run("E5 default 256thr grid=1/SM", k_full<LD_DEF, ST_WB, 1, 256>, sms, 256);
  run("E6 ldcs/stcs 64thr grid=1/SM", k_full<LD_CS, ST_CS, 1, 64>, sms, 64);
  run("E7 ldcs/stcs 64thr grid=2/SM", k_full<LD_CS, ST_CS, 2, 64>, sms * 2, 64);
  run("E8 ldcs/stcs 256thr grid=2/SM", k_full<LD_CS, ST_CS, 1, 256>, sms * 2, 256);
  run("E9 ld.nc/stcs 256thr grid=1/SM", k_full<LD_NC, ST_CS, 1, 256>, sms, 256);
  run("E10 ldcs/stcs 128thr grid=148*3/2", k_full<LD_CS, ST_CS, 2>, sms * 3 / 2);
  // plain copy of the same bytes for reference
  {
    float* y;
    CK(cudaMalloc(&y, rows * D * 4));
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) cudaMemcpyAsync(y, x, rows * D * 4, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s             %7.3f ms/copy   %7.1f GB/s\n", "cudaMemcpy D2D (same bytes)", ms / 10,
           2.0 * rows * D * 4 * 10 / (ms / 1e3) / 1e9);
  }
  return 0;
}
