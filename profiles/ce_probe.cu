// ce_probe.cu -- copy-engine peer pulls vs SM peer loads over NVLink.
// Every GPU pulls `bytes` from each other GPU at once (all-to-all ingress),
// either with cudaMemcpyPeerAsync (copy engines, one stream per source) or
// with an SM kernel of 128-bit loads (+ local stores).  Prints per-GPU
// ingress GB/s.  nvcc -arch=sm_100a -O3 ce_probe.cu -o ce_probe
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                          \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__global__ void pull(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// TMA bulk pull: one thread per CTA streams CH-byte chunks of the peer buffer
// into a shared-memory ring (cp.async.bulk g2s, mbarrier complete_tx) and
// writes each chunk back out with a bulk s2g store to local memory.
constexpr int CH = 16384, ST = 8;
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__global__ void bulk_pull(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) char ring[];
  __shared__ __align__(8) unsigned long long bar[ST];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < ST; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t n = bytes / CH;
  unsigned phase[ST] = {0};
  size_t issued = 0, done = 0;
  size_t mine[ST];
  for (size_t c = blockIdx.x; c < n || done < issued;) {
    // issue while there is room
    while (c < n && issued - done < ST) {
      const int slot = issued % ST;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[slot])), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(ring + (size_t)slot * CH)), "l"(src + c * CH), "r"(CH), "r"(smem_u32(&bar[slot])) : "memory");
      mine[slot] = c;
      ++issued;
      c += gridDim.x;
    }
    const int slot = done % ST;
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
                 ::"r"(smem_u32(&bar[slot])), "r"(phase[slot]) : "memory");
    phase[slot] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + mine[slot] * CH),
                 "r"(smem_u32(ring + (size_t)slot * CH)), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slot reusable
    ++done;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  int G = 0;
  CK(cudaGetDeviceCount(&G));
  if (argc > 1) G = atoi(argv[1]) < G ? atoi(argv[1]) : G;
  if (G < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  const size_t bytes = (size_t)2 << 30;  // per (dst, src) pair
  std::vector<void*> src(G), dst(G * G);
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; ++h)
      if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    cudaGetLastError();
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMemset(src[g], 1, bytes));
    for (int h = 0; h < G; ++h)
      if (h != g) CK(cudaMalloc(&dst[g * G + h], bytes));
  }
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaFuncSetAttribute(bulk_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST));
  }
  for (int mode = 0; mode < 5; ++mode) {
    const char* name = mode == 0 ? "copy engine (memcpyPeerAsync)" :
                       mode == 1 ? "SM loads, grid 148x4" : mode == 2 ? "SM loads, grid 148x8" :
                       mode == 3 ? "TMA bulk ring, 1 CTA/SM" : "TMA bulk ring, 2 CTA/SM";
    std::vector<double> gbs(G);
    for (int rep = 0; rep < 3; ++rep) {
      std::vector<std::thread> th;
      for (int g = 0; g < G; ++g)
        th.emplace_back([&, g] {
          cudaSetDevice(g);
          std::vector<cudaStream_t> st(G);
          for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
          cudaDeviceSynchronize();
          auto t0 = std::chrono::steady_clock::now();
          for (int h = 0; h < G; ++h) {
            if (h == g) continue;
            if (mode == 0)
              cudaMemcpyPeerAsync(dst[g * G + h], g, src[h], h, bytes, st[h]);
            else if (mode >= 3)
              bulk_pull<<<148 * (mode - 2) / (G - 1) + 1, 32, CH * ST, st[h]>>>(
                  (const char*)src[h], (char*)dst[g * G + h], bytes);
            else
              pull<<<148 * (mode == 1 ? 4 : 8) / (G - 1) + 1, 256, 0, st[h]>>>(
                  (const float4*)src[h], (float4*)dst[g * G + h], bytes / 16);
          }
          cudaDeviceSynchronize();
          double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          gbs[g] = (double)bytes * (G - 1) / s / 1e9;
          for (auto& s2 : st) cudaStreamDestroy(s2);
        });
      for (auto& t : th) t.join();
    }
    printf("%-32s G=%d ingress per GPU:", name, G);
    for (int g = 0; g < G; ++g) printf(" %.0f", gbs[g]);
    printf(" GB/s\n");
  }
  return 0;
}
