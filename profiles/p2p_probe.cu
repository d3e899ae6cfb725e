// p2p_probe.cu -- NVLink ceiling for the cross-GPU Moshpit round's traffic
// pattern on 2 GPUs (one process, peer access enabled): every GPU reads from
// (and/or writes to) the other's HBM at the same time, with LDG/STG.128 from
// a full grid, as the fused cross kernel does.  Reports per-GPU ingress GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p profiles/p2p_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                          \
      return 1;                                                               \
    }                                                                         \
  } while (0)

// mode 0: read remote; 1: write remote; 2: read remote + write remote (half each)
__global__ void k(float4* __restrict__ local, float4* __restrict__ remote, std::uint64_t n,
                  int mode) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (std::uint64_t)gridDim.x * blockDim.x) {
    if (mode == 0) {
      float4 v = remote[i];
      acc.x += v.x;
      acc.y += v.y;
    } else if (mode == 1) {
      remote[i] = make_float4(1.f, 2.f, 3.f, (float)i);
    } else {
      if (i & 1) {
        float4 v = remote[i];
        acc.x += v.x;
      } else {
        remote[i] = make_float4(1.f, 2.f, 3.f, (float)i);
      }
    }
  }
  if (acc.x == 12345.f) local[0] = acc;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  const std::uint64_t bytes = 4ull << 30, nv = bytes / 16;
  float4* buf[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&buf[g], bytes));
    CK(cudaMemset(buf[g], 0, bytes));
  }
  cudaEvent_t e0[2], e1[2];
  for (int g = 0; g < 2; ++g) {
    cudaSetDevice(g);
    cudaEventCreate(&e0[g]);
    cudaEventCreate(&e1[g]);
  }
  const char* names[3] = {"read remote", "write remote", "read+write remote"};
  for (int both = 0; both < 2; ++both)
    for (int mode = 0; mode < 3; ++mode)
      for (int grid_mul : {2, 4, 8}) {
        for (int rep = 0; rep < 2; ++rep) {
          for (int g = 0; g < 1 + both; ++g) {
            cudaSetDevice(g);
            cudaEventRecord(e0[g]);
            k<<<148 * grid_mul, 256>>>(buf[g], buf[1 - g], nv, mode);
            cudaEventRecord(e1[g]);
          }
          for (int g = 0; g < 1 + both; ++g) {
            cudaSetDevice(g);
            CK(cudaEventSynchronize(e1[g]));
          }
        }
        float ms = 0;
        cudaSetDevice(0);
        cudaEventElapsedTime(&ms, e0[0], e1[0]);
        printf("%-20s %-14s grid=148x%d  GPU0: %.1f GB/s over NVLink\n", names[mode],
               both ? "(both GPUs)" : "(GPU0 only)", grid_mul, bytes / (ms / 1e3) / 1e9);
      }
  return 0;
}
