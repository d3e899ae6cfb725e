// dadd_chain.cu -- the floor of the EXACT diagnostics: one dependent fp64
// add chain per peer (core.hpp:118-122 sums j sequentially).  Measures, on
// one thread, cycles per element of (a) a register-only DADD chain and
// (b) the chain the EXACT kernel runs: a = a + sq[k] with sq[k] in shared
// memory (LDS + DADD).    nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>

__global__ void chain_reg(double* out, long long* cyc, int n, double x) {
  double a = 0.0, b = x;
  const long long t0 = clock64();
  for (int k = 0; k < n; ++k) a = __dadd_rn(a, b);
  const long long t1 = clock64();
  out[0] = a;
  cyc[0] = t1 - t0;
}

__global__ void chain_smem(double* out, long long* cyc, int n) {
  __shared__ double sq[512];
  for (int k = threadIdx.x; k < 512; k += blockDim.x) sq[k] = 1.0 / (k + 1);
  __syncthreads();
  if (threadIdx.x != 0) return;
  double a = 0.0;
  const long long t0 = clock64();
  for (int r = 0; r < n / 512; ++r) {
#pragma unroll 16
    for (int k = 0; k < 512; ++k) a = __dadd_rn(a, sq[k]);
  }
  const long long t1 = clock64();
  out[0] = a;
  cyc[0] = t1 - t0;
}

int main() {
  double* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&d_cyc, 8);
  const int n = 1 << 20;
  long long c = 0;
  chain_reg<<<1, 1>>>(d_out, d_cyc, n, 1e-9);
  chain_reg<<<1, 1>>>(d_out, d_cyc, n, 1e-9);
  cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"dadd_chain_cycles_per_add\": %.3f, ", (double)c / n);
  chain_smem<<<1, 32>>>(d_out, d_cyc, n);
  chain_smem<<<1, 32>>>(d_out, d_cyc, n);
  cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
  printf("\"lds_dadd_chain_cycles_per_element\": %.3f}\n", (double)c / n);
  return 0;
}
