// tc_logit.cu -- the LogisticRegression local step (optimizer.hpp:75-146,
// 231-242) for fp32 peer state on the 5th-generation tensor cores.
//
// Batched over peers the step is two GEMMs:
//   margins  M = Theta . X^T   (N x S, K = D), epilogue c = -y / (1 + exp(y m))
//   gradient G = C . X         (N x D, K = S), epilogue theta -= gamma (G/S + l2 theta + n)
// The fp64 path (reference precision) keeps the SIMT kernels of sgd.cu: the
// reference sums every margin / gradient sequentially, which no tensor-core
// schedule reproduces.  The fp32 path promises fp32-level agreement (1e-6
// relative), so it runs here as 3xTF32: each operand is split a = hi + lo
// with hi, lo representable in tf32 and the product is accumulated as
// lo*hi + hi*lo + hi*hi in fp32 (the lo*lo term is below fp32 resolution).
//
// Kernel shape (one CTA = one 128 x 128 output tile, 128 threads, warp
// specialised):
//  * operands arrive pre-split (hi, lo fp32 arrays, K contiguous); warp 0
//    (one lane) streams 32-wide K slabs of A_hi, A_lo, B_hi, B_lo with TMA
//    (cp.async.bulk.tensor.2d, 128B swizzle: exactly the UMMA K-major
//    SWIZZLE_128B layout -- 8-row atoms of 128-byte rows, 16-byte chunk c of
//    row r at c ^ (r & 7)) into a 3-stage ring (full/empty mbarriers,
//    complete_tx byte counts);
//  * warp 1 (one lane) issues tcgen05.mma.cta_group::1.kind::tf32 (M = N =
//    128, K = 8 per instruction, 3 per K step) from shared-memory descriptors
//    into a 128-column fp32 accumulator in tensor memory; tcgen05.commit
//    hands each stage back to the producer and, after the last slab, the
//    accumulator to the epilogue;
//  * the epilogue reads the accumulator with tcgen05.ld (warp w owns TMEM
//    lanes 32w..32w+31 = tile rows) 32 columns at a time.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "philox.cuh"
#include "plane.cuh"

namespace mb200 {
namespace {

constexpr int kTcM = 128, kTcK = 32;  // tile rows; kTcK fp32 = one 128-byte row
constexpr int kTcThreads = 128;
constexpr int kTileBytes = kTcM * kTcK * 4;  // 16 KB per A tile
// stage: A_hi, A_lo (128 rows) + B_hi, B_lo (BN rows)
template <int BN>
__host__ __device__ constexpr int stage_bytes() { return 2 * kTileBytes + 2 * BN * kTcK * 4; }
// as many ring stages as fit (the K loop is TMA-latency bound): 3 of 64 KB for
// 128-wide tiles, 4 of 48 KB for 64-wide
template <int BN>
__host__ __device__ constexpr int tc_stages() {
  return (200 * 1024) / stage_bytes<BN>() > 4 ? 4 : (200 * 1024) / stage_bytes<BN>();
}
template <int BN>
__host__ __device__ constexpr std::size_t tc_smem() {
  return (std::size_t)tc_stages<BN>() * stage_bytes<BN>() + 1024 + 128;
}

__device__ __forceinline__ std::uint32_t su32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: start >> 4 in bits
// [0,14), LBO (unused for swizzled K-major) = 1, SBO = 1024 B (one 8-row atom)
// in bits [32,46), version 1 (sm100) at bit 46, layout type 2 (128B swizzle)
// in bits [61,64) (cute/arch/mma_sm100_desc.hpp SmemDescriptor).
__device__ __forceinline__ std::uint64_t sw128_desc(std::uint32_t saddr) {
  std::uint64_t d = (std::uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (std::uint64_t)1 << 16;
  d |= (std::uint64_t)(1024 >> 4) << 32;
  d |= (std::uint64_t)1 << 46;
  d |= (std::uint64_t)2 << 61;
  return d;
}

// Instruction descriptor kind::tf32 (InstrDescriptor): D f32 (bits 4-5 = 1),
// A, B tf32 (bits 7-9, 10-12 = 2), both K-major, N >> 3 at bit 17, M >> 4 at 24.
template <int BN>
__host__ __device__ constexpr std::uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((std::uint32_t)(BN >> 3) << 17) |
         ((std::uint32_t)(kTcM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(std::uint32_t tmem_d, std::uint64_t a, std::uint64_t b,
                                         std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_init1(std::uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
}

// Bounded wait: a lost arrival traps (an error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_bounded(std::uint64_t* bar, std::uint32_t parity) {
  const std::uint32_t a = su32(bar);
  for (long long it = 0;; ++it) {
    std::uint32_t done = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
    if (it > (1ll << 24)) __trap();
  }
}

__device__ __forceinline__ void tmem_ld32(std::uint32_t taddr, float (&v)[32]) {
  std::uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
}

// tf32 split of one fp32 value: hi = rna-rounded to tf32, lo = tf32(a - hi)
__device__ __forceinline__ void tf32_split(float a, float& hi, float& lo) {
  std::uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(a));
  hi = __uint_as_float(h);
  const float r = __fsub_rn(a, hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
  lo = __uint_as_float(l);
}

// Split a [rows x cols] matrix (row stride lds, double or float) into hi/lo
// fp32 arrays [rows x cols] (or, transposed, [cols x rows]).
template <typename S>
__global__ void split_kernel(const S* __restrict__ src, std::uint64_t rows, std::uint64_t cols,
                             std::uint64_t lds, int transpose, float* __restrict__ hi,
                             float* __restrict__ lo) {
  const std::uint64_t total = rows * cols;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t r = e / cols, c = e % cols;
    float h, l;
    tf32_split((float)src[r * lds + c], h, l);
    const std::uint64_t o = transpose ? c * rows + r : r * cols + c;
    hi[o] = h;
    lo[o] = l;
  }
}

struct TcArgs {
  const float *a_hi, *a_lo, *b_hi, *b_lo;  // [M x K], [N x K], K contiguous
  std::uint64_t M, N, K, lda, ldb;
  // epilogue 0: coefficients (margins GEMM)
  const double* ys;
  float *c_hi, *c_lo;  // [M x N] split coefficients
  // epilogue 1: gradient + update (gradient GEMM)
  float* theta;
  std::uint64_t ld_theta;
  const float* noise;  // host-drawn noise rows [M x N] (reference stream) or null
  double S, l2;
  float gamma;
  double coord_std;
  int philox;
  PhiloxKeys pk;
  std::uint64_t step;
  std::uint32_t* nonfinite;
  double* nsq_out;
};

template <int EPI, int BN>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_kernel(TcArgs a, const __grid_constant__ CUtensorMap tm_ah,
                   const __grid_constant__ CUtensorMap tm_al,
                   const __grid_constant__ CUtensorMap tm_bh,
                   const __grid_constant__ CUtensorMap tm_bl) {
  constexpr int kStage = stage_bytes<BN>();
  constexpr int kBTile = BN * kTcK * 4;
  constexpr int kTcStages = tc_stages<BN>();
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  // 1024-byte alignment of the operand tiles (the 128B-swizzle atom)
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<std::uintptr_t>(tc_smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + kTcStages * kStage);
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 2 * kTcStages + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const std::uint64_t m0 = (std::uint64_t)blockIdx.y * kTcM, n0 = (std::uint64_t)blockIdx.x * BN;

  if (tid == 0) {
    for (int s = 0; s < 2 * kTcStages + 1; ++s) mbar_init1(&bars[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const std::uint32_t tmem = *tmem_slot;

  const std::uint64_t nk = (a.K + kTcK - 1) / kTcK;
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + kTcStages;
  std::uint64_t* done = bars + 2 * kTcStages;
  if (warp == 0 && lane == 0) {
    // ===== TMA producer =====
    const std::uint64_t maps[4] = {reinterpret_cast<std::uint64_t>(&tm_ah),
                                   reinterpret_cast<std::uint64_t>(&tm_al),
                                   reinterpret_cast<std::uint64_t>(&tm_bh),
                                   reinterpret_cast<std::uint64_t>(&tm_bl)};
    const std::uint32_t toff[4] = {0u, (std::uint32_t)kTileBytes, 2u * kTileBytes,
                                   2u * kTileBytes + kBTile};
    for (std::uint64_t kb = 0; kb < nk; ++kb) {
      const int st = (int)(kb % kTcStages);
      if (kb >= (std::uint64_t)kTcStages)  // MMAs of slab kb - kTcStages freed this stage
        mbar_wait_bounded(&empty[st], (std::uint32_t)((kb / kTcStages - 1) & 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])),
                   "r"(kStage)
                   : "memory");
      const std::uint32_t base = su32(smem + st * kStage);
      const int k0 = (int)(kb * kTcK);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int r0 = (int)(t < 2 ? m0 : n0);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(base + toff[t]),
            "l"(maps[t]), "r"(k0), "r"(r0), "r"(su32(&full[st]))
            : "memory");
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ===== MMA issuer =====
    constexpr std::uint32_t idesc = idesc_tf32<BN>();
    for (std::uint64_t kb = 0; kb < nk; ++kb) {
      const int st = (int)(kb % kTcStages);
      mbar_wait_bounded(&full[st], (std::uint32_t)((kb / kTcStages) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const std::uint32_t sb = su32(smem + st * kStage);
#pragma unroll
      for (int kk = 0; kk < kTcK / 8; ++kk) {  // K = 8 tf32 (32 bytes) per MMA
        const std::uint32_t off = kk * 32;
        const std::uint64_t ah = sw128_desc(sb + off);
        const std::uint64_t al = sw128_desc(sb + kTileBytes + off);
        const std::uint64_t bh = sw128_desc(sb + 2 * kTileBytes + off);
        const std::uint64_t bl = sw128_desc(sb + 2 * kTileBytes + kBTile + off);
        mma_tf32(tmem, al, bh, idesc, (kb | kk) != 0);
        mma_tf32(tmem, ah, bl, idesc, 1);
        mma_tf32(tmem, ah, bh, idesc, 1);
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              su32(&empty[st]))
          : "memory");
    }
    // the last commit covers every MMA issued before it: the accumulator is final
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            su32(done))
        : "memory");
  }
  __syncwarp();
  if (nk) mbar_wait_bounded(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // Epilogue: thread (warp, lane) owns tile row 32 warp + lane (its TMEM lane),
  // 32 columns per TMEM load.  Global traffic goes through a per-warp 32 x 33
  // shared-memory transpose (the operand ring is idle now), so every global
  // access is a 128-byte row segment.
  float* tw = reinterpret_cast<float*>(smem) + warp * 3 * 32 * 33;  // 3 tiles per warp
  float* t0 = tw;
  float* t1 = tw + 32 * 33;
  float* t2 = tw + 2 * 32 * 33;
  const std::uint64_t row = m0 + warp * 32 + lane;
  const std::uint64_t rbase = m0 + warp * 32;
  double nsq = 0.0;
  bool bad = false;
  for (int cc = 0; cc < BN; cc += 32) {
    float acc[32];
    tmem_ld32(tmem + ((std::uint32_t)(warp * 32) << 16) + (std::uint32_t)cc, acc);
    if (nk == 0) {
#pragma unroll
      for (int q = 0; q < 32; ++q) acc[q] = 0.f;
    }
    const std::uint64_t col = n0 + cc + lane;  // this lane's column in the coalesced passes
    if constexpr (EPI == 0) {
      // c = -y / (1 + exp(y m))  (optimizer.hpp:126) in fp32 (this is the fp32
      // path), then the tf32 split; y of column cc + q
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const std::uint64_t cq = n0 + cc + q;
        const float y = cq < a.N ? (float)a.ys[cq] : 0.f;
        const float c = __fdiv_rn(-y, __fadd_rn(1.0f, expf(__fmul_rn(y, acc[q]))));
        float h, l;
        tf32_split(c, h, l);
        t0[lane * 33 + q] = h;
        t1[lane * 33 + q] = l;
      }
      __syncwarp();
      for (int r = 0; r < 32; ++r) {
        const std::uint64_t gr = rbase + r;
        if (gr < a.M && col < a.N) {
          a.c_hi[gr * a.N + col] = t0[r * 33 + lane];
          a.c_lo[gr * a.N + col] = t1[r * 33 + lane];
        }
      }
      __syncwarp();
    } else {
      // g = G / S + l2 theta (+ noise); theta -= gamma g  (optimizer.hpp:133-135,
      // 356-373): the same per-element arithmetic and Philox quads as
      // logit_grad_tiled.  theta rows in and out through the transpose tile.
      for (int r = 0; r < 32; ++r) {
        const std::uint64_t gr = rbase + r;
        t2[r * 33 + lane] = (gr < a.M && col < a.N) ? a.theta[gr * a.ld_theta + col] : 0.f;
      }
      __syncwarp();
      if (row < a.M) {
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const std::uint64_t j4 = n0 + cc + q4 * 4;
          if (j4 >= a.N) break;
          float z[4] = {0.f, 0.f, 0.f, 0.f};
          if (a.philox && !a.noise) philox_normals4(a.pk, a.step, row, j4 >> 2, z);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const std::uint64_t j = j4 + u;
            if (j >= a.N) break;
            float& th = t2[lane * 33 + q4 * 4 + u];
            const double g = __dadd_rn(__ddiv_rn((double)acc[q4 * 4 + u], a.S),
                                       __dmul_rn(a.l2, (double)th));
            float gt = (float)g;
            if (a.noise) {
              gt = __fadd_rn(gt, a.noise[row * a.N + j]);
            } else if (a.philox) {
              const float nj = noise_component(z[u], a.coord_std, (float*)nullptr);
              nsq += (double)nj * (double)nj;
              gt = __fadd_rn(gt, nj);
            }
            if (!isfinite(gt)) bad = true;
            th = __fsub_rn(th, __fmul_rn(a.gamma, gt));
          }
        }
      }
      __syncwarp();
      for (int r = 0; r < 32; ++r) {
        const std::uint64_t gr = rbase + r;
        if (gr < a.M && col < a.N) a.theta[gr * a.ld_theta + col] = t2[r * 33 + lane];
      }
      __syncwarp();
    }
  }
  if constexpr (EPI == 1) {
    if (bad) atomicOr(a.nonfinite, 1u);
    if (a.philox) {
      for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
      if (lane == 0) atomicAdd(a.nsq_out, nsq);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    MB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      throw CudaError("cuTensorMapEncodeTiled is not available from the driver");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D fp32 map over [rows x cols] (row stride ld elements): boxes of
// kTcK x 128 (one 128-byte row per tile row), 128B swizzle, zero fill.
CUtensorMap operand_map(const float* base, std::uint64_t rows, std::uint64_t cols,
                        std::uint64_t ld, std::uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)kTcK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(
      &m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

template <int EPI, int BN>
void launch_tc(const TcArgs& a, cudaStream_t s) {
  static int attr_dev = -1;
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    MB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<EPI, BN>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem<BN>()));
    attr_dev = dev;
  }
  const dim3 grid((unsigned)((a.N + BN - 1) / BN), (unsigned)((a.M + kTcM - 1) / kTcM));
  const CUtensorMap ah = operand_map(a.a_hi, a.M, a.K, a.lda, kTcM);
  const CUtensorMap al = operand_map(a.a_lo, a.M, a.K, a.lda, kTcM);
  const CUtensorMap bh = operand_map(a.b_hi, a.N, a.K, a.ldb, BN);
  const CUtensorMap bl = operand_map(a.b_lo, a.N, a.K, a.ldb, BN);
  tc_gemm_kernel<EPI, BN><<<grid, kTcThreads, tc_smem<BN>(), s>>>(a, ah, al, bh, bl);
  MB_LAUNCH_CHECK();
}

}  // namespace

bool logit_tc_enabled(std::uint64_t dim, std::uint64_t samples) {
  const char* e = std::getenv("MOSHPIT_LOGIT_TC");  // read per run (tests toggle it)
  const int mode = e ? std::atoi(e) : 1;
  return mode != 0 && dim % 4 == 0 && samples % 4 == 0 && dim > 0 && samples > 0;
}

// One-time operand preparation: X [S x D] (double) -> X_hi/X_lo [S x D] and
// X^T_hi/X^T_lo [D x S] (fp32 tf32 pairs).
void logit_tc_prepare(const double* xs, std::uint64_t S, std::uint64_t dim, float* x_hi,
                      float* x_lo, float* xt_hi, float* xt_lo, cudaStream_t s) {
  const unsigned g = (unsigned)std::min<std::uint64_t>((S * dim + 255) / 256, 148 * 32);
  split_kernel<double><<<g, 256, 0, s>>>(xs, S, dim, dim, 0, x_hi, x_lo);
  MB_LAUNCH_CHECK();
  split_kernel<double><<<g, 256, 0, s>>>(xs, S, dim, dim, 1, xt_hi, xt_lo);
  MB_LAUNCH_CHECK();
}

// The fp32 logistic local step of n peers (theta: n x ld floats) on the
// tensor cores.  Scratch: th_hi/th_lo [n x dim], c_hi/c_lo [n x S].
void logit_tc_step(float* theta, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                   std::uint64_t S, const float* x_hi, const float* x_lo, const float* xt_hi,
                   const float* xt_lo, const double* ys, double l2, float gamma,
                   const float* noise, double coord_std, int philox, std::uint64_t seed,
                   std::uint64_t step, std::uint32_t* nonfinite, double* nsq_out, float* th_hi,
                   float* th_lo, float* c_hi, float* c_lo, cudaStream_t s) {
  const unsigned g = (unsigned)std::min<std::uint64_t>((n * dim + 255) / 256, 148 * 32);
  split_kernel<float><<<g, 256, 0, s>>>(theta, n, dim, ld, 0, th_hi, th_lo);
  MB_LAUNCH_CHECK();
  TcArgs a{};
  a.a_hi = th_hi;
  a.a_lo = th_lo;
  a.b_hi = x_hi;
  a.b_lo = x_lo;
  a.M = n;
  a.N = S;
  a.K = dim;
  a.lda = dim;
  a.ldb = dim;
  a.ys = ys;
  a.c_hi = c_hi;
  a.c_lo = c_lo;
  launch_tc<0, 128>(a, s);
  TcArgs b{};
  b.a_hi = c_hi;
  b.a_lo = c_lo;
  b.b_hi = xt_hi;
  b.b_lo = xt_lo;
  b.M = n;
  b.N = dim;
  b.K = S;
  b.lda = S;
  b.ldb = S;
  b.theta = theta;
  b.ld_theta = ld;
  b.S = (double)S;
  b.noise = noise;
  b.l2 = l2;
  b.gamma = gamma;
  b.coord_std = coord_std;
  b.philox = philox;
  b.pk = philox_keys(seed);
  b.step = step;
  b.nonfinite = nonfinite;
  b.nsq_out = nsq_out;
  // 64-wide tiles: 128 output tiles for N = D = 1024 instead of 64 on 148 SMs
  // (MOSHPIT_TC_GRAD_BN=128 for the 128-wide form)
  const char* e = std::getenv("MOSHPIT_TC_GRAD_BN");
  if (e && std::atoi(e) == 128) launch_tc<1, 128>(b, s);
  else launch_tc<1, 64>(b, s);
}

}  // namespace mb200
