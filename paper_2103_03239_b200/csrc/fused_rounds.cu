// fused_rounds.cu -- several Moshpit rounds (optionally preceded by the local
// SGD step) in ONE pass over the state: temporal blocking over column tiles
// (SURVEY 8d "run_rounds_fused", a separately reported mode; the per-round
// metric stays kernel 2's one read + one write per round).
//
// Coordinates are independent and the round tables (groups, voids) do not
// depend on the vectors, so a CTA can hold a column tile of ALL n peers in
// shared memory and apply R rounds to it before writing it back: 2 * n * D
// * sizeof(T) bytes of HBM traffic per pass instead of per round.  Each round
// is the reference butterfly_allreduce per active group (allreduce.hpp:
// 79-121): the pairwise tree of core.hpp:72-81 over the members in priority
// order, divided by the member count, written to every member; voided groups
// are not in the active list and keep their rows.  The optional step is
// kernel 3's (optimizer.hpp:356-373: separately rounded, the same Philox
// normals per (step, peer, quad)), so results are bit-identical to kernel 3
// + kernel 2 (tests/test_gpu_fused_rounds.py).
//
// Layout: a persistent CTA per SM (512 threads) keeps the R rounds' tables in
// shared memory (member rows, and (beg, count) of every active group) and two
// tile buffers of n rows x 4 16-byte vectors (rows XOR-swizzled), one per
// team of 256 threads: each team loads its tile with cp.async, steps it,
// averages it R times and stores it, synchronising on its own named barrier,
// so one team's load and barrier waits overlap the other's compute.  Round
// phase: a quad of lanes per (active group, vector), one tree leaf per lane
// (<= 4 sequential leaves of <= 8 members for n <= 32; the runtime tree
// beyond).
#include <algorithm>

#include "common.cuh"
#include "pairwise.cuh"
#include "philox.cuh"

namespace mb200 {
namespace {

#ifndef MB_FR_TV
#define MB_FR_TV 4
#endif
// 2 or 3 teams of 256 threads, each with its own tile: 3 when their tiles
// and the tables fit in shared memory (C2: 10 rounds in 21.3 ms with 3 teams
// vs 27.1 with 2; profiles/r02/fused_rounds.md)
constexpr int kFrTeamsMax = 3, kFrTeamThreads = 256;
constexpr int kFrThreads = kFrTeamsMax * kFrTeamThreads;
constexpr int kFrTV = MB_FR_TV;  // 16-byte vectors per row in a tile
static_assert(kFrTV == 1 || kFrTV == 2 || kFrTV == 4, "tile row = 1, 2 or 4 vectors");
constexpr std::size_t kFrSmemMax = 226 * 1024;  // 227 KB opt-in less the static reduction buffer

template <typename T>
struct FrVec;
template <>
struct FrVec<float> {
  using V = float4;
  static constexpr int W = 4;
};
template <>
struct FrVec<double> {
  using V = double2;
  static constexpr int W = 2;
};

template <typename T>
struct FrArgs {
  T* state;
  std::uint64_t ld_vec, nvec, n_tiles, dim;
  std::uint32_t n, R;
  std::uint32_t gcap;  // >= active groups of any round (<= min(n, M^(d-1)))
  const FusedRound* rounds;  // [R] device tables
  // optional local step before round 0 (kernel 3's prologue)
  const T* curv;
  const T* tgt;
  T gamma;
  double coord_std;
  std::uint64_t step_no;
  PhiloxKeys pk;
  std::uint32_t* nonfinite;
  double* noise_partial;
};

__device__ __forceinline__ void fr_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<std::uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ float fr_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double fr_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float fr_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double fr_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float fr_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double fr_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float fr_div(float a, std::uint32_t n) { return __fdiv_rn(a, (float)n); }
__device__ __forceinline__ double fr_div(double a, std::uint32_t n) {
  return __ddiv_rn(a, (double)n);
}
__device__ __forceinline__ float fr_fma0(float g, float acc) { return __fmaf_rn(g, 0.f, acc); }
__device__ __forceinline__ double fr_fma0(double g, double acc) { return __fma_rn(g, 0.0, acc); }

template <typename V>
__device__ __forceinline__ V fr_zero();
template <>
__device__ __forceinline__ float4 fr_zero<float4>() { return make_float4(0.f, 0.f, 0.f, 0.f); }
template <>
__device__ __forceinline__ double2 fr_zero<double2>() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ float4 fr_vadd(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ double2 fr_vadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ float4 fr_vdiv(float4 a, std::uint32_t n) {
  const float f = (float)n;
  return make_float4(__fdiv_rn(a.x, f), __fdiv_rn(a.y, f), __fdiv_rn(a.z, f), __fdiv_rn(a.w, f));
}
__device__ __forceinline__ double2 fr_vdiv(double2 a, std::uint32_t n) {
  const double f = (double)n;
  return make_double2(__ddiv_rn(a.x, f), __ddiv_rn(a.y, f));
}
__device__ __forceinline__ float4 fr_shfl_xor(unsigned mask, float4 v, int o) {
  return make_float4(__shfl_xor_sync(mask, v.x, o), __shfl_xor_sync(mask, v.y, o),
                     __shfl_xor_sync(mask, v.z, o), __shfl_xor_sync(mask, v.w, o));
}
__device__ __forceinline__ double2 fr_shfl_xor(unsigned mask, double2 v, int o) {
  return make_double2(__shfl_xor_sync(mask, v.x, o), __shfl_xor_sync(mask, v.y, o));
}

// Tile position of (row, vector): the kFrTV vectors of a row are XOR-swizzled
// by the row bits above those that pick its 16-byte slot in a 128-byte bank
// line, so the 8 lanes of an LDS.128 phase reading one vector index of 8
// random rows spread over 8 bank groups (4 vectors: row bits 1-2; 2: bit 2).
__device__ __forceinline__ std::uint32_t fr_pos(std::uint32_t row, std::uint32_t v) {
  constexpr int sh = kFrTV == 4 ? 1 : 2;
  return row * kFrTV + (v ^ ((row >> sh) & (std::uint32_t)(kFrTV - 1)));
}
__device__ __forceinline__ float4 fr_shfl(unsigned mask, float4 v, int src) {
  return make_float4(__shfl_sync(mask, v.x, src), __shfl_sync(mask, v.y, src),
                     __shfl_sync(mask, v.z, src), __shfl_sync(mask, v.w, src));
}
__device__ __forceinline__ double2 fr_shfl(unsigned mask, double2 v, int src) {
  return make_double2(__shfl_sync(mask, v.x, src), __shfl_sync(mask, v.y, src));
}

// The reference tree for n <= 32 as at most four sequential leaves of <= 8
// (n <= 8: one; n <= 16: split at floor(n/2); n <= 32: both halves split
// again, a half of <= 8 staying one leaf) joined L0 | L0+L1 | L0+(L1+L2) |
// (L0+L1)+(L2+L3) -- kernel 3's form (step_kernel.cu).
__device__ __forceinline__ int fr_leaves(std::uint32_t n, std::uint32_t* b) {
  if (n <= 8) {
    b[0] = 0; b[1] = n;
    return 1;
  }
  const std::uint32_t h = n / 2;
  if (n <= 16) {
    b[0] = 0; b[1] = h; b[2] = n;
    return 2;
  }
  const std::uint32_t n2 = n - h;
  if (h <= 8) {
    b[0] = 0; b[1] = h; b[2] = h + n2 / 2; b[3] = n;
    return 3;
  }
  b[0] = 0; b[1] = h / 2; b[2] = h; b[3] = h + n2 / 2; b[4] = n;
  return 4;
}

template <typename T, bool STEP, bool NOISY>
__global__ void __launch_bounds__(kFrThreads, 1)
    rounds_fused_kernel(const __grid_constant__ FrArgs<T> a) {
  using V = typename FrVec<T>::V;
  constexpr int W = FrVec<T>::W;
  constexpr int TC = kFrTV * W;  // columns per tile row
  extern __shared__ __align__(16) unsigned char fr_raw[];
  const std::uint32_t n = a.n, R = a.R;
  const int teams = (int)blockDim.x / kFrTeamThreads;
  V* const tiles = reinterpret_cast<V*>(fr_raw);  // [teams][n][kFrTV]
  std::uint32_t* const s_grp = reinterpret_cast<std::uint32_t*>(tiles + teams * n * kFrTV);  // [R][gcap]: beg << 16 | count
  std::uint32_t* const s_cnt = s_grp + (std::size_t)R * a.gcap;  // [R] active groups
  std::uint16_t* const s_mem = reinterpret_cast<std::uint16_t*>(s_cnt + R);  // [R][n] member rows
  const int tid = threadIdx.x;

  // the R rounds' tables, once per CTA
  for (std::uint32_t r = 0; r < R; ++r) {
    const FusedRound rt = a.rounds[r];
    const std::uint32_t A = rt.counts[1];
    if (A > a.gcap) __trap();  // more groups than the grid has lines: a caller bug
    for (std::uint32_t i = tid; i < n; i += blockDim.x)
      s_mem[r * n + i] = (std::uint16_t)rt.members[i];
    for (std::uint32_t i = tid; i < A; i += blockDim.x) {
      const std::uint32_t g = rt.act[i];
      const std::uint32_t beg = rt.goff[g];
      s_grp[r * a.gcap + i] = beg << 16 | (rt.goff[g + 1] - beg);
    }
    if (tid == 0) s_cnt[r] = A;
  }

  __syncthreads();  // the tables are in place

  // Two teams of 256 threads, each with its own tile buffer, named barrier
  // and tile sequence: while one team waits on its tile's loads or on a
  // round barrier, the other computes.
  const int team = tid / kFrTeamThreads, ttid = tid % kFrTeamThreads;
  auto team_sync = [&] {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(kFrTeamThreads) : "memory");
  };
  V* const gvec = reinterpret_cast<V*>(a.state);
  V* const tile = tiles + (std::size_t)team * n * kFrTV;
  __shared__ V s_ct[kFrTeamsMax][2][kFrTV];

  T chk = T(0);
  double nsq = 0.0;
  const std::uint64_t stride = (std::uint64_t)gridDim.x * teams;
  for (std::uint64_t t = (std::uint64_t)blockIdx.x * teams + team; t < a.n_tiles; t += stride) {
    const std::uint64_t v0 = t * kFrTV;
    for (std::uint32_t idx = ttid; idx < n * kFrTV; idx += kFrTeamThreads) {
      const std::uint32_t row = idx / kFrTV, v = idx % kFrTV;
      if (v0 + v < a.nvec)
        fr_cp16(tile + fr_pos(row, v), gvec + (std::uint64_t)row * a.ld_vec + v0 + v);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    team_sync();  // every thread's copies of this tile have landed

    if constexpr (STEP) {
      // kernel 3's step on every (row, vector): g = c (theta - t) [+ n_j],
      // theta' = theta - gamma g, separately rounded; the tile's curvature and
      // target vectors staged in shared memory once
      if (ttid < 2 * kFrTV) {
        const std::uint64_t cv = v0 + (ttid % kFrTV);
        const T* src = ttid < kFrTV ? a.curv : a.tgt;
        s_ct[team][ttid / kFrTV][ttid % kFrTV] =
            cv < a.nvec ? __ldg(reinterpret_cast<const V*>(src) + cv) : fr_zero<V>();
      }
      team_sync();
      for (std::uint32_t idx = ttid; idx < n * kFrTV; idx += kFrTeamThreads) {
        const std::uint32_t row = idx / kFrTV, v = idx % kFrTV;
        const std::uint64_t cv = v0 + v;
        if (cv >= a.nvec) continue;
        V e = tile[fr_pos(row, v)];
        const V c = s_ct[team][0][v];
        const V tg = s_ct[team][1][v];
        T* pe = reinterpret_cast<T*>(&e);
        const T* pc = reinterpret_cast<const T*>(&c);
        const T* pt = reinterpret_cast<const T*>(&tg);
        float z[4] = {0.f, 0.f, 0.f, 0.f};
        const std::uint64_t j0 = cv * W;
        if constexpr (NOISY) philox_normals4(a.pk, a.step_no, row, j0 / 4, z);
        const T cst = (T)a.coord_std;
        T q = T(0);
#pragma unroll
        for (int w = 0; w < W; ++w) {
          if (j0 + w >= a.dim) break;
          T g = fr_mul(pc[w], fr_sub(pe[w], pt[w]));
          if constexpr (NOISY) {
            const T nj = fr_mul(cst, (T)z[(j0 + w) & 3]);
            nsq_add(q, nj);
            g = fr_add(g, nj);
          }
          chk = fr_fma0(g, chk);
          pe[w] = fr_sub(pe[w], fr_mul(a.gamma, g));
        }
        if constexpr (NOISY) nsq += (double)q;
        tile[fr_pos(row, v)] = e;
      }
      team_sync();
    }

    // R rounds on the tile: 4 x kFrTV lanes per active group, lane (l, v)
    // summing leaf l of the group's tree (<= 8 members, loads independent of
    // the adds) over 16-byte vector v.  The kFrTV lanes of one leaf read the
    // same member row, i.e. one contiguous row of the tile per leaf step (a
    // phase of 8 lanes touches 2 rows instead of 8 random (row, vector) slots:
    // fewer shared-memory bank conflicts).  The lanes of a vector swap their
    // leaf sums with shuffles, every lane joins them in the tree's order
    // (identical ops, identical bits) and writes the mean to its own leaf's
    // members.  Groups of more than 32: the leaf-0 lanes walk the runtime tree.
    constexpr std::uint32_t GL = 4 * kFrTV;  // lanes per group
    for (std::uint32_t r = 0; r < R; ++r) {
      const std::uint32_t A = s_cnt[r];
      const std::uint16_t* mem = s_mem + (std::size_t)r * n;
      const std::uint32_t leaf = ((std::uint32_t)tid / kFrTV) & 3u;
      const int gbase = tid & (int)(32 - GL);
      const unsigned gmask = (GL == 32 ? 0xffffffffu : ((1u << GL) - 1u)) << gbase;
      for (std::uint32_t item = ttid; item < A * GL; item += kFrTeamThreads) {
        const std::uint32_t gi = item / GL, v = item % kFrTV;
        const std::uint32_t pk = s_grp[(std::size_t)r * a.gcap + gi];
        const std::uint32_t beg = pk >> 16, cnt = pk & 0xffffu;
        const std::uint16_t* m = mem + beg;
        if (cnt <= 32) {
          std::uint32_t b[5] = {0, 0, 0, 0, 0};
          const int nl = fr_leaves(cnt, b);
          std::uint32_t lb = 0, le = 0;
#pragma unroll
          for (int l = 0; l < 4; ++l)
            if ((std::uint32_t)l == leaf && l < nl) {
              lb = b[l];
              le = b[l + 1];
            }
          std::uint32_t pos[8];
          V sl = fr_zero<V>();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            pos[k] = lb + k < le ? fr_pos(m[lb + k], v) : 0u;
            if (lb + k < le) sl = fr_vadd(sl, tile[pos[k]]);
          }
          // leaf j's sum for vector v lives on lane gbase + j * kFrTV + v
          const int src = gbase + (int)v;
          const V L0 = fr_shfl(gmask, sl, src);
          V sum = L0;
          if (nl >= 2) {
            const V L1 = fr_shfl(gmask, sl, src + kFrTV);
            if (nl == 2) {
              sum = fr_vadd(L0, L1);
            } else {
              const V L2 = fr_shfl(gmask, sl, src + 2 * kFrTV);
              if (nl == 3) {
                sum = fr_vadd(L0, fr_vadd(L1, L2));
              } else {
                const V L3 = fr_shfl(gmask, sl, src + 3 * kFrTV);
                sum = fr_vadd(fr_vadd(L0, L1), fr_vadd(L2, L3));
              }
            }
          }
          const V mean = fr_vdiv(sum, cnt);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (lb + k < le) tile[pos[k]] = mean;
        } else if (leaf == 0) {
          auto ld = [&](std::uint32_t k) { return tile[fr_pos(m[k], v)]; };
          const V sum = pairwise_rt<V>(ld, cnt, [](V x, V y) { return fr_vadd(x, y); },
                                       fr_zero<V>());
          const V mean = fr_vdiv(sum, cnt);
          for (std::uint32_t k = 0; k < cnt; ++k) tile[fr_pos(m[k], v)] = mean;
        }
      }
      team_sync();
    }

    for (std::uint32_t idx = ttid; idx < n * kFrTV; idx += kFrTeamThreads) {
      const std::uint32_t row = idx / kFrTV, v = idx % kFrTV;
      if (v0 + v < a.nvec) gvec[(std::uint64_t)row * a.ld_vec + v0 + v] = tile[fr_pos(row, v)];
    }
    team_sync();  // the buffer is refilled by the team's next tile
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  if constexpr (STEP) {
    if (chk != T(0)) atomicOr(a.nonfinite, 1u);
    if constexpr (NOISY) {
      __shared__ double red[kFrThreads / 32];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
      if ((tid & 31) == 0) red[tid >> 5] = nsq;
      __syncthreads();
      if (tid == 0 && a.noise_partial) {
        double s = 0.0;
        for (int i = 0; i < (int)blockDim.x / 32; ++i) s += red[i];
        a.noise_partial[blockIdx.x] = s;
      }
    }
  }
}

std::size_t fr_smem(int teams, std::uint32_t n, std::uint32_t gcap, std::uint32_t R) {
  return (std::size_t)teams * n * kFrTV * 16 + (std::size_t)R * ((std::size_t)n * 2 + (std::size_t)gcap * 4 + 4) + 16;
}

template <typename T, bool STEP, bool NOISY>
void launch_fr(const FrArgs<T>& a, int teams, std::size_t smem, cudaStream_t s) {
  static thread_local int attr_dev = -1;
  int dev = 0;
  MB_CUDA(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    MB_CUDA(cudaFuncSetAttribute(rounds_fused_kernel<T, STEP, NOISY>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFrSmemMax));
    attr_dev = dev;
  }
  int sms = 0;
  MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = (unsigned)std::min<std::uint64_t>((std::uint64_t)sms, a.n_tiles);
  rounds_fused_kernel<T, STEP, NOISY><<<grid, teams * kFrTeamThreads, smem, s>>>(a);
  MB_LAUNCH_CHECK();
}

}  // namespace

std::uint32_t fused_rounds_max(std::uint64_t n, std::uint64_t gcap) {
  if (n == 0 || n > 4096) return 0;
  gcap = std::min(gcap, n);
  const std::size_t tiles = (std::size_t)2 * n * kFrTV * 16;  // two teams at least
  if (tiles + 64 >= kFrSmemMax) return 0;
  const std::size_t per = (std::size_t)n * 2 + (std::size_t)gcap * 4 + 4;
  return (std::uint32_t)std::min<std::size_t>((kFrSmemMax - tiles - 16) / per, 64);
}

template <typename T>
void launch_rounds_fused(T* state, std::uint64_t ld, std::uint64_t dim, std::uint32_t n,
                         std::uint32_t gcap, const FusedRound* rounds_dev, std::uint32_t R,
                         const StepPrologue<T>* step, cudaStream_t s) {
  constexpr int W = FrVec<T>::W;
  if (dim == 0 || n == 0 || (R == 0 && !step)) return;
  gcap = std::min(gcap, n);
  if (R > fused_rounds_max(n, gcap)) throw std::invalid_argument("fused rounds: tables exceed shared memory");
  FrArgs<T> a{};
  a.state = state;
  a.ld_vec = ld / W;
  a.nvec = (dim + W - 1) / W;
  a.n_tiles = (a.nvec + kFrTV - 1) / kFrTV;
  a.dim = dim;
  a.n = n;
  a.R = R;
  a.gcap = gcap;
  a.rounds = rounds_dev;
  const int teams = fr_smem(3, n, gcap, R) <= kFrSmemMax ? 3 : 2;
  const std::size_t smem = fr_smem(teams, n, gcap, R);
  if (step) {
    a.curv = step->curv;
    a.tgt = step->tgt;
    a.gamma = step->gamma;
    a.coord_std = step->coord_std;
    a.step_no = step->step_no;
    a.pk = philox_keys(step->seed);
    a.nonfinite = step->nonfinite;
    a.noise_partial = step->noise_partial;
    if (step->philox) launch_fr<T, true, true>(a, teams, smem, s);
    else launch_fr<T, true, false>(a, teams, smem, s);
  } else {
    launch_fr<T, false, false>(a, teams, smem, s);
  }
}

template void launch_rounds_fused<float>(float*, std::uint64_t, std::uint64_t, std::uint32_t, std::uint32_t,
                                         const FusedRound*, std::uint32_t,
                                         const StepPrologue<float>*, cudaStream_t);
template void launch_rounds_fused<double>(double*, std::uint64_t, std::uint64_t, std::uint32_t, std::uint32_t,
                                          const FusedRound*, std::uint32_t,
                                          const StepPrologue<double>*, cudaStream_t);

}  // namespace mb200
