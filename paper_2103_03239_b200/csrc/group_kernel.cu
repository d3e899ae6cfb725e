// group_kernel.cu -- Kernel 1: integer-exact group formation.
//
// Replaces matchmaking::form_groups_uncontested (matchmaking.hpp:300-323) +
// the per-member bookkeeping of run_moshpit (protocols.hpp:143-170):
//   cohorts = peers with equal GroupKey, in ascending lexicographic key order
//             (std::map order), each sorted by Priority{timestamp, id}
//             (matchmaking.hpp:20-25), split every `cap` members;
//   rank    = position inside the group (allreduce.hpp:92-93, chunk index);
//   void    = OR of the failure mask over the group (allreduce.hpp:95-102);
//   next key= next_group_key(key, rank) for EVERY member (protocols.hpp:168).
// One CTA of 1024 threads: a bitonic sort of peer indices under the
// (key, timestamp, id, index) order (for <= 1024 peers with small keys: in
// registers over a composite 64-bit key, shuffles for strides < 32), then
// segmented scans.  The peer count of
// a Moshpit trial is <= M^d (a few thousand at the north-star configs), so
// the whole table fits in shared memory and the kernel costs microseconds
// next to the HBM-bound group mean; larger n spills the sort to global memory
// (same code, same result).
#include <type_traits>

#include "common.cuh"
#include "pairwise.cuh"

namespace mb200 {
namespace {

constexpr int kThreads = 1024;

__host__ __device__ inline std::uint32_t pow2_ceil(std::uint32_t n) {
  std::uint32_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

struct PackedView {
  const std::uint64_t* key;
  __device__ int cmp(std::uint32_t a, std::uint32_t b) const {
    const std::uint64_t ka = key[a], kb = key[b];
    return ka < kb ? -1 : (ka > kb ? 1 : 0);
  }
};

struct DigitView {
  const std::uint32_t* key;
  std::uint32_t klen;
  __device__ int cmp(std::uint32_t a, std::uint32_t b) const {
    for (std::uint32_t k = 0; k < klen; ++k) {
      const std::uint32_t ka = key[(std::uint64_t)a * klen + k];
      const std::uint32_t kb = key[(std::uint64_t)b * klen + k];
      if (ka != kb) return ka < kb ? -1 : 1;
    }
    return 0;
  }
};

// Block-wide exclusive scan of one value per thread.  op: 0 = sum, 1 = max.
template <int OP>
__device__ std::uint32_t block_exclusive_scan(std::uint32_t v,
                                              std::uint32_t identity,
                                              std::uint32_t* total) {
  __shared__ std::uint32_t warp_tot[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = OP == 0 ? x + y : (x > y ? x : y);
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    std::uint32_t w = lane < kThreads / 32 ? warp_tot[lane] : identity;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = OP == 0 ? w + y : (w > y ? w : y);
    }
    warp_tot[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const std::uint32_t before_warp = warp == 0 ? identity : warp_tot[warp - 1];
  std::uint32_t excl_in_warp = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) excl_in_warp = identity;
  std::uint32_t r;
  if (OP == 0)
    r = before_warp + excl_in_warp;
  else
    r = before_warp > excl_in_warp ? before_warp : excl_in_warp;
  if (total) *total = warp_tot[kThreads / 32 - 1];
  __syncthreads();
  return r;
}

// Kernel 2 for narrow vectors inside kernel 1's CTA: one thread per
// (active group, column), the reference pairwise tree (core.hpp:72-81) over
// the members in group order, divided by the member count (core.hpp:91-106),
// written back to every member.  Items touch disjoint (row, column) sets.
template <typename T>
__device__ void fused_group_means(const GroupArgs& a, std::uint32_t n_act) {
  T* x = static_cast<T*>(a.fuse_x) + (a.batch ? blockIdx.x * a.fuse_stride : 0);
  const std::uint64_t dim = a.fuse_dim, ld = a.fuse_ld, items = (std::uint64_t)n_act * dim;
  for (std::uint64_t it = threadIdx.x; it < items; it += kThreads) {
    const std::uint32_t g = a.act[it / dim];
    const std::uint64_t j = it % dim;
    const std::uint32_t beg = a.goff[g], cnt = a.goff[g + 1] - beg;
    const std::uint32_t* mem = a.members + beg;
    auto ld_fn = [&](std::uint32_t k) -> T { return x[(std::uint64_t)mem[k] * ld + j]; };
    T m;
    if constexpr (std::is_same_v<T, double>) {
      const double s = pairwise_rt<double>(ld_fn, cnt, [](double u, double v) { return __dadd_rn(u, v); }, 0.0);
      m = __ddiv_rn(s, (double)cnt);
    } else {
      const float s = pairwise_rt<float>(ld_fn, cnt, [](float u, float v) { return __fadd_rn(u, v); }, 0.0f);
      m = __fdiv_rn(s, (float)cnt);
    }
    for (std::uint32_t k = 0; k < cnt; ++k) x[(std::uint64_t)mem[k] * ld + j] = m;
  }
}

template <class View>
__global__ void __launch_bounds__(kThreads, 1)
    form_groups_kernel(GroupArgs a, View view, int use_smem) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (a.batch) {  // CTA b handles trial b of a batch
    const std::uint64_t t = blockIdx.x, n = a.n;
    std::uint64_t np = 1;
    while (np < n) np <<= 1;
    a.keys += t * n;
    a.ts += t * n;
    if (a.failed) a.failed += t * n;
    a.members += t * n;
    a.goff += t * (n + 1);
    a.gvoid += t * n;
    if (a.rank) a.rank += t * n;
    if (a.act) a.act += t * n;
    if (a.counts) a.counts += t * 4;
    a.totals = nullptr;
    a.sidx += t * np;
    a.scs += t * n;
    a.sgi += t * n;
    if constexpr (std::is_same_v<View, PackedView>) view.key = a.keys;
  }
  const std::uint32_t n = a.n;
  const std::uint32_t np = pow2_ceil(n);
  const std::uint32_t tid = threadIdx.x;

  std::uint32_t* idx = use_smem ? reinterpret_cast<std::uint32_t*>(smem) : a.sidx;
  const std::uint64_t* ts = a.ts;
  if constexpr (std::is_same_v<View, PackedView>) {
    // Packed mode: stage keys and timestamps next to the index array.
    if (use_smem) {
      std::uint64_t* skey = reinterpret_cast<std::uint64_t*>(smem + np * 4 + ((np * 4) & 4));
      std::uint64_t* sts = skey + n;
      for (std::uint32_t i = tid; i < n; i += kThreads) {
        skey[i] = view.key[i];
        sts[i] = a.ts[i];
      }
      view.key = skey;
      ts = sts;
    }
  }
  // Fast path (the engine's common case: n <= 1024 peers, packed keys below
  // 2^16 - 1, ids == indices): one element per thread in REGISTERS, sorted by
  // the composite (key << 48 | timestamp, index) -- the same strict order as
  // the general comparator below -- with bitonic exchanges through warp
  // shuffles for strides < 32 and shared memory (2 barriers) above.
  bool fast = false;
  if constexpr (std::is_same_v<View, PackedView>) {
    const bool big = tid < n && (view.key[tid] >= 0xFFFFull || (ts[tid] >> 48) != 0);
    fast = n <= (std::uint32_t)kThreads && a.ids == nullptr && !__syncthreads_or(big);
  }
  if (fast) {
    std::uint64_t c = ~0ull;
    std::uint32_t id = 0xFFFFFFFFu;  // padding sorts last
    if (tid < n) {
      std::uint64_t kv = 0;
      if constexpr (std::is_same_v<View, PackedView>) kv = view.key[tid];
      c = (kv << 48) | (ts[tid] & 0xFFFFFFFFFFFFull);
      id = tid;
    }
    std::uint64_t* xc = reinterpret_cast<std::uint64_t*>(smem + np * 4 + ((np * 4) & 4)) + 2 * n;
    std::uint32_t* xi = reinterpret_cast<std::uint32_t*>(xc + np);
    for (std::uint32_t k = 2; k <= np; k <<= 1) {
      for (std::uint32_t j = k >> 1; j > 0; j >>= 1) {
        std::uint64_t oc;
        std::uint32_t oi;
        if (j < 32) {
          oc = __shfl_xor_sync(0xffffffffu, c, j);
          oi = __shfl_xor_sync(0xffffffffu, id, j);
        } else {
          if (tid < np) {
            xc[tid] = c;
            xi[tid] = id;
          }
          __syncthreads();
          if (tid < np) {
            oc = xc[tid ^ j];
            oi = xi[tid ^ j];
          }
          __syncthreads();
        }
        if (tid < np) {
          const bool other_less = oc < c || (oc == c && oi < id);
          const bool lower = (tid & j) == 0, up = (tid & k) == 0;
          // ascending blocks: the lower position keeps the min
          if (lower == up ? other_less : !other_less) {
            c = oc;
            id = oi;
          }
        }
      }
    }
    if (tid < np) idx[tid] = id;
    __syncthreads();
  } else {
  for (std::uint32_t i = tid; i < np; i += kThreads) idx[i] = i;
  __syncthreads();

  // Strict weak order: key, Priority{timestamp, id}, then input index.
  // Indices >= n are padding and compare greatest.
  auto less = [&](std::uint32_t x, std::uint32_t y) -> bool {
    if (y >= n) return x < n;
    if (x >= n) return false;
    const int c = view.cmp(x, y);
    if (c != 0) return c < 0;
    if (ts[x] != ts[y]) return ts[x] < ts[y];
    const std::uint32_t ix = a.ids ? a.ids[x] : x, iy = a.ids ? a.ids[y] : y;
    if (ix != iy) return ix < iy;
    return x < y;
  };

  for (std::uint32_t k = 2; k <= np; k <<= 1) {
    for (std::uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (std::uint32_t i = tid; i < np; i += kThreads) {
        const std::uint32_t p = i ^ j;
        if (p > i) {
          const std::uint32_t x = idx[i], y = idx[p];
          const bool up = (i & k) == 0;
          if (up ? less(y, x) : less(x, y)) {
            idx[i] = y;
            idx[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  }

  // Each thread owns a contiguous run of sorted positions.
  const std::uint32_t per = (n + kThreads - 1) / kThreads;
  const std::uint32_t lo = tid * per < n ? tid * per : n;
  const std::uint32_t hi = lo + per < n ? lo + per : n;

  // Pass 1: cohort starts (max-scan of "key changes here" positions).
  std::uint32_t cur = 0, have = 0;
  for (std::uint32_t p = lo; p < hi; ++p) {
    if (p == 0 || view.cmp(idx[p], idx[p - 1]) != 0) {
      cur = p;
      have = 1;
    }
  }
  const std::uint32_t carry_in =
      block_exclusive_scan<1>(have ? cur + 1 : 0u, 0u, nullptr);
  // Pass 2: cohort start per position and group-start counts.
  cur = carry_in ? carry_in - 1 : 0;
  std::uint32_t starts = 0;
  for (std::uint32_t p = lo; p < hi; ++p) {
    if (p == 0 || view.cmp(idx[p], idx[p - 1]) != 0) cur = p;
    a.scs[p] = cur;
    starts += ((p - cur) % a.cap) == 0;
  }
  std::uint32_t n_groups = 0;
  const std::uint32_t gbase = block_exclusive_scan<0>(starts, 0u, &n_groups);
  // Pass 3: group ids, member table, offsets, ranks, next keys.
  std::uint32_t g = gbase;
  for (std::uint32_t p = lo; p < hi; ++p) {
    const std::uint32_t cs = a.scs[p];
    const std::uint32_t r = (p - cs) % a.cap;
    if (r == 0) a.goff[g++] = p;
    a.sgi[p] = g - 1;
    const std::uint32_t who = idx[p];
    a.members[p] = a.ids ? a.ids[who] : who;
    if (a.rank) a.rank[who] = r;
  }
  if (tid == 0) {
    a.goff[n_groups] = n;
    if (a.counts) a.counts[0] = n_groups;
  }
  if (a.advance_keys) {
    // Keys are read from the staged copy (view) and written to global.
    for (std::uint32_t p = lo; p < hi; ++p) {
      const std::uint32_t who = idx[p];
      const std::uint32_t r = (p - a.scs[p]) % a.cap;
      if (a.klen_zero) {
        a.keys[who] = 0;
      } else {
        std::uint64_t oldk;
        if constexpr (std::is_same_v<View, PackedView>) {
          oldk = view.key[who];
        } else {
          oldk = 0;
        }
        a.keys[who] = (oldk % a.pow_drop) * a.M + r;
      }
    }
  }
  // Void flags: any failed member voids the group.
  for (std::uint32_t q = tid; q < n_groups; q += kThreads) a.gvoid[q] = 0;
  __syncthreads();
  if (a.failed) {
    for (std::uint32_t p = lo; p < hi; ++p)
      if (a.failed[idx[p]]) a.gvoid[a.sgi[p]] = 1;
  }
  __syncthreads();
  // Compact the non-voided groups into the work list of kernel 2.
  const std::uint32_t gper = (n_groups + kThreads - 1) / kThreads;
  const std::uint32_t glo = tid * gper < n_groups ? tid * gper : n_groups;
  const std::uint32_t ghi = glo + gper < n_groups ? glo + gper : n_groups;
  std::uint32_t mine = 0, rows = 0;
  for (std::uint32_t q = glo; q < ghi; ++q)
    if (!a.gvoid[q]) {
      ++mine;
      rows += a.goff[q + 1] - a.goff[q];
    }
  std::uint32_t n_act = 0, n_rows = 0;
  std::uint32_t pos = block_exclusive_scan<0>(mine, 0u, &n_act);
  (void)block_exclusive_scan<0>(rows, 0u, &n_rows);
  if (a.act)
    for (std::uint32_t q = glo; q < ghi; ++q)
      if (!a.gvoid[q]) a.act[pos++] = q;
  if (tid == 0) {
    if (a.counts) {
      a.counts[1] = n_act;
      a.counts[2] = n_rows;
    }
    if (a.totals) a.totals[0] += n_rows;
  }
  if (a.fuse_x && a.act) {
    __syncthreads();  // act / goff / members of this CTA are written
    if (a.fuse_f64) fused_group_means<double>(a, n_act);
    else fused_group_means<float>(a, n_act);
  }
}

__global__ void initial_keys_kernel(const std::uint64_t* cells,
                                    std::uint64_t* keys, std::uint64_t n,
                                    std::uint32_t M, std::uint32_t d) {
  const std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // matchmaking.hpp:46-59: key index j-1 = digit j of the cell; index 0 is
  // the most significant position of the packed key (Horner over j).
  std::uint64_t rest = cells[i] / M, key = 0;
  for (std::uint32_t j = 1; j < d; ++j) {
    key = key * M + rest % M;
    rest /= M;
  }
  keys[i] = key;
}

}  // namespace

std::size_t group_smem_bytes(std::uint32_t n, bool packed) {
  const std::size_t np = pow2_ceil(n);
  std::size_t b = np * 4;
  b += b & 4;
  if (packed) b += std::size_t(n) * 16;
  if (packed && n <= (std::uint32_t)kThreads) b += np * 12;  // fast-path exchange buffers
  return b;
}

void launch_form_groups(const GroupArgs& a, bool packed, cudaStream_t s) {
  if (a.n == 0) return;
  static constexpr std::size_t kMaxSmem = 200 * 1024;
  const std::size_t smem = group_smem_bytes(a.n, packed);
  const int use_smem = smem <= kMaxSmem;
  const std::size_t dyn = use_smem ? smem : 0;
  if (packed) {
    auto* k = form_groups_kernel<PackedView>;
    if (dyn > 48 * 1024)
      MB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)dyn));
    k<<<a.batch ? a.batch : 1, kThreads, dyn, s>>>(a, PackedView{a.keys}, use_smem);
  } else {
    auto* k = form_groups_kernel<DigitView>;
    if (dyn > 48 * 1024)
      MB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)dyn));
    k<<<1, kThreads, dyn, s>>>(a, DigitView{a.digit_keys, a.dklen}, use_smem);
  }
  MB_LAUNCH_CHECK();
}

void launch_initial_keys(const std::uint64_t* cells, std::uint64_t* keys,
                         std::uint64_t n, std::uint32_t M, std::uint32_t d,
                         cudaStream_t s) {
  if (n == 0) return;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  initial_keys_kernel<<<blocks, 256, 0, s>>>(cells, keys, n, M, d);
  MB_LAUNCH_CHECK();
}

}  // namespace mb200
