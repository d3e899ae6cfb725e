// shard.cu -- peer-sharded multi-GPU Moshpit rounds (north-star
// layout).
//
// Placement.  Peers sit cell-major: global row = current grid cell, GPU =
// row / R with R = M^d / G, i.e. the most significant grid digit x_{d-1} is
// split across the G GPUs.  Keys evolve by shift-append of ranks
// (matchmaking.hpp:62-71); relabelling the active coordinate to the member's
// rank after every round makes round t a set of grid lines along axis
// (t-1) mod d, so rounds on axes 0..d-2 are GPU-local and only
// axis d-1 crosses GPUs.  Locally, a peer's row is an indirection (loc[p]):
// voided groups keep their rows and nothing moves.
//
// Cross round (axis d-1).  The tree order spans GPUs, so no partial sums can
// be shipped: GPU g owns coordinate chunk g of every group and evaluates the
// reference tree over the members' raw chunk-g vectors, loading remote rows
// straight from peer HBM over NVLink (CUDA IPC mappings) and storing the mean
// into every member row, remote ones included -- one fused kernel, the
// transfer overlapped with the arithmetic tile by tile.  Members of a
// non-voided group whose rank moves them to another GPU inherit, on that GPU,
// the row of a member that left it (same group), so the mean lands in place
// and only voided groups move data (staged pull, then write).
//
// The integer plane (draws, kernel 1, placement) is replicated on every rank:
// every rank computes identical tables, so no metadata is exchanged.  Ranks
// synchronise with a P2P flag barrier kernel (no host round-trip).
//
// Hosting.  A process hosts `nhost` consecutive ranks (their pools on its
// GPU; the data-plane launches loop over them); processes exchange CUDA IPC
// handles once and barrier among themselves.  nhost = 1: one rank per GPU
// (production); nhost = world: every rank on one GPU (the 1-GPU emulation
// harness); in between: e.g. world 8 on 4 GPUs with 2 ranks per process,
// which exercises the 8-way cross round over real NVLink without ever running
// two spinning kernels of one GPU against each other.
//
// Slab pipeline (slabs = S > 1).  Coordinates are independent, so the
// columns are cut into S slabs that run one round apart on S streams: at
// every step one slab is in a cross round (NVLink-bound) while the others
// are in local rounds (HBM-bound) -- the two rooflines overlap instead of
// adding up.  Each round's tables are computed once (control stream) into a
// ring of S+1 slots; slab k replays round r's slot at step r+k; flush()
// completes the lagging slabs.  Bit-identical to S = 1 (tests).
#include <algorithm>
#include <cstdlib>
#include <memory>

#include "plane.cuh"

namespace mb200 {
namespace {

constexpr int kMaxWorld = 8;

struct PlaceArgs {
  std::uint32_t n = 0, world = 1, Mg = 1;
  std::uint64_t R = 0;
  int cross = 0;
  const std::uint32_t* members = nullptr;
  const std::uint32_t* goff = nullptr;
  const std::uint32_t* counts = nullptr;
  const std::uint8_t* gvoid = nullptr;
  std::uint32_t* loc = nullptr;         // [n] global row per peer (in/out)
  std::uint32_t* rows_local = nullptr;  // [n] local row per member position
  std::uint32_t* act_local = nullptr;   // [world][n]
  std::uint32_t* cnt_local = nullptr;   // [world][4]: [1] n_act, [2] rows
  std::uint32_t* src_row = nullptr;     // [n] by position (cross)
  std::uint32_t* dst_row = nullptr;     // [n] by position (cross)
  std::uint32_t* act_cross = nullptr;   // [n]
  std::uint32_t* cnt_cross = nullptr;   // [4]: [1] n_act, [2] rows
  std::uint32_t* moves = nullptr;       // [world][R][2] (src, dst), grouped by dst GPU
  std::uint32_t* n_moves = nullptr;     // [world]
  std::uint32_t* err = nullptr;         // [1]
  std::uint32_t* goff_out = nullptr;    // [n+1] copy of goff for the data plane (slot)
  unsigned long long* totals = nullptr; // [0] cross active groups, [1] cross rounds,
                                        // [2+h] local active rows on GPU h,
                                        // [2+kMaxWorld+h] voided rows moved to GPU h
};

// Replicated bookkeeping for one round (one CTA, one thread per group).
__global__ void __launch_bounds__(1024) place_kernel(PlaceArgs a) {
  const std::uint32_t ng = a.counts[0];
  if (threadIdx.x < a.world * 4) a.cnt_local[threadIdx.x] = 0;
  if (threadIdx.x < 4) a.cnt_cross[threadIdx.x] = 0;
  if (threadIdx.x < a.world) a.n_moves[threadIdx.x] = 0;
  if (threadIdx.x == 0 && a.cross) a.totals[1] += 1;
  for (std::uint32_t g = threadIdx.x; g <= ng; g += blockDim.x) a.goff_out[g] = a.goff[g];
  __syncthreads();
  for (std::uint32_t g = threadIdx.x; g < ng; g += blockDim.x) {
    const std::uint32_t b = a.goff[g], e = a.goff[g + 1];
    const bool voided = a.gvoid[g] != 0;
    if (!a.cross) {
      const std::uint32_t owner = (std::uint32_t)(a.loc[a.members[b]] / a.R);
      for (std::uint32_t pos = b; pos < e; ++pos) {
        const std::uint32_t r = a.loc[a.members[pos]];
        if (r / a.R != owner) atomicOr(a.err, 1u);  // a local round must be GPU-local
        a.rows_local[pos] = (std::uint32_t)(r % a.R);
      }
      if (!voided) {
        const std::uint32_t k = atomicAdd(&a.cnt_local[owner * 4 + 1], 1u);
        a.act_local[owner * a.n + k] = g;
        atomicAdd(&a.cnt_local[owner * 4 + 2], e - b);
        atomicAdd(&a.totals[2 + owner], (unsigned long long)(e - b));
      }
      continue;
    }
    // cross round: stayers keep their row; arrivals on GPU h take, in
    // position order, the rows of this group's members leaving h.
    for (std::uint32_t pos = b; pos < e; ++pos) {
      const std::uint32_t src = a.loc[a.members[pos]];
      const std::uint32_t og = (std::uint32_t)(src / a.R), nw = (pos - b) / a.Mg;
      a.src_row[pos] = src;
      a.dst_row[pos] = og == nw ? src : 0xffffffffu;
    }
    for (std::uint32_t h = 0; h < a.world; ++h) {
      std::uint32_t li = b;
      for (std::uint32_t pos = b; pos < e; ++pos) {
        const std::uint32_t og = (std::uint32_t)(a.src_row[pos] / a.R), nw = (pos - b) / a.Mg;
        if (nw != h || og == h) continue;  // not an arrival on h
        while (li < e && !((std::uint32_t)(a.src_row[li] / a.R) == h && (li - b) / a.Mg != h)) ++li;
        if (li == e) {
          atomicOr(a.err, 2u);  // unbalanced line: sharded mode needs a full grid
          break;
        }
        a.dst_row[pos] = a.src_row[li++];
      }
    }
    for (std::uint32_t pos = b; pos < e; ++pos) {
      a.loc[a.members[pos]] = a.dst_row[pos];
      if (voided && a.dst_row[pos] != a.src_row[pos]) {
        const std::uint32_t h = (std::uint32_t)(a.dst_row[pos] / a.R);
        const std::uint32_t k = atomicAdd(&a.n_moves[h], 1u);
        atomicAdd(&a.totals[2 + kMaxWorld + h], 1ull);
        a.moves[((std::uint64_t)h * a.R + k) * 2] = a.src_row[pos];
        a.moves[((std::uint64_t)h * a.R + k) * 2 + 1] = a.dst_row[pos];
      }
    }
    if (!voided) {
      const std::uint32_t k = atomicAdd(&a.cnt_cross[1], 1u);
      a.act_cross[k] = g;
      atomicAdd(&a.cnt_cross[2], e - b);
      atomicAdd(&a.totals[0], 1ull);
    }
  }
}

__global__ void init_loc_kernel(const std::uint64_t* cells, std::uint32_t* loc, std::uint64_t n) {
  const std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (i < n) loc[i] = (std::uint32_t)cells[i];
}

template <typename T>
struct V16s;
template <>
struct V16s<float> {
  using type = float4;
};
template <>
struct V16s<double> {
  using type = double2;
};
__device__ __forceinline__ float4 sadd(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ double2 sadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ float4 sdiv(float4 a, std::uint32_t n) {
  const float f = (float)n;
  return make_float4(__fdiv_rn(a.x, f), __fdiv_rn(a.y, f), __fdiv_rn(a.z, f), __fdiv_rn(a.w, f));
}
__device__ __forceinline__ double2 sdiv(double2 a, std::uint32_t n) {
  const double f = (double)n;
  return make_double2(__ddiv_rn(a.x, f), __ddiv_rn(a.y, f));
}
__device__ __forceinline__ float4 szero(float4*) { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ double2 szero(double2*) { return make_double2(0.0, 0.0); }

template <int N, int B, typename V>
__device__ __forceinline__ V stree(const V (&x)[32]) {
  if constexpr (N <= 8) {
    V s = szero((V*)nullptr);
#pragma unroll
    for (int i = 0; i < N; ++i) s = sadd(s, x[B + i]);
    return s;
  } else {
    constexpr int H = N / 2;
    return sadd(stree<H, B>(x), stree<N - H, B + H>(x));
  }
}

constexpr int kCrossThreads = 128;

template <typename T>
struct CrossArgs {
  T* pools[kMaxWorld];
  std::uint64_t ld_vec = 0, R = 0;
  std::uint64_t c0 = 0, c1 = 0, n_tiles = 0;
  std::uint64_t vb = 0, ve = 0;  // the slab's column range (16-byte vectors)
  std::uint32_t me = 0, world = 1;
  const std::uint32_t* goff = nullptr;
  const std::uint32_t* src_row = nullptr;
  const std::uint32_t* dst_row = nullptr;
  const std::uint32_t* act = nullptr;
  const std::uint32_t* cnt = nullptr;
};

template <int N, typename V>
__device__ __forceinline__ void cross_fixed(V* const* src, V* const* dst, std::uint64_t col) {
  V x[32];
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = __ldcs(src[k] + col);
  const V m = sdiv(stree<N, 0>(x), (std::uint32_t)N);
#pragma unroll
  for (int k = 0; k < N; ++k)
    if (dst[k]) __stcs(dst[k] + col, m);
}

// Fused cross-GPU round: this GPU's coordinate chunk of every active group,
// member rows read from (and the mean written to) local or peer HBM.
template <typename T>
__global__ void __launch_bounds__(kCrossThreads, 3) cross_mean_kernel(CrossArgs<T> a) {
  using V = typename V16s<T>::type;
  __shared__ V* s_src[32];
  __shared__ V* s_dst[32];
  const std::uint32_t n_act = a.cnt[1];
  const std::uint64_t n_items = (std::uint64_t)n_act * a.n_tiles;
  std::uint32_t cached = 0xffffffffu, cnt = 0;
  for (std::uint64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
    const std::uint32_t g = a.act[w / a.n_tiles];
    if (g != cached) {
      __syncthreads();
      const std::uint32_t beg = a.goff[g];
      cnt = a.goff[g + 1] - beg;
      if (threadIdx.x < cnt) {
        const std::uint32_t s = a.src_row[beg + threadIdx.x], d = a.dst_row[beg + threadIdx.x];
        const std::uint32_t dg = (std::uint32_t)(d / a.R);
        // Pull-only NVLink traffic: the mean of this GPU's chunk goes to its
        // LOCAL member rows only; other GPUs pull it in phase B
        // (shard_pull_kernel).  Mixing remote loads and remote stores in one
        // kernel costs ~2x NVLink throughput (profiles/r01/p2p_probe.txt).
        const bool store = dg == a.me;
        s_src[threadIdx.x] = reinterpret_cast<V*>(a.pools[s / a.R]) + (s % a.R) * a.ld_vec;
        s_dst[threadIdx.x] =
            store ? reinterpret_cast<V*>(a.pools[dg]) + (d % a.R) * a.ld_vec : nullptr;
      }
      cached = g;
      __syncthreads();
    }
    const std::uint64_t col = a.c0 + (w % a.n_tiles) * kCrossThreads + threadIdx.x;
    if (col >= a.c1) continue;
    switch (cnt) {
#define MB_XCASE(N)                       \
  case N:                                 \
    cross_fixed<N, V>(s_src, s_dst, col); \
    break;
      MB_XCASE(1) MB_XCASE(2) MB_XCASE(3) MB_XCASE(4) MB_XCASE(5) MB_XCASE(6) MB_XCASE(7)
      MB_XCASE(8) MB_XCASE(9) MB_XCASE(10) MB_XCASE(11) MB_XCASE(12) MB_XCASE(13)
      MB_XCASE(14) MB_XCASE(15) MB_XCASE(16) MB_XCASE(17) MB_XCASE(18) MB_XCASE(19)
      MB_XCASE(20) MB_XCASE(21) MB_XCASE(22) MB_XCASE(23) MB_XCASE(24) MB_XCASE(25)
      MB_XCASE(26) MB_XCASE(27) MB_XCASE(28) MB_XCASE(29) MB_XCASE(30) MB_XCASE(31)
      MB_XCASE(32)
#undef MB_XCASE
      default: break;
    }
  }
}

// Phase B of the cross round (after a barrier): for every active group, pull
// each foreign coordinate chunk c once from GPU c's first member row of the
// group (in group order) -- a remote READ -- and write it into this GPU's
// member rows of the group (local writes).  Every GPU derives the same rows
// from the replicated tables, so no metadata travels.
// Voided groups' row moves riding in the cross-round launches as extra work
// items (interleaved 1:1 with the group items while both last): phase 0
// pulls the rows that leave their GPU into staging (partial_sum_kernel),
// phase 1 writes them into their new rows (shard_pull_kernel).
struct MoveItems {
  const std::uint32_t* moves = nullptr;    // [world][R][2] (src, dst) by dst GPU
  const std::uint32_t* n_moves = nullptr;  // [world]
  void* staging = nullptr;                 // this rank's staging block
};

// Item w of a launch with n_grp group items and n_mov move items.
__device__ __forceinline__ bool pick_item(std::uint64_t w, std::uint64_t n_grp,
                                          std::uint64_t n_mov, std::uint64_t& i) {
  const std::uint64_t n_both = 2 * (n_grp < n_mov ? n_grp : n_mov);
  if (w < n_both) {
    i = w >> 1;
    return w & 1;
  }
  i = w - n_both / 2;
  return n_mov > n_grp;
}

constexpr int kPullU = 2;  // 16-byte vectors per thread and item (loads in flight)

// Phase B of the cross round (after a barrier): for every active group, pull
// each foreign coordinate chunk c once from GPU c's first member row of the
// group (in group order) -- a remote READ -- and write it into this GPU's
// member rows of the group (local writes).  Every GPU derives the same rows
// from the replicated tables, so no metadata travels.  With `mv`, the
// voided rows staged in phase 0 are written to their new rows in the same
// launch.
template <typename T>
__global__ void __launch_bounds__(kCrossThreads)
    shard_pull_kernel(CrossArgs<T> a, MoveItems mv) {
  using V = typename V16s<T>::type;
  __shared__ V* s_rows[32];
  __shared__ const V* s_rep[kMaxWorld];
  __shared__ std::uint32_t s_n;
  const std::uint32_t world = a.world;
  const std::uint64_t W = a.ve - a.vb;
  constexpr std::uint64_t kSpan = (std::uint64_t)kPullU * kCrossThreads;
  const std::uint64_t tiles = (W + kSpan - 1) / kSpan;
  const std::uint64_t n_grp = (std::uint64_t)a.cnt[1] * tiles;
  const std::uint64_t n_mov = mv.moves ? (std::uint64_t)mv.n_moves[a.me] * tiles : 0;
  std::uint32_t cached = 0xffffffffu;
  // contiguous runs of items per CTA: the group (and its member table) stays
  // the same for many consecutive items
  const std::uint64_t run = (n_grp + n_mov + gridDim.x - 1) / gridDim.x;
  const std::uint64_t w_end = min((std::uint64_t)(blockIdx.x + 1) * run, n_grp + n_mov);
  for (std::uint64_t w = blockIdx.x * run; w < w_end; ++w) {
    std::uint64_t i;
    if (pick_item(w, n_grp, n_mov, i)) {
      const std::uint64_t mk = i / tiles;
      const std::uint32_t dst = mv.moves[((std::uint64_t)a.me * a.R + mk) * 2 + 1];
      V* to = reinterpret_cast<V*>(a.pools[dst / a.R]) + (dst % a.R) * a.ld_vec;
      const V* from = reinterpret_cast<const V*>(mv.staging) + mk * a.ld_vec;
      V v[kPullU];
#pragma unroll
      for (int u = 0; u < kPullU; ++u) {
        const std::uint64_t rel = (i % tiles) * kSpan + u * kCrossThreads + threadIdx.x;
        if (rel < W) v[u] = __ldcs(from + a.vb + rel);
      }
#pragma unroll
      for (int u = 0; u < kPullU; ++u) {
        const std::uint64_t rel = (i % tiles) * kSpan + u * kCrossThreads + threadIdx.x;
        if (rel < W) __stcs(to + a.vb + rel, v[u]);
      }
      continue;
    }
    const std::uint32_t g = a.act[i / tiles];
    if (g != cached) {
      __syncthreads();
      if (threadIdx.x < 32) {  // warp 0: one lane per member position
        const std::uint32_t lane = threadIdx.x, beg = a.goff[g], n = a.goff[g + 1] - beg;
        const std::uint32_t d = lane < n ? a.dst_row[beg + lane] : 0u;
        const std::uint32_t h = lane < n ? (std::uint32_t)(d / a.R) : 0xffffffffu;
        V* row = reinterpret_cast<V*>(a.pools[lane < n ? h : 0]) + (d % a.R) * a.ld_vec;
        const unsigned mine = __ballot_sync(0xffffffffu, h == a.me);
        if (h == a.me) s_rows[__popc(mine & ((1u << lane) - 1u))] = row;
        for (std::uint32_t q = 0; q < world; ++q) {  // first row (position order) on GPU q
          const unsigned on = __ballot_sync(0xffffffffu, h == q);
          if (on && lane == (std::uint32_t)(__ffs(on) - 1)) s_rep[q] = row;
          if (!on && lane == 0) s_rep[q] = nullptr;
        }
        if (lane == 0) s_n = __popc(mine);
      }
      cached = g;
      __syncthreads();
    }
    V v[kPullU];
    bool ok[kPullU];
#pragma unroll
    for (int u = 0; u < kPullU; ++u) {
      const std::uint64_t rel = (i % tiles) * kSpan + u * kCrossThreads + threadIdx.x;
      const std::uint64_t col = a.vb + rel;
      ok[u] = rel < W && !(col >= a.c0 && col < a.c1);
      if (!ok[u]) continue;
      // owner of this column: chunk c covers [vb + W*c/world, vb + W*(c+1)/world)
      std::uint32_t c = (std::uint32_t)((rel * world) / W);
      while (c + 1 < world && (W * (c + 1)) / world <= rel) ++c;
      while (c > 0 && (W * c) / world > rel) --c;
      v[u] = *(s_rep[c] + col);
    }
    const std::uint32_t n = s_n;
    for (std::uint32_t k = 0; k < n; ++k) {
#pragma unroll
      for (int u = 0; u < kPullU; ++u)
        if (ok[u]) s_rows[k][a.vb + (i % tiles) * kSpan + u * kCrossThreads + threadIdx.x] = v[u];
    }
  }
}

// ---------------------------------------------------------------------------
// Partial-sum cross round (MOSHPIT_CROSS_PARTIAL).  The reference tree spans
// GPUs, so the exact round ships every remote member's raw chunk: per GPU
// (M - Mg) / world rows' worth of NVLink ingress per group.  This mode sums
// each GPU's own members first and ships one partial row per GPU and group:
//   phase 0 (local)  GPU h: P_h = its members' rows summed in position order
//                    (sequentially, in T), stored IN PLACE into its first
//                    member row p_h (a member row: it gets the mean anyway);
//   phase A (pull)   GPU r, coordinate chunk r: m = (P_0 + ... + P_{w-1}) / n
//                    in fp64 (the w partials pulled over NVLink in rank
//                    order), rounded to T, stored into its member rows;
//   phase B          unchanged (shard_pull_kernel): the foreign chunk means
//                    pulled once per group.
// NVLink ingress per GPU and group: 2 (w-1)/w rows instead of
// ((M - Mg) + (w-1)) / w.  The summation order is no longer the reference's
// ("within 1e-6 relative in fp32" where the order is not
// matched); deterministic (fixed order), and group formation, failures and
// placement are unchanged (replicated integer plane).  p_h is the first
// member of the group on GPU h in position order by SOURCE row, which is
// also one of its destination rows there (the row set of a group on a GPU
// does not change in a cross round), so phase A's stores cover it.
//
// The voided groups' row moves (phase 0: remote rows pulled into staging,
// NVLink-bound) ride in the same launch as extra work items (MoveItems), so
// the partial sums (HBM-bound) and the pulls overlap instead of adding up;
// both need the peers' rows final, hence the barrier before this launch.

template <typename T>
__global__ void __launch_bounds__(kCrossThreads)
    partial_sum_kernel(CrossArgs<T> a, MoveItems mv) {
  using V = typename V16s<T>::type;
  __shared__ const V* s_src[32];
  __shared__ std::uint32_t s_n;
  const std::uint64_t n_grp = (std::uint64_t)a.cnt[1] * a.n_tiles;
  const std::uint64_t n_mov = mv.moves ? (std::uint64_t)mv.n_moves[a.me] * a.n_tiles : 0;
  const std::uint64_t n_items = n_grp + n_mov;
  V* const pool = reinterpret_cast<V*>(a.pools[a.me]);
  std::uint32_t cached = 0xffffffffu, k = 0;
  const std::uint64_t run = (n_items + gridDim.x - 1) / gridDim.x;  // contiguous runs
  const std::uint64_t w_end = min((std::uint64_t)(blockIdx.x + 1) * run, n_items);
  for (std::uint64_t w = blockIdx.x * run; w < w_end; ++w) {
    std::uint64_t i;
    if (pick_item(w, n_grp, n_mov, i)) {
      const std::uint64_t mk = i / a.n_tiles;
      const std::uint64_t col = a.vb + (i % a.n_tiles) * kCrossThreads + threadIdx.x;
      if (col >= a.ve) continue;
      const std::uint32_t src = mv.moves[((std::uint64_t)a.me * a.R + mk) * 2];
      const V* from = reinterpret_cast<const V*>(a.pools[src / a.R]) + (src % a.R) * a.ld_vec;
      reinterpret_cast<V*>(mv.staging)[mk * a.ld_vec + col] = __ldcs(from + col);
      continue;
    }
    const std::uint64_t w2 = i;
    const std::uint32_t g = a.act[w2 / a.n_tiles];
    if (g != cached) {
      __syncthreads();
      if (threadIdx.x < 32) {  // warp 0: one lane per member position
        const std::uint32_t lane = threadIdx.x, beg = a.goff[g], n = a.goff[g + 1] - beg;
        const std::uint32_t sr = lane < n ? a.src_row[beg + lane] : 0u;
        const bool here = lane < n && sr / a.R == a.me;
        const unsigned mine = __ballot_sync(0xffffffffu, here);
        if (here) s_src[__popc(mine & ((1u << lane) - 1u))] = pool + (sr % a.R) * a.ld_vec;
        if (lane == 0) s_n = __popc(mine);
      }
      cached = g;
      __syncthreads();
      k = s_n;
    }
    const std::uint64_t rel = (w2 % a.n_tiles) * kCrossThreads + threadIdx.x;
    const std::uint64_t col = a.vb + rel;
    if (col >= a.ve || k == 0) continue;
    V acc = szero((V*)nullptr);
    for (std::uint32_t i = 0; i < k; i += 8) {
      V x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i + u < k) x[u] = __ldcs(s_src[i + u] + col);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i + u < k) acc = sadd(acc, x[u]);
    }
    const_cast<V*>(s_src[0])[col] = acc;
  }
}

__device__ __forceinline__ void dacc(double (&s)[4], float4 v) {
  s[0] = __dadd_rn(s[0], (double)v.x);
  s[1] = __dadd_rn(s[1], (double)v.y);
  s[2] = __dadd_rn(s[2], (double)v.z);
  s[3] = __dadd_rn(s[3], (double)v.w);
}
__device__ __forceinline__ void dacc(double (&s)[4], double2 v) {
  s[0] = __dadd_rn(s[0], v.x);
  s[1] = __dadd_rn(s[1], v.y);
}
__device__ __forceinline__ float4 dmean(const double (&s)[4], double n, float4*) {
  return make_float4((float)__ddiv_rn(s[0], n), (float)__ddiv_rn(s[1], n),
                     (float)__ddiv_rn(s[2], n), (float)__ddiv_rn(s[3], n));
}
__device__ __forceinline__ double2 dmean(const double (&s)[4], double n, double2*) {
  return make_double2(__ddiv_rn(s[0], n), __ddiv_rn(s[1], n));
}

// NW: the world size this instance is unrolled for (its partial loads sit in
// registers), kMaxWorld for any other world.
template <typename T, int NW>
__global__ void __launch_bounds__(kCrossThreads)
    partial_combine_kernel(CrossArgs<T> a) {
  using V = typename V16s<T>::type;
  __shared__ const V* s_part[kMaxWorld];
  __shared__ V* s_dst[32];
  __shared__ std::uint32_t s_nd, s_cnt;
  const std::uint32_t world = a.world;
  const std::uint64_t n_items = (std::uint64_t)a.cnt[1] * a.n_tiles;
  std::uint32_t cached = 0xffffffffu, nd = 0;
  double cntd = 1.0;
  const std::uint64_t run = (n_items + gridDim.x - 1) / gridDim.x;  // contiguous runs
  const std::uint64_t w_end = min((std::uint64_t)(blockIdx.x + 1) * run, n_items);
  for (std::uint64_t w = blockIdx.x * run; w < w_end; ++w) {
    const std::uint32_t g = a.act[w / a.n_tiles];
    if (g != cached) {
      __syncthreads();
      if (threadIdx.x < 32) {  // warp 0: one lane per member position
        const std::uint32_t lane = threadIdx.x, beg = a.goff[g], n = a.goff[g + 1] - beg;
        const std::uint32_t sr = lane < n ? a.src_row[beg + lane] : 0u;
        const std::uint32_t d = lane < n ? a.dst_row[beg + lane] : 0u;
        const std::uint32_t h = lane < n ? (std::uint32_t)(sr / a.R) : 0xffffffffu;
        const bool here = lane < n && d / a.R == a.me;
        const unsigned mine = __ballot_sync(0xffffffffu, here);
        if (here)
          s_dst[__popc(mine & ((1u << lane) - 1u))] =
              reinterpret_cast<V*>(a.pools[a.me]) + (d % a.R) * a.ld_vec;
        for (std::uint32_t q = 0; q < world; ++q) {  // partial row: first source row on GPU q
          const unsigned on = __ballot_sync(0xffffffffu, h == q);
          if (on && lane == (std::uint32_t)(__ffs(on) - 1))
            s_part[q] = reinterpret_cast<const V*>(a.pools[q]) + (sr % a.R) * a.ld_vec;
          if (!on && lane == 0) s_part[q] = nullptr;
        }
        if (lane == 0) {
          s_nd = __popc(mine);
          s_cnt = n;
        }
      }
      cached = g;
      __syncthreads();
      nd = s_nd;
      cntd = (double)s_cnt;
    }
    // kPullU vectors per thread: the remote partial loads of both in flight
    const std::uint64_t col0 = a.c0 + (w % a.n_tiles) * (kPullU * kCrossThreads) + threadIdx.x;
    V x[kPullU][NW];
#pragma unroll
    for (int u = 0; u < kPullU; ++u) {
      const std::uint64_t col = col0 + u * kCrossThreads;
#pragma unroll
      for (std::uint32_t h = 0; h < (std::uint32_t)NW; ++h)
        if (col < a.c1 && h < world && s_part[h]) x[u][h] = __ldcg(s_part[h] + col);
    }
    V m[kPullU];
#pragma unroll
    for (int u = 0; u < kPullU; ++u) {
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (std::uint32_t h = 0; h < (std::uint32_t)NW; ++h)
        if (h < world && s_part[h]) dacc(s, x[u][h]);
      m[u] = dmean(s, cntd, (V*)nullptr);
    }
    for (std::uint32_t q = 0; q < nd; ++q) {
#pragma unroll
      for (int u = 0; u < kPullU; ++u)
        if (col0 + u * kCrossThreads < a.c1) __stcs(s_dst[q] + col0 + u * kCrossThreads, m[u]);
    }
  }
}

// Copy-engine cross round (MOSHPIT_CROSS_CE=1).  SM loads from peer HBM top
// out at ~660 GB/s of NVLink ingress per GPU, one large copy-engine pull
// reaches ~760 GB/s (profiles/ce_probe.cu, profiles/r01/ce_probe.txt).  In
// the round itself the staged form measured no faster (C5-valid on 2 GPUs:
// phase A 115 vs 114 ms, phase B slower without the fused fan-out), so the
// SM-pull kernels stay the default; this path is kept, tested, for the
// comparison.  Phase A
// stages the raw chunk-g vectors of each group's REMOTE members into local
// HBM with peer copies (one async copy per member chunk on two copy streams,
// double-buffered by batches of groups) and this kernel evaluates the same
// tree from local memory: member k reads its local row, or staging slot
// (group-in-batch * nrem + k-th remote member) when it lives on another GPU.
template <typename T>
__global__ void __launch_bounds__(kCrossThreads, 3)
    cross_staged_kernel(CrossArgs<T> a, const T* stage, std::uint32_t gb, std::uint32_t ge,
                        std::uint32_t nrem) {
  using V = typename V16s<T>::type;
  __shared__ const V* s_src[32];
  __shared__ V* s_dst[32];
  const std::uint64_t cvec = a.c1 - a.c0;
  const std::uint64_t n_items = (std::uint64_t)(ge - gb) * a.n_tiles;
  std::uint32_t cached = 0xffffffffu, cnt = 0;
  for (std::uint64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
    const std::uint32_t gi = gb + (std::uint32_t)(w / a.n_tiles);
    const std::uint32_t g = a.act[gi];
    if (g != cached) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const std::uint32_t beg = a.goff[g];
        cnt = a.goff[g + 1] - beg;
        std::uint32_t slot = 0;
        for (std::uint32_t k = 0; k < cnt; ++k) {
          const std::uint32_t sr = a.src_row[beg + k], d = a.dst_row[beg + k];
          // row-relative pointers: element col of member k is at s_src[k][col - c0]
          if (sr / a.R == a.me)
            s_src[k] = reinterpret_cast<const V*>(a.pools[a.me]) + (sr % a.R) * a.ld_vec + a.c0;
          else
            s_src[k] = reinterpret_cast<const V*>(stage) +
                       ((std::uint64_t)(gi - gb) * nrem + slot++) * cvec;
          const std::uint32_t dg = (std::uint32_t)(d / a.R);
          s_dst[k] = dg == a.me ? reinterpret_cast<V*>(a.pools[dg]) + (d % a.R) * a.ld_vec + a.c0
                                : nullptr;
        }
      }
      cached = g;
      __syncthreads();
      cnt = a.goff[g + 1] - a.goff[g];
    }
    const std::uint64_t rel = (w % a.n_tiles) * kCrossThreads + threadIdx.x;
    if (rel >= cvec) continue;
    switch (cnt) {
#define MB_SCASE(N)                                          \
  case N:                                                    \
    cross_fixed<N, V>((V* const*)s_src, s_dst, rel);         \
    break;
      MB_SCASE(1) MB_SCASE(2) MB_SCASE(3) MB_SCASE(4) MB_SCASE(5) MB_SCASE(6) MB_SCASE(7)
      MB_SCASE(8) MB_SCASE(9) MB_SCASE(10) MB_SCASE(11) MB_SCASE(12) MB_SCASE(13)
      MB_SCASE(14) MB_SCASE(15) MB_SCASE(16) MB_SCASE(17) MB_SCASE(18) MB_SCASE(19)
      MB_SCASE(20) MB_SCASE(21) MB_SCASE(22) MB_SCASE(23) MB_SCASE(24) MB_SCASE(25)
      MB_SCASE(26) MB_SCASE(27) MB_SCASE(28) MB_SCASE(29) MB_SCASE(30) MB_SCASE(31)
      MB_SCASE(32)
#undef MB_SCASE
      default: break;
    }
  }
}

// Phase B of the copy-engine round: the foreign chunk means were copied (by
// the copy engines) into each group's FIRST local member row; fan them out to
// the group's other local member rows (local HBM only; nothing for Mg = 1).
template <typename T>
__global__ void __launch_bounds__(kCrossThreads)
    local_fanout_kernel(CrossArgs<T> a, std::uint64_t nvec) {
  using V = typename V16s<T>::type;
  __shared__ V* s_rows[32];
  __shared__ std::uint32_t s_n;
  const std::uint64_t n_items = (std::uint64_t)a.cnt[1] * a.n_tiles;
  std::uint32_t cached = 0xffffffffu;
  for (std::uint64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
    const std::uint32_t g = a.act[w / a.n_tiles];
    if (g != cached) {
      __syncthreads();
      if (threadIdx.x == 0) {
        std::uint32_t k = 0;
        for (std::uint32_t pos = a.goff[g]; pos < a.goff[g + 1]; ++pos) {
          const std::uint32_t d = a.dst_row[pos];
          if (d / a.R == a.me)
            s_rows[k++] = reinterpret_cast<V*>(a.pools[a.me]) + (d % a.R) * a.ld_vec;
        }
        s_n = k;
      }
      cached = g;
      __syncthreads();
    }
    const std::uint64_t col = (w % a.n_tiles) * kCrossThreads + threadIdx.x;
    if (col >= nvec || (col >= a.c0 && col < a.c1)) continue;
    const V v = s_rows[0][col];
    for (std::uint32_t k = 1; k < s_n; ++k) s_rows[k][col] = v;
  }
}

// Voided cross groups: rows whose owner GPU changes are pulled into staging
// (phase 0), then written to their new rows after a barrier (phase 1).
template <typename T>
__global__ void move_rows_kernel(T* const* pools, const std::uint32_t* moves,
                                 const std::uint32_t* n_moves, std::uint32_t me, std::uint64_t R,
                                 std::uint64_t ld_vec, std::uint64_t vb, std::uint64_t ve,
                                 T* staging, int phase) {
  using V = typename V16s<T>::type;
  const std::uint32_t cnt = n_moves[me];
  const std::uint64_t W = ve - vb;
  const std::uint64_t total = (std::uint64_t)cnt * W;
  V* st = reinterpret_cast<V*>(staging);
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t k = e / W, c = vb + e % W;
    const std::uint32_t* mv = moves + ((std::uint64_t)me * R + k) * 2;
    if (phase == 0) {
      const std::uint32_t s = mv[0];
      const V* src = reinterpret_cast<const V*>(pools[s / R]) + (s % R) * ld_vec;
      st[k * ld_vec + c] = src[c];
    } else {
      const std::uint32_t d = mv[1];
      V* dst = reinterpret_cast<V*>(pools[d / R]) + (d % R) * ld_vec;
      dst[c] = st[k * ld_vec + c];
    }
  }
}

// P2P flag barrier: each rank publishes `epoch` into every peer's flag slot,
// then waits for all peers' slots to reach it.  Bounded spin -> __trap()
// (an error, never a hang).
// Flags are [slab][process]: one row per slab stream (their barriers
// interleave), one slot per writing process.
__global__ void peer_barrier_kernel(unsigned long long* my_flags, unsigned long long* const* peer_flags,
                                    std::uint32_t me, std::uint32_t world, unsigned long long epoch,
                                    std::uint32_t row) {
  if (threadIdx.x != 0) return;
  my_flags += (std::uint64_t)row * kMaxWorld;
  __threadfence_system();
  for (std::uint32_t h = 0; h < world; ++h) {
    if (h == me) continue;
    unsigned long long* f = peer_flags[h] + (std::uint64_t)row * kMaxWorld + me;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
  }
  const long long t0 = clock64();
  for (std::uint32_t h = 0; h < world; ++h) {
    if (h == me) continue;
    unsigned long long v = 0;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flags + h) : "memory");
      if (v >= epoch) break;
      if (clock64() - t0 > 40000000000ll) __trap();  // ~20 s at 1.96 GHz
    }
  }
  __threadfence_system();
}

template <typename T>
__global__ void shard_fill_kernel(T* pool, const std::uint32_t* loc, std::uint64_t n,
                                  std::uint64_t dim, std::uint64_t ld, std::uint64_t R,
                                  std::uint32_t me, std::uint64_t seed) {
  const std::uint64_t total = n * dim;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t p = e / dim, j = e % dim;
    const std::uint32_t r = loc[p];
    if (r / R != me) continue;
    std::uint64_t z = (seed ^ (p << 32) ^ j) + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    pool[(r % R) * ld + j] = (T)((double)(z >> 40) * 0x1.0p-24);
  }
}

// Copy resident peers' rows to/from a by-id buffer (device) on this GPU.
template <typename T>
__global__ void shard_gather_kernel(const T* pool, const std::uint32_t* loc, std::uint64_t n,
                                    std::uint64_t dim, std::uint64_t ld, std::uint64_t R,
                                    std::uint32_t me, T* out, std::uint8_t* mask, int to_pool) {
  const std::uint64_t total = n * dim;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t p = e / dim, j = e % dim;
    const std::uint32_t r = loc[p];
    const bool mine = r / R == me;
    if (j == 0 && mask) mask[p] = mine ? 1 : 0;
    if (!mine) continue;
    if (to_pool)
      const_cast<T*>(pool)[(r % R) * ld + j] = out[p * dim + j];
    else
      out[p * dim + j] = pool[(r % R) * ld + j];
  }
}

unsigned grid_cap(std::uint64_t work) {
  std::uint64_t b = (work + 255) / 256;
  if (b > 148ull * 32) b = 148ull * 32;
  return (unsigned)(b ? b : 1);
}

}  // namespace

// ---------------------------------------------------------------------------
constexpr int kMaxSlabs = 8;

// One round's replicated tables (ring slot of the slab pipeline).
struct TableSlot {
  DeviceBuffer goff, rows_local, act_local, cnt_local, src_row, dst_row, act_cross, cnt_cross,
      moves, n_moves;
  cudaEvent_t ready = nullptr;             // written (control stream)
  cudaEvent_t freed[kMaxSlabs] = {};       // slab k is done with it
  bool used[kMaxSlabs] = {};
  int cross = 0;
  int partial = 0;  // cross round in the partial-sum mode (MOSHPIT_CROSS_PARTIAL)
  ~TableSlot() {
    if (ready) cudaEventDestroy(ready);
    for (auto e : freed)
      if (e) cudaEventDestroy(e);
  }
};

struct Shard {
  std::unique_ptr<Plane> plane;
  Xoshiro fail, clock;
  double p = 0.0;
  int dtype = MOSHPIT_F32;
  std::size_t es = 4;
  std::uint64_t dim = 0, ld = 0, R = 0;
  std::uint32_t world = 1, me = 0, Mg = 1, M = 1, d = 1;
  std::uint32_t nhost = 1, proc = 0, procs = 1;  // ranks [me, me+nhost) live here
  int device = 0;
  bool emulate = false;    // nhost == world: no peers, no barriers
  bool connected = false;  // peers' pools/flags mapped (open_peers)
  bool probe = false;      // profiling only: no inter-rank barriers (results invalid)
  int cross_mode = 0;      // MOSHPIT_CROSS_EXACT (reference tree) / MOSHPIT_CROSS_PARTIAL
  // slab pipeline: SMs' worth of CTAs for the local (kernel 2) and cross
  // kernels while they share the GPU (0 = all; MOSHPIT_PIPE_LOCAL_SMS /
  // MOSHPIT_PIPE_CROSS_SMS)
  int pipe_local_sms = 0, pipe_cross_sms = 0;
  std::uint32_t round_no = 0;
  // replicated per-trial state and the table ring
  DeviceBuffer loc, err, pool_tab, flag_tab, totals;
  std::vector<std::unique_ptr<TableSlot>> ring;
  // slab pipeline
  std::uint32_t S = 1;
  std::uint64_t vb[kMaxSlabs] = {}, ve[kMaxSlabs] = {};
  std::uint32_t slab_done[kMaxSlabs] = {};  // rounds completed (enqueued) per slab
  unsigned long long epoch[kMaxSlabs] = {};
  std::unique_ptr<StreamHolder> cs, ss[kMaxSlabs];
  cudaEvent_t ev_user = nullptr, ev_slab[kMaxSlabs] = {};
  cudaStream_t user = nullptr;
  // pools of the hosted ranks; IPC mappings of the others
  std::vector<std::unique_ptr<DeviceBuffer>> own_pools;
  std::unique_ptr<DeviceBuffer> staging;  // voided-row moves (shared: slabs own columns)
  void* pools[kMaxWorld] = {};
  DeviceBuffer flags;  // [kMaxSlabs][kMaxWorld] u64 (this process's slots)
  unsigned long long* peer_flags[kMaxWorld] = {};  // by process
  std::vector<void*> opened;  // IPC mappings to close
  // timing of the data-plane kernels (CUDA events on their streams)
  bool timing = false;
  struct TEv {
    cudaEvent_t a, b;
    int kind;  // 0 local, 1 cross phase A, 2 cross phase B
  };
  std::vector<TEv> tev;
  std::size_t tev_used = 0;
  double last_a_ms = 0.0, last_b_ms = 0.0;
  // copy-engine cross round (MOSHPIT_CROSS_CE=1, S = 1 only; the default is
  // the SM-pull kernels)
  bool ce = false;
  PinnedBuffer htab;
  std::unique_ptr<StreamHolder> cstream[2];
  DeviceBuffer cstage[2];
  cudaEvent_t ev_copied[2] = {}, ev_free[2] = {}, ev_go = nullptr;
  std::vector<void*> cdst, csrc;
  std::vector<std::size_t> csize;

  ~Shard() {
    for (cudaEvent_t e : {ev_copied[0], ev_copied[1], ev_free[0], ev_free[1], ev_go, ev_user})
      if (e) cudaEventDestroy(e);
    for (auto e : ev_slab)
      if (e) cudaEventDestroy(e);
    for (void* q : opened) cudaIpcCloseMemHandle(q);
    for (auto& t : tev) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
  }

  bool hosts(std::uint32_t r) const { return r >= me && r < me + nhost; }
  std::uint64_t nvec() const { return (dim + (16 / es) - 1) / (16 / es); }
  std::uint32_t n() const { return (std::uint32_t)plane->n; }
  cudaStream_t slab_stream(std::uint32_t k) const { return S == 1 ? user : ss[k]->s; }
  cudaStream_t ctl_stream() const { return S == 1 ? user : cs->s; }

  TEv& tpair(int kind) {
    if (tev_used == tev.size()) {
      TEv t{};
      MB_CUDA(cudaEventCreate(&t.a));
      MB_CUDA(cudaEventCreate(&t.b));
      tev.push_back(t);
    }
    TEv& t = tev[tev_used++];
    t.kind = kind;
    return t;
  }

  void alloc_slot(TableSlot& t) {
    const std::uint64_t nn = n();
    t.goff.resize((nn + 1) * 4 + 16);
    t.rows_local.resize(nn * 4);
    t.act_local.resize((std::uint64_t)world * nn * 4);
    t.cnt_local.resize((std::uint64_t)world * 16 + 16);
    t.src_row.resize(nn * 4);
    t.dst_row.resize(nn * 4);
    t.act_cross.resize(nn * 4);
    t.cnt_cross.resize(16);
    t.moves.resize((std::uint64_t)world * R * 8);
    t.n_moves.resize(world * 4 + 16);
    MB_CUDA(cudaEventCreateWithFlags(&t.ready, cudaEventDisableTiming));
    for (std::uint32_t k = 0; k < S; ++k)
      MB_CUDA(cudaEventCreateWithFlags(&t.freed[k], cudaEventDisableTiming));
  }

  void barrier(std::uint32_t k, cudaStream_t s) {
    if (emulate || procs == 1 || probe) return;
    ++epoch[k];
    peer_barrier_kernel<<<1, 32, 0, s>>>(flags.as<unsigned long long>(),
                                        flag_tab.as<unsigned long long* const>(), proc, procs,
                                        epoch[k], k);
    MB_LAUNCH_CHECK();
  }

  template <typename T>
  CrossArgs<T> cross_args(const TableSlot& t, std::uint32_t r, std::uint32_t k, bool full_slab) {
    CrossArgs<T> a;
    for (std::uint32_t h = 0; h < world; ++h) a.pools[h] = static_cast<T*>(pools[h]);
    a.ld_vec = ld * es / 16;
    a.R = R;
    a.vb = vb[k];
    a.ve = ve[k];
    const std::uint64_t W = a.ve - a.vb;
    a.c0 = a.vb + W * r / world;
    a.c1 = a.vb + W * (r + 1) / world;
    a.n_tiles = ((full_slab ? W : a.c1 - a.c0) + kCrossThreads - 1) / kCrossThreads;
    a.me = r;
    a.world = world;
    a.goff = t.goff.as<std::uint32_t>();
    a.src_row = t.src_row.as<std::uint32_t>();
    a.dst_row = t.dst_row.as<std::uint32_t>();
    a.act = t.act_cross.as<std::uint32_t>();
    a.cnt = t.cnt_cross.as<std::uint32_t>();
    return a;
  }

  int sm_count() const {
    int sms = 0;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    return sms;
  }

  template <typename T>
  void cross_launch(const TableSlot& t, std::uint32_t r, std::uint32_t k, cudaStream_t s) {
    CrossArgs<T> a = cross_args<T>(t, r, k, false);
    static int per = -1;
    if (per < 0) {
      MB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cross_mean_kernel<T>,
                                                            kCrossThreads, 0));
      if (const char* e = std::getenv("MOSHPIT_CROSS_CTAS")) per = std::min(per, std::atoi(e));
      if (per < 1) per = 1;
    }
    int sms = sm_count();
    if (S > 1 && pipe_cross_sms > 0) sms = std::min(sms, pipe_cross_sms);
    if (a.n_tiles) cross_mean_kernel<T><<<sms * per, kCrossThreads, 0, s>>>(a);
    MB_LAUNCH_CHECK();
  }

  // partial-sum mode: phase 0 (rank r's members summed into its first member
  // row, whole slab width) and phase A (chunk r of the means from the w
  // partial rows)
  template <typename T>
  void partial_launch(const TableSlot& t, std::uint32_t r, std::uint32_t k, cudaStream_t s) {
    CrossArgs<T> a = cross_args<T>(t, r, k, true);
    MoveItems mv;
    if (p > 0.0) {  // the voided groups' row pulls ride along (phase 0 of the moves)
      mv.moves = t.moves.as<std::uint32_t>();
      mv.n_moves = t.n_moves.as<std::uint32_t>();
      mv.staging = staging->as<T>() + (hosts(r) ? (r - me) : 0) * R * ld;
    }
    int sms = sm_count();
    if (S > 1 && pipe_cross_sms > 0) sms = std::min(sms, pipe_cross_sms);
    if (a.n_tiles) partial_sum_kernel<T><<<sms * 8, kCrossThreads, 0, s>>>(a, mv);
    MB_LAUNCH_CHECK();
  }
  template <typename T>
  void combine_launch(const TableSlot& t, std::uint32_t r, std::uint32_t k, cudaStream_t s) {
    CrossArgs<T> a = cross_args<T>(t, r, k, false);
    a.n_tiles = (a.c1 - a.c0 + kPullU * kCrossThreads - 1) / (kPullU * kCrossThreads);
    int sms = sm_count();
    if (S > 1 && pipe_cross_sms > 0) sms = std::min(sms, pipe_cross_sms);
    if (a.n_tiles) {
      if (world == 2) partial_combine_kernel<T, 2><<<sms * 8, kCrossThreads, 0, s>>>(a);
      else if (world == 4) partial_combine_kernel<T, 4><<<sms * 8, kCrossThreads, 0, s>>>(a);
      else partial_combine_kernel<T, kMaxWorld><<<sms * 8, kCrossThreads, 0, s>>>(a);
    }
    MB_LAUNCH_CHECK();
  }

  template <typename T>
  void pull_launch(const TableSlot& t, std::uint32_t r, std::uint32_t k, cudaStream_t s) {
    if (world < 2) return;
    CrossArgs<T> a = cross_args<T>(t, r, k, true);
    static int per = -1;
    if (per < 0) {
      per = 8;
      if (const char* e = std::getenv("MOSHPIT_PULL_CTAS")) per = std::max(1, std::atoi(e));
    }
    MoveItems mv;
    if (p > 0.0) {  // the staged voided rows go to their new rows in the same launch
      mv.moves = t.moves.as<std::uint32_t>();
      mv.n_moves = t.n_moves.as<std::uint32_t>();
      mv.staging = staging->as<T>() + (hosts(r) ? (r - me) : 0) * R * ld;
    }
    int sms = sm_count();
    if (S > 1 && pipe_cross_sms > 0) sms = std::min(sms, pipe_cross_sms);
    if (a.n_tiles) shard_pull_kernel<T><<<sms * per, kCrossThreads, 0, s>>>(a, mv);
    MB_LAUNCH_CHECK();
  }

  template <typename T>
  void moves_launch(const TableSlot& t, std::uint32_t r, std::uint32_t k, int phase,
                    cudaStream_t s) {
    if (p <= 0.0) return;  // no voided groups without failures
    move_rows_kernel<T><<<grid_cap(R * (ve[k] - vb[k])), 256, 0, s>>>(
        pool_tab.as<T* const>(), t.moves.as<std::uint32_t>(), t.n_moves.as<std::uint32_t>(), r,
        R, ld * es / 16, vb[k], ve[k], staging->as<T>() + (hosts(r) ? (r - me) : 0) * R * ld,
        phase);
    MB_LAUNCH_CHECK();
  }

  // Copy a list of (dst, src, bytes) on stream cs: one async copy each (the
  // copy engines take peer pointers of the IPC-mapped pools directly).
  void copy_list(cudaStream_t c) {
    for (std::size_t i = 0; i < cdst.size(); ++i)
      MB_CUDA(cudaMemcpyAsync(cdst[i], csrc[i], csize[i], cudaMemcpyDefault, c));
    cdst.clear();
    csrc.clear();
    csize.clear();
  }

  void ce_init() {
    if (cstream[0]) return;
    for (int i = 0; i < 2; ++i) {
      cstream[i] = std::make_unique<StreamHolder>();
      MB_CUDA(cudaEventCreateWithFlags(&ev_copied[i], cudaEventDisableTiming));
      MB_CUDA(cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming));
    }
    MB_CUDA(cudaEventCreateWithFlags(&ev_go, cudaEventDisableTiming));
  }

  // Host copy of the cross round's replicated tables (synchronises s once).
  void ce_fetch_tables(const TableSlot& t, cudaStream_t s) {
    const std::uint64_t nn = n();
    htab.resize((4 * nn + 8) * 4);
    auto* h = htab.as<std::uint32_t>();
    MB_CUDA(cudaMemcpyAsync(h, t.src_row.ptr, nn * 4, cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaMemcpyAsync(h + nn, t.dst_row.ptr, nn * 4, cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaMemcpyAsync(h + 2 * nn, t.goff.ptr, (nn + 1) * 4, cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaMemcpyAsync(h + 3 * nn + 1, t.act_cross.ptr, nn * 4, cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaMemcpyAsync(h + 4 * nn + 1, t.cnt_cross.ptr, 16, cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaStreamSynchronize(s));
  }

  // Phase A for rank r (copy engines): staged remote chunks + tree kernel.
  template <typename T>
  void cross_ce(const TableSlot& t, std::uint32_t r, cudaStream_t s) {
    ce_init();
    const std::uint64_t nn = n();
    const auto* h = htab.as<std::uint32_t>();
    const std::uint32_t* hsrc = h;
    const std::uint32_t* hgoff = h + 2 * nn;
    const std::uint32_t* hact = h + 3 * nn + 1;
    const std::uint32_t nact = h[4 * nn + 1 + 1];
    CrossArgs<T> a = cross_args<T>(t, r, 0, false);
    const std::uint64_t cbytes = (a.c1 - a.c0) * 16;
    if (nact == 0 || cbytes == 0) return;
    const std::uint32_t nrem = M - Mg;  // full grid: Mg members of a line per GPU
    const std::uint64_t per_group = (std::uint64_t)nrem * cbytes;
    std::uint32_t B = (std::uint32_t)std::max<std::uint64_t>(
        1, std::min<std::uint64_t>(nact, (512ull << 20) / std::max<std::uint64_t>(per_group, 1)));
    for (int i = 0; i < 2; ++i) cstage[i].resize(B * per_group + 16);
    int per = 0;
    MB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cross_staged_kernel<T>,
                                                          kCrossThreads, 0));
    MB_CUDA(cudaEventRecord(ev_go, s));  // after the barrier: peers' rows are final
    for (int i = 0; i < 2; ++i) MB_CUDA(cudaStreamWaitEvent(cstream[i]->s, ev_go, 0));
    std::uint32_t batch = 0;
    for (std::uint32_t gb = 0; gb < nact; gb += B, ++batch) {
      const std::uint32_t ge = std::min(nact, gb + B);
      const int slot = batch & 1;
      cudaStream_t c = cstream[slot]->s;
      if (batch >= 2) MB_CUDA(cudaStreamWaitEvent(c, ev_free[slot], 0));
      char* st = cstage[slot].as<char>();
      for (std::uint32_t gi = gb; gi < ge; ++gi) {
        const std::uint32_t g = hact[gi];
        std::uint32_t q = 0;
        for (std::uint32_t pos = hgoff[g]; pos < hgoff[g + 1]; ++pos) {
          const std::uint32_t sr = hsrc[pos];
          if (sr / R == r) continue;
          cdst.push_back(st + ((std::uint64_t)(gi - gb) * nrem + q++) * cbytes);
          csrc.push_back(static_cast<char*>(pools[sr / R]) + (sr % R) * ld * es + a.c0 * 16);
          csize.push_back(cbytes);
        }
      }
      copy_list(c);
      MB_CUDA(cudaEventRecord(ev_copied[slot], c));
      MB_CUDA(cudaStreamWaitEvent(s, ev_copied[slot], 0));
      cross_staged_kernel<T><<<sm_count() * (per > 0 ? per : 1), kCrossThreads, 0, s>>>(
          a, cstage[slot].as<T>(), gb, ge, nrem);
      MB_LAUNCH_CHECK();
      MB_CUDA(cudaEventRecord(ev_free[slot], s));
    }
  }

  // Phase B for rank r (copy engines): foreign chunk means into the group's
  // first local member row, then the local fan-out.
  template <typename T>
  void pull_ce(const TableSlot& t, std::uint32_t r, cudaStream_t s) {
    if (world < 2) return;
    const std::uint64_t nn = n();
    const auto* h = htab.as<std::uint32_t>();
    const std::uint32_t* hdst = h + nn;
    const std::uint32_t* hgoff = h + 2 * nn;
    const std::uint32_t* hact = h + 3 * nn + 1;
    const std::uint32_t nact = h[4 * nn + 1 + 1];
    const std::uint64_t nv = nvec();
    for (std::uint32_t gi = 0; gi < nact; ++gi) {
      const std::uint32_t g = hact[gi];
      std::uint32_t rep[kMaxWorld];
      for (std::uint32_t q = 0; q < world; ++q) rep[q] = 0xffffffffu;
      for (std::uint32_t pos = hgoff[g]; pos < hgoff[g + 1]; ++pos) {
        const std::uint32_t dd = hdst[pos], q = (std::uint32_t)(dd / R);
        if (rep[q] == 0xffffffffu) rep[q] = dd;
      }
      char* mine = static_cast<char*>(pools[r]) + (rep[r] % R) * ld * es;
      for (std::uint32_t q = 0; q < world; ++q) {
        if (q == r) continue;
        const std::uint64_t c0 = nv * q / world, c1 = nv * (q + 1) / world;
        if (c1 == c0) continue;
        cdst.push_back(mine + c0 * 16);
        csrc.push_back(static_cast<char*>(pools[q]) + (rep[q] % R) * ld * es + c0 * 16);
        csize.push_back((c1 - c0) * 16);
      }
    }
    copy_list(s);
    if (Mg > 1) {
      CrossArgs<T> a = cross_args<T>(t, r, 0, true);
      local_fanout_kernel<T><<<sm_count() * 8, kCrossThreads, 0, s>>>(a, nv);
      MB_LAUNCH_CHECK();
    }
  }

  // Round `rr` of slab k from its ring slot: the data plane of every hosted
  // rank on the slab's columns.
  void run_slab(std::uint32_t k, std::uint32_t rr) {
    TableSlot& t = *ring[rr % ring.size()];
    cudaStream_t s = slab_stream(k);
    if (S > 1) MB_CUDA(cudaStreamWaitEvent(s, t.ready, 0));
    const bool f32 = dtype == MOSHPIT_F32;
    if (!t.cross) {
      TEv* te = timing ? &tpair(0) : nullptr;
      if (te) MB_CUDA(cudaEventRecord(te->a, s));
      const std::uint64_t kv = 16 / es;
      const std::uint64_t c0 = vb[k] * kv, c1 = std::min<std::uint64_t>(ve[k] * kv, dim);
      if (S > 1) set_k2_grid_sms(pipe_local_sms);
      for (std::uint32_t r = me; r < me + nhost; ++r) {
        const std::uint32_t* act = t.act_local.as<std::uint32_t>() + (std::uint64_t)r * n();
        const std::uint32_t* cnt = t.cnt_local.as<std::uint32_t>() + r * 4;
        if (c1 <= c0) break;
        if (f32)
          launch_group_mean<float>(static_cast<float*>(pools[r]) + c0, ld, c1 - c0,
                                   t.rows_local.as<std::uint32_t>(), t.goff.as<std::uint32_t>(),
                                   act, cnt, M, 0, s);
        else
          launch_group_mean<double>(static_cast<double*>(pools[r]) + c0, ld, c1 - c0,
                                    t.rows_local.as<std::uint32_t>(), t.goff.as<std::uint32_t>(),
                                    act, cnt, M, 0, s);
      }
      if (S > 1) set_k2_grid_sms(0);
      if (te) MB_CUDA(cudaEventRecord(te->b, s));
    } else {
      if (ce) ce_fetch_tables(t, s);
      TEv* ta = timing ? &tpair(1) : nullptr;
      barrier(k, s);  // peers finished writing the rows we are about to read
      if (ta) MB_CUDA(cudaEventRecord(ta->a, s));
      if (t.partial) {
        // phase 0: partial rows (local HBM) + the voided rows' pulls (NVLink)
        // in one launch; the barrier then publishes the partial rows
        for (std::uint32_t r = me; r < me + nhost; ++r) {
          if (f32) partial_launch<float>(t, r, k, s);
          else partial_launch<double>(t, r, k, s);
        }
        barrier(k, s);
      }
      for (std::uint32_t r = me; r < me + nhost; ++r) {
        if (f32) {
          if (ce) cross_ce<float>(t, r, s);
          else if (t.partial) combine_launch<float>(t, r, k, s);
          else cross_launch<float>(t, r, k, s);
          if (!t.partial) moves_launch<float>(t, r, k, 0, s);
        } else {
          if (ce) cross_ce<double>(t, r, s);
          else if (t.partial) combine_launch<double>(t, r, k, s);
          else cross_launch<double>(t, r, k, s);
          if (!t.partial) moves_launch<double>(t, r, k, 0, s);
        }
      }
      if (ta) MB_CUDA(cudaEventRecord(ta->b, s));
      barrier(k, s);  // every chunk mean is in its owner's rows; raw reads are done
      TEv* tb = timing ? &tpair(2) : nullptr;
      if (tb) MB_CUDA(cudaEventRecord(tb->a, s));
      for (std::uint32_t r = me; r < me + nhost; ++r) {
        if (f32) {
          if (ce) {
            pull_ce<float>(t, r, s);
            moves_launch<float>(t, r, k, 1, s);
          } else {
            pull_launch<float>(t, r, k, s);  // + the voided rows' writes
          }
        } else {
          if (ce) {
            pull_ce<double>(t, r, s);
            moves_launch<double>(t, r, k, 1, s);
          } else {
            pull_launch<double>(t, r, k, s);
          }
        }
      }
      if (tb) MB_CUDA(cudaEventRecord(tb->b, s));
      barrier(k, s);  // peers finished pulling from our rows before we touch them again
    }
    if (S > 1) {
      MB_CUDA(cudaEventRecord(t.freed[k], s));
      t.used[k] = true;
    }
    slab_done[k] = rr + 1;
  }

  // One round: identical host draws, kernel 1 and placement on every rank
  // (into ring slot r), then the slabs' data planes -- slab k runs round r-k.
  std::uint32_t round(cudaStream_t s, int* crossed) {
    user = s;
    const std::uint32_t r = round_no;
    const std::uint32_t axis = d ? r % d : 0;
    const int cross = (world > 1 && axis == d - 1) ? 1 : 0;
    TableSlot& t = *ring[r % ring.size()];
    cudaStream_t c = ctl_stream();
    if (S > 1) {
      // caller's prior work on s (e.g. the synthetic init) comes first
      MB_CUDA(cudaEventRecord(ev_user, s));
      MB_CUDA(cudaStreamWaitEvent(c, ev_user, 0));
      for (std::uint32_t k = 0; k < S; ++k) MB_CUDA(cudaStreamWaitEvent(ss[k]->s, ev_user, 0));
      for (std::uint32_t k = 0; k < S; ++k)
        if (t.used[k]) MB_CUDA(cudaStreamWaitEvent(c, t.freed[k], 0));  // slot reuse
    }
    ++round_no;
    const std::uint32_t active = plane->round(&fail, p, clock, dtype, nullptr, 0, 0, c, 0);
    PlaceArgs a;
    a.n = n();
    a.world = world;
    a.Mg = Mg;
    a.R = R;
    a.cross = cross;
    a.members = plane->members.as<std::uint32_t>();
    a.goff = plane->goff.as<std::uint32_t>();
    a.counts = plane->counts.as<std::uint32_t>();
    a.gvoid = plane->gvoid.as<std::uint8_t>();
    a.loc = loc.as<std::uint32_t>();
    a.rows_local = t.rows_local.as<std::uint32_t>();
    a.act_local = t.act_local.as<std::uint32_t>();
    a.cnt_local = t.cnt_local.as<std::uint32_t>();
    a.src_row = t.src_row.as<std::uint32_t>();
    a.dst_row = t.dst_row.as<std::uint32_t>();
    a.act_cross = t.act_cross.as<std::uint32_t>();
    a.cnt_cross = t.cnt_cross.as<std::uint32_t>();
    a.moves = t.moves.as<std::uint32_t>();
    a.n_moves = t.n_moves.as<std::uint32_t>();
    a.err = err.as<std::uint32_t>();
    a.goff_out = t.goff.as<std::uint32_t>();
    a.totals = totals.as<unsigned long long>();
    place_kernel<<<1, 1024, 0, c>>>(a);
    MB_LAUNCH_CHECK();
    t.cross = cross;
    t.partial = cross && cross_mode == MOSHPIT_CROSS_PARTIAL;
    plane->mark_done(c);
    if (S > 1) MB_CUDA(cudaEventRecord(t.ready, c));
    for (std::uint32_t k = 0; k < S; ++k)
      if (r >= k && slab_done[k] == r - k) run_slab(k, r - k);
    if (crossed) *crossed = cross;
    return active;
  }

  // Complete the lagging slabs (rounds already tabled) and order `s` after
  // every slab stream.  S = 1: nothing to do.
  void flush(cudaStream_t s) {
    if (S == 1) return;
    catch_up();
    join(s);
  }
  // issue every round still owed to the lagging slabs
  void catch_up() {
    for (std::uint32_t step = 0; step + 1 < S; ++step)
      for (std::uint32_t k = 0; k < S; ++k)
        if (slab_done[k] < round_no) run_slab(k, slab_done[k]);
  }
  // order s after everything issued on the slab streams
  void join(cudaStream_t s) {
    for (std::uint32_t k = 0; k < S; ++k) {
      MB_CUDA(cudaEventRecord(ev_slab[k], ss[k]->s));
      MB_CUDA(cudaStreamWaitEvent(s, ev_slab[k], 0));
    }
  }
  // Host <-> pool copies of hosted rank r's rows.  With the slab pipeline
  // each slab's columns move on that slab's stream, so a load overlaps the
  // first slabs' rounds and a store overlaps the last slabs' catch-up rounds.
  void copy_rows(std::uint32_t r, void* host, std::uint64_t host_ld, bool to_host,
                 cudaStream_t s) {
    const auto kind = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
    auto copy = [&](std::uint64_t c0, std::uint64_t c1, cudaStream_t cs) {
      if (c1 <= c0) return;
      char* dev = static_cast<char*>(pools[r]) + c0 * es;
      char* hst = static_cast<char*>(host) + c0 * es;
      if (to_host)
        MB_CUDA(cudaMemcpy2DAsync(hst, host_ld, dev, ld * es, (c1 - c0) * es, R, kind, cs));
      else
        MB_CUDA(cudaMemcpy2DAsync(dev, ld * es, hst, host_ld, (c1 - c0) * es, R, kind, cs));
    };
    if (S == 1) {
      copy(0, dim, s);
      return;
    }
    MB_CUDA(cudaEventRecord(ev_user, s));
    for (std::uint32_t k = 0; k < S; ++k) MB_CUDA(cudaStreamWaitEvent(ss[k]->s, ev_user, 0));
    if (to_host) catch_up();
    const std::uint64_t kv = 16 / es;
    for (std::uint32_t k = 0; k < S; ++k)
      copy(vb[k] * kv, std::min<std::uint64_t>(ve[k] * kv, dim), ss[k]->s);
    // a store joins the caller's stream; a load stays on the slab streams
    // (joining would make every slab's first round wait for the whole load):
    // the shard's later rounds / stores / reads are ordered after it, and
    // `s` passes it at the next flush or store_rows
    if (to_host) join(s);
  }
};

}  // namespace mb200

using namespace mb200;

struct moshpit_shard {
  std::unique_ptr<Shard> s;
};

namespace {

void shard_require(moshpit_shard* h) {
  if (!h || !h->s) throw std::invalid_argument("shard: null handle");
}

}  // namespace

extern "C" {

int moshpit_shard_create_ex(int dtype, std::uint32_t M, std::uint32_t d, std::uint64_t n,
                            double p_round, std::uint64_t seed, std::uint64_t dim,
                            std::int32_t first_rank, std::int32_t ranks_here, std::int32_t world,
                            std::int32_t slabs, std::int32_t device, moshpit_shard** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("shard_create: null out");
    const std::size_t es = elem_size(dtype);
    if (M < 1 || d < 1) throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
    if (p_round < 0.0 || p_round > 1.0)
      throw std::invalid_argument("FailureModel: p_round must be in [0,1]");
    if (world < 1 || world > kMaxWorld) throw std::invalid_argument("shard: world in [1, 8]");
    if (ranks_here < 1 || world % ranks_here != 0)
      throw std::invalid_argument("shard: ranks per process must divide world");
    if (first_rank < 0 || first_rank % ranks_here != 0 || first_rank + ranks_here > world)
      throw std::invalid_argument("shard: hosted ranks must be an aligned block of [0, world)");
    if (slabs < 1 || slabs > kMaxSlabs) throw std::invalid_argument("shard: slabs in [1, 8]");
    if (M % (std::uint32_t)world != 0)
      throw std::invalid_argument("shard: the GPU count must divide M (split of grid digit d-1)");
    if (M > 32) throw std::invalid_argument("shard: groups larger than 32 are not sharded");
    const std::uint64_t cap = moshpit_grid_capacity(M, d);
    if (n != cap)
      throw std::invalid_argument("shard: peer sharding needs a full grid (N == M^d)");
    if (cap > 0xffffffffull) throw std::invalid_argument("shard: grid larger than 2^32 cells");
    require_device();
    DeviceGuard g(device);
    auto sh = std::make_unique<Shard>();
    Shard& S = *sh;
    MB_CUDA(cudaGetDevice(&S.device));
    S.dtype = dtype;
    S.es = es;
    S.dim = dim;
    S.ld = padded_ld(dim, es);
    S.world = (std::uint32_t)world;
    S.me = (std::uint32_t)first_rank;
    S.nhost = (std::uint32_t)ranks_here;
    S.proc = S.me / S.nhost;
    S.procs = S.world / S.nhost;
    S.emulate = S.nhost == S.world;
    S.M = M;
    S.d = d;
    S.Mg = M / (std::uint32_t)world;
    S.R = cap / (std::uint64_t)world;
    S.p = p_round;
    if (const char* e = std::getenv("MOSHPIT_CROSS_CE")) S.ce = std::atoi(e) != 0;
    const std::uint64_t nv = S.nvec();
    S.S = (std::uint32_t)std::max<std::uint64_t>(1, std::min<std::uint64_t>(slabs, nv));
    if (S.ce && S.S > 1) throw std::invalid_argument("shard: the copy-engine round needs slabs = 1");
    // measured on 2 and 4 B200s (C2, profiles/r02/pipe_sweep_*.txt): ~70 % of the
    // SMs' worth of kernel-2 CTAs and ~30 % for the cross kernels beat
    // uncapped grids (4080 vs 3570 GB/s at 2 GPUs, slabs = 4)
    if (S.S > 1) {
      int sms = 0;
      MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, S.device));
      S.pipe_local_sms = (sms * 104 + 74) / 148;
      S.pipe_cross_sms = sms - S.pipe_local_sms;
    }
    if (const char* e = std::getenv("MOSHPIT_PIPE_LOCAL_SMS")) S.pipe_local_sms = std::atoi(e);
    if (const char* e = std::getenv("MOSHPIT_PIPE_CROSS_SMS")) S.pipe_cross_sms = std::atoi(e);
    for (std::uint32_t k = 0; k < S.S; ++k) {
      S.vb[k] = nv * k / S.S;
      S.ve[k] = nv * (k + 1) / S.S;
    }
    S.plane = std::make_unique<Plane>(M, d, n, S.device);
    Xoshiro cells = Xoshiro::named(seed, "cells");
    S.fail = Xoshiro::named(seed, "failures");
    S.clock = Xoshiro::named(seed, "priorities");
    StreamHolder st;
    S.plane->init_cells(cells, st.s);
    S.loc.resize(n * 4);
    init_loc_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st.s>>>(
        S.plane->cellbuf.as<std::uint64_t>(), S.loc.as<std::uint32_t>(), n);
    MB_LAUNCH_CHECK();
    S.plane->mark_done(st.s);
    const std::uint32_t nslots = S.S == 1 ? 1 : S.S + 1;
    for (std::uint32_t q = 0; q < nslots; ++q) {
      S.ring.push_back(std::make_unique<TableSlot>());
      S.alloc_slot(*S.ring.back());
    }
    if (S.S > 1) {
      S.cs = std::make_unique<StreamHolder>();
      for (std::uint32_t k = 0; k < S.S; ++k) {
        S.ss[k] = std::make_unique<StreamHolder>();
        MB_CUDA(cudaEventCreateWithFlags(&S.ev_slab[k], cudaEventDisableTiming));
      }
      MB_CUDA(cudaEventCreateWithFlags(&S.ev_user, cudaEventDisableTiming));
    }
    S.err.resize(16);
    MB_CUDA(cudaMemsetAsync(S.err.ptr, 0, 16, st.s));
    S.totals.resize(8 * (2 * kMaxWorld + 2));
    MB_CUDA(cudaMemsetAsync(S.totals.ptr, 0, 8 * (2 * kMaxWorld + 2), st.s));
    for (std::uint32_t k = 0; k < S.nhost; ++k) {
      S.own_pools.push_back(std::make_unique<DeviceBuffer>(S.R * S.ld * es));
      MB_CUDA(cudaMemsetAsync(S.own_pools.back()->ptr, 0, S.R * S.ld * es, st.s));
      S.pools[S.me + k] = S.own_pools.back()->ptr;
    }
    if (p_round > 0.0)  // voided-row moves stage through here (one block per hosted rank)
      S.staging = std::make_unique<DeviceBuffer>((std::uint64_t)S.nhost * S.R * S.ld * es);
    S.flags.resize((std::uint64_t)kMaxSlabs * kMaxWorld * 8);
    MB_CUDA(cudaMemsetAsync(S.flags.ptr, 0, (std::uint64_t)kMaxSlabs * kMaxWorld * 8, st.s));
    S.pool_tab.resize(kMaxWorld * 8);
    S.flag_tab.resize(kMaxWorld * 8);
    MB_CUDA(cudaMemcpyAsync(S.pool_tab.ptr, S.pools, sizeof(S.pools), cudaMemcpyHostToDevice,
                            st.s));
    MB_CUDA(cudaStreamSynchronize(st.s));
    *out = new moshpit_shard{std::move(sh)};
  });
}

int moshpit_shard_create(int dtype, std::uint32_t M, std::uint32_t d, std::uint64_t n,
                         double p_round, std::uint64_t seed, std::uint64_t dim,
                         std::int32_t rank, std::int32_t world, std::int32_t emulate,
                         std::int32_t device, moshpit_shard** out) {
  if (emulate) {
    if (rank < 0 || rank >= world) {
      g_last_error = "shard: rank outside [0, world)";
      return MOSHPIT_ERR_INVALID_ARGUMENT;
    }
    return moshpit_shard_create_ex(dtype, M, d, n, p_round, seed, dim, 0, world, world, 1,
                                   device, out);
  }
  if (rank < 0 || rank >= world) {
    g_last_error = "shard: rank outside [0, world)";
    return MOSHPIT_ERR_INVALID_ARGUMENT;
  }
  return moshpit_shard_create_ex(dtype, M, d, n, p_round, seed, dim, rank, 1, world, 1, device,
                                 out);
}

int moshpit_shard_destroy(moshpit_shard* h) {
  return guarded([&] {
    if (!h) return;
    if (h->s) {
      DeviceGuard g(h->s->device);
      cudaDeviceSynchronize();
      h->s.reset();
    }
    delete h;
  });
}

// Per hosted rank r (in order): 128 bytes = cudaIpcMemHandle_t of rank r's
// pool and of this process's barrier flags.  out: ranks_here * 128 bytes.
int moshpit_shard_ipc_handles(moshpit_shard* h, void* out) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    if (S.emulate) throw std::invalid_argument("shard: emulation mode has no IPC handles");
    DeviceGuard g(S.device);
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
    cudaIpcMemHandle_t fl;
    MB_CUDA(cudaIpcGetMemHandle(&fl, S.flags.ptr));
    for (std::uint32_t k = 0; k < S.nhost; ++k) {
      cudaIpcMemHandle_t a;
      MB_CUDA(cudaIpcGetMemHandle(&a, S.own_pools[k]->ptr));
      std::memcpy(static_cast<char*>(out) + k * 128, &a, 64);
      std::memcpy(static_cast<char*>(out) + k * 128 + 64, &fl, 64);
    }
  });
}

// all: world * 128 bytes, rank-ordered entries from moshpit_shard_ipc_handles.
int moshpit_shard_open_peers(moshpit_shard* h, const void* all) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    if (S.emulate) return;
    DeviceGuard g(S.device);
    for (std::uint32_t r = 0; r < S.world; ++r) {
      const std::uint32_t q = r / S.nhost;  // owning process
      if (S.hosts(r)) {
        S.peer_flags[q] = S.flags.as<unsigned long long>();
        continue;
      }
      cudaIpcMemHandle_t a, b;
      std::memcpy(&a, static_cast<const char*>(all) + r * 128, 64);
      std::memcpy(&b, static_cast<const char*>(all) + r * 128 + 64, 64);
      void* pa = nullptr;
      MB_CUDA(cudaIpcOpenMemHandle(&pa, a, cudaIpcMemLazyEnablePeerAccess));
      S.opened.push_back(pa);
      S.pools[r] = pa;
      if (r % S.nhost == 0) {  // one flags mapping per remote process
        void* pb = nullptr;
        MB_CUDA(cudaIpcOpenMemHandle(&pb, b, cudaIpcMemLazyEnablePeerAccess));
        S.opened.push_back(pb);
        S.peer_flags[q] = static_cast<unsigned long long*>(pb);
      }
    }
    MB_CUDA(cudaMemcpy(S.pool_tab.ptr, S.pools, sizeof(S.pools), cudaMemcpyHostToDevice));
    MB_CUDA(cudaMemcpy(S.flag_tab.ptr, S.peer_flags, sizeof(S.peer_flags),
                       cudaMemcpyHostToDevice));
    S.connected = true;
  });
}

// Profiling harness (profiles/nvlink_ncu.py): map the other ranks' pools from
// raw device pointers of THIS process (other GPUs, peer access enabled here)
// instead of IPC handles, and switch the inter-rank barriers off, so that one
// process can drive one rank's cross-round kernels under ncu without any
// kernel waiting on another GPU.  The averages it computes are meaningless.
int moshpit_shard_probe_peers(moshpit_shard* h, void* const* pools_by_rank) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    if (S.emulate) throw std::invalid_argument("shard: emulation mode has no peers");
    DeviceGuard g(S.device);
    for (std::uint32_t r = 0; r < S.world; ++r) {
      if (S.hosts(r)) continue;
      cudaPointerAttributes a{};
      MB_CUDA(cudaPointerGetAttributes(&a, pools_by_rank[r]));
      if (a.type != cudaMemoryTypeDevice) throw std::invalid_argument("probe_peers: not device memory");
      if (a.device != S.device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) MB_CUDA(e);
        cudaGetLastError();
      }
      S.pools[r] = pools_by_rank[r];
    }
    for (std::uint32_t q = 0; q < S.procs; ++q) S.peer_flags[q] = S.flags.as<unsigned long long>();
    MB_CUDA(cudaMemcpy(S.pool_tab.ptr, S.pools, sizeof(S.pools), cudaMemcpyHostToDevice));
    MB_CUDA(cudaMemcpy(S.flag_tab.ptr, S.peer_flags, sizeof(S.peer_flags),
                       cudaMemcpyHostToDevice));
    S.probe = true;
    S.connected = true;
  });
}

int moshpit_shard_fill_synthetic(moshpit_shard* h, std::uint64_t seed, void* stream) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    DeviceGuard g(S.device);
    auto s = static_cast<cudaStream_t>(stream);
    for (std::uint32_t r = S.me; r < S.me + S.nhost; ++r) {
      if (S.dtype == MOSHPIT_F32)
        shard_fill_kernel<float><<<grid_cap(S.plane->n * S.dim), 256, 0, s>>>(
            static_cast<float*>(S.pools[r]), S.loc.as<std::uint32_t>(), S.plane->n, S.dim, S.ld,
            S.R, r, seed);
      else
        shard_fill_kernel<double><<<grid_cap(S.plane->n * S.dim), 256, 0, s>>>(
            static_cast<double*>(S.pools[r]), S.loc.as<std::uint32_t>(), S.plane->n, S.dim, S.ld,
            S.R, r, seed);
      MB_LAUNCH_CHECK();
    }
  });
}

int moshpit_shard_round(moshpit_shard* h, void* stream, std::uint32_t* active_out,
                        std::int32_t* crossed_out) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    // without the peers' IPC mappings the cross round would dereference null
    // device pointers (a sticky CUDA fault); refuse instead
    if (!S.emulate && S.procs > 1 && !S.connected)
      throw std::invalid_argument("shard: open_peers not called");
    DeviceGuard g(S.device);
    int crossed = 0;
    const std::uint32_t a = S.round(static_cast<cudaStream_t>(stream), &crossed);
    if (active_out) *active_out = a;
    if (crossed_out) *crossed_out = crossed;
  });
}

// Slab pipeline: complete every round already issued on the lagging slabs and
// order `stream` after them (a no-op with slabs = 1).
int moshpit_shard_flush(moshpit_shard* h, void* stream) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    DeviceGuard g(S.device);
    S.flush(static_cast<cudaStream_t>(stream));
  });
}

// Copy the vectors of the peers resident on this process to host
// out[n*dim] by peer id; mask[p] = 1 where written.  Flushes, synchronises.
int moshpit_shard_read(moshpit_shard* h, void* out, std::uint8_t* mask) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    DeviceGuard g(S.device);
    StreamHolder st;
    if (S.S > 1) S.flush(st.s);
    const std::uint64_t n = S.plane->n;
    S.plane->sync_done();
    MB_CUDA(cudaDeviceSynchronize());
    DeviceBuffer buf(n * S.dim * S.es + 16), m(n + 16);
    std::vector<std::uint8_t> hm(n), tot(n, 0);
    for (std::uint32_t r = S.me; r < S.me + S.nhost; ++r) {
      if (S.dtype == MOSHPIT_F32)
        shard_gather_kernel<float><<<grid_cap(n * S.dim), 256, 0, st.s>>>(
            static_cast<float*>(S.pools[r]), S.loc.as<std::uint32_t>(), n, S.dim, S.ld, S.R, r,
            buf.as<float>(), m.as<std::uint8_t>(), 0);
      else
        shard_gather_kernel<double><<<grid_cap(n * S.dim), 256, 0, st.s>>>(
            static_cast<double*>(S.pools[r]), S.loc.as<std::uint32_t>(), n, S.dim, S.ld, S.R, r,
            buf.as<double>(), m.as<std::uint8_t>(), 0);
      MB_LAUNCH_CHECK();
      MB_CUDA(cudaMemcpyAsync(hm.data(), m.ptr, n, cudaMemcpyDeviceToHost, st.s));
      MB_CUDA(cudaStreamSynchronize(st.s));
      for (std::uint64_t i = 0; i < n; ++i) tot[i] |= hm[i];
    }
    MB_CUDA(cudaMemcpy(out, buf.ptr, n * S.dim * S.es, cudaMemcpyDeviceToHost));
    if (mask) std::memcpy(mask, tot.data(), n);
    std::uint32_t e = 0;
    MB_CUDA(cudaMemcpy(&e, S.err.ptr, 4, cudaMemcpyDeviceToHost));
    if (e) throw std::runtime_error("shard: placement invariant violated (code " +
                                    std::to_string(e) + ")");
  });
}

// Cross-round summation: MOSHPIT_CROSS_EXACT (default; the reference tree over
// the members' raw chunks, bit-exact) or MOSHPIT_CROSS_PARTIAL (per-GPU
// partial sums, fixed order, tolerance parity; see partial_sum_kernel).
// Applies to the rounds enqueued after the call.
int moshpit_shard_set_cross_mode(moshpit_shard* h, std::int32_t mode) {
  return guarded([&] {
    shard_require(h);
    if (mode != MOSHPIT_CROSS_EXACT && mode != MOSHPIT_CROSS_PARTIAL)
      throw std::invalid_argument("shard: unknown cross-round mode");
    if (mode == MOSHPIT_CROSS_PARTIAL && h->s->ce)
      throw std::invalid_argument("shard: the copy-engine round has no partial-sum mode");
    Shard& S = *h->s;
    S.cross_mode = mode;
    // the slab pipeline's SM split: the exact round's cross kernels are
    // NVLink-bound (~30 % of the SMs), the partial round's carry HBM-bound
    // partial sums too: the local kernels get the local rounds' share,
    // (d-1)/d of the SMs (d = 2: an even split, C2 2 GPUs 5378 -> 5758 GB/s,
    // 4 GPUs 8384 -> 8563 against 104 / 44; profiles/r02/partial/p7_sweep_*.txt)
    if (S.S > 1 && !std::getenv("MOSHPIT_PIPE_LOCAL_SMS") &&
        !std::getenv("MOSHPIT_PIPE_CROSS_SMS")) {
      const int sms = S.sm_count();
      S.pipe_local_sms = mode == MOSHPIT_CROSS_PARTIAL
                             ? (int)((std::uint64_t)sms * (S.d - 1) / std::max<std::uint32_t>(S.d, 2))
                             : (sms * 104 + 74) / 148;
      if (S.pipe_local_sms < 1) S.pipe_local_sms = sms / 2;
      S.pipe_cross_sms = sms - S.pipe_local_sms;
    }
  });
}

// Bracket the local-round and cross-round data-plane kernels with CUDA events.
int moshpit_shard_set_timing(moshpit_shard* h, std::int32_t enable) {
  return guarded([&] {
    shard_require(h);
    h->s->timing = enable != 0;
    h->s->tev_used = 0;
  });
}

// Summed device ms of the bracketed local / cross data planes since the last
// call (with slabs > 1 the slabs overlap: sums can exceed the wall time).
int moshpit_shard_kernel_time(moshpit_shard* h, double* local_ms, std::uint64_t* local_n,
                              double* cross_ms, std::uint64_t* cross_n) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    DeviceGuard g(S.device);
    double lt = 0, a = 0, b = 0;
    std::uint64_t ln = 0, cn = 0;
    for (std::size_t i = 0; i < S.tev_used; ++i) {
      MB_CUDA(cudaEventSynchronize(S.tev[i].b));
      float ms = 0;
      MB_CUDA(cudaEventElapsedTime(&ms, S.tev[i].a, S.tev[i].b));
      if (S.tev[i].kind == 0) {
        lt += ms;
        ++ln;
      } else if (S.tev[i].kind == 1) {
        a += ms;
        ++cn;
      } else {
        b += ms;
        ++cn;
      }
    }
    *local_ms = lt;
    *local_n = ln;
    *cross_ms = a + b;
    *cross_n = cn;
    S.last_a_ms = a;
    S.last_b_ms = b;
    S.tev_used = 0;
  });
}

// Cumulative counters (synchronises): cross rounds, active groups summed over
// cross rounds, and rows in non-voided local groups on rank `k` (a hosted
// rank; otherwise this process's first rank).
int moshpit_shard_stats(moshpit_shard* h, std::int32_t k, std::uint64_t* cross_rounds,
                        std::uint64_t* cross_active_groups, std::uint64_t* local_active_rows) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    DeviceGuard g(S.device);
    MB_CUDA(cudaDeviceSynchronize());
    unsigned long long t[2 * kMaxWorld + 2];
    MB_CUDA(cudaMemcpy(t, S.totals.ptr, sizeof(t), cudaMemcpyDeviceToHost));
    const std::uint32_t r = S.hosts((std::uint32_t)k) ? (std::uint32_t)k : S.me;
    *cross_rounds = t[1];
    *cross_active_groups = t[0];
    *local_active_rows = t[2 + r];
  });
}

int moshpit_shard_cross_detail(moshpit_shard* h, std::int32_t k, double* phase_a_ms,
                               double* phase_b_ms, std::uint64_t* moved_rows_in) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    DeviceGuard g(S.device);
    MB_CUDA(cudaDeviceSynchronize());
    unsigned long long t[2 * kMaxWorld + 2];
    MB_CUDA(cudaMemcpy(t, S.totals.ptr, sizeof(t), cudaMemcpyDeviceToHost));
    const std::uint32_t r = S.hosts((std::uint32_t)k) ? (std::uint32_t)k : S.me;
    *phase_a_ms = S.last_a_ms;
    *phase_b_ms = S.last_b_ms;
    *moved_rows_in = t[2 + kMaxWorld + r];
  });
}

// Device pointer / rows / stride of hosted rank k's pool (else the first).
// Host I/O of a hosted rank's pool (its R resident rows, dim coordinates
// each): the peer held by every row, and pinned-or-pageable host <-> pool
// copies on `stream` (ordered with round / flush on the same stream).
int moshpit_shard_row_peers(moshpit_shard* h, std::int32_t k, std::uint32_t* peer_of_row) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    if (!S.hosts((std::uint32_t)k)) throw std::invalid_argument("shard: rank not hosted here");
    DeviceGuard g(S.device);
    StreamHolder st;
    if (S.S > 1) S.flush(st.s);
    S.plane->sync_done();
    MB_CUDA(cudaDeviceSynchronize());
    const std::uint64_t n = S.plane->n;
    std::vector<std::uint32_t> loc(n);
    MB_CUDA(cudaMemcpy(loc.data(), S.loc.ptr, n * 4, cudaMemcpyDeviceToHost));
    for (std::uint64_t r = 0; r < S.R; ++r) peer_of_row[r] = 0xffffffffu;
    for (std::uint64_t i = 0; i < n; ++i)
      if (loc[i] / S.R == (std::uint64_t)k) peer_of_row[loc[i] % S.R] = (std::uint32_t)i;
  });
}

int moshpit_shard_load_rows(moshpit_shard* h, std::int32_t k, const void* host,
                            std::uint64_t host_ld_bytes, void* stream) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    if (!S.hosts((std::uint32_t)k)) throw std::invalid_argument("shard: rank not hosted here");
    if (host_ld_bytes < S.dim * S.es) throw std::invalid_argument("shard: host row stride");
    DeviceGuard g(S.device);
    S.copy_rows((std::uint32_t)k, const_cast<void*>(host), host_ld_bytes, false,
                static_cast<cudaStream_t>(stream));
  });
}

int moshpit_shard_store_rows(moshpit_shard* h, std::int32_t k, void* host,
                             std::uint64_t host_ld_bytes, void* stream) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    if (!S.hosts((std::uint32_t)k)) throw std::invalid_argument("shard: rank not hosted here");
    if (host_ld_bytes < S.dim * S.es) throw std::invalid_argument("shard: host row stride");
    DeviceGuard g(S.device);
    // the lagging slabs finish their rounds first, each slab's columns leave
    // as soon as its own rounds are done
    S.copy_rows((std::uint32_t)k, host, host_ld_bytes, true, static_cast<cudaStream_t>(stream));
  });
}

int moshpit_shard_pool(moshpit_shard* h, std::int32_t k, void** ptr, std::uint64_t* rows,
                       std::uint64_t* ld) {
  return guarded([&] {
    shard_require(h);
    Shard& S = *h->s;
    const std::uint32_t r = S.hosts((std::uint32_t)k) ? (std::uint32_t)k : S.me;
    *ptr = S.pools[r];
    *rows = S.R;
    *ld = S.ld;
  });
}

}  // extern "C"
