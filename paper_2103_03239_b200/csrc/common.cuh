// common.cuh -- shared host/device plumbing for the Moshpit B200 engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace mb200 {

// ---------------------------------------------------------------------------
// Errors: the C ABI maps these onto MOSHPIT_ERR_* (reference exception types).
// ---------------------------------------------------------------------------
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define MB_CUDA(expr)                                                        \
  do {                                                                       \
    cudaError_t mb_err_ = (expr);                                            \
    if (mb_err_ != cudaSuccess)                                              \
      throw ::mb200::CudaError(std::string(#expr) + ": " +                   \
                               cudaGetErrorString(mb_err_));                 \
  } while (0)

#define MB_LAUNCH_CHECK() MB_CUDA(cudaGetLastError())

// ---------------------------------------------------------------------------
// Host RNG -- the reference's generator (rng.hpp:12-127): splitmix64 seeding,
// xoshiro256**, fnv1a-named streams.  Draws stay on the host: they are
// sequential by construction and cost O(n) per round (hard part 6).
// ---------------------------------------------------------------------------
inline std::uint64_t splitmix64(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

inline std::uint64_t fnv1a(std::string_view s) {
  std::uint64_t h = 0xCBF29CE484222325ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001B3ULL;
  }
  return h;
}

struct Xoshiro {
  std::uint64_t s[4]{};
  bool have_spare = false;
  double spare = 0.0;

  Xoshiro() = default;
  explicit Xoshiro(std::uint64_t seed) {
    std::uint64_t sm = seed;
    for (auto& w : s) w = splitmix64(sm);
  }
  static Xoshiro named(std::uint64_t root, std::string_view name) {
    std::uint64_t mix = root ^ fnv1a(name);
    return Xoshiro(splitmix64(mix));
  }
  static Xoshiro named(std::uint64_t root, std::string_view name,
                       std::uint64_t index) {
    std::uint64_t mix = root ^ fnv1a(name);
    mix = splitmix64(mix) ^ (0x9E3779B97F4A7C15ULL * (index + 1));
    return Xoshiro(splitmix64(mix));
  }
  static std::uint64_t rotl(std::uint64_t x, int k) {
    return (x << k) | (x >> (64 - k));
  }
  std::uint64_t next() {
    const std::uint64_t result = rotl(s[1] * 5, 7) * 9;
    const std::uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  std::uint64_t below(std::uint64_t n) {
    const std::uint64_t threshold = (~n + 1) % n;
    for (;;) {
      const std::uint64_t r = next();
      if (r >= threshold) return r % n;
    }
  }
  double normal();
  bool bernoulli(double p) { return uniform() < p; }
};

// ---------------------------------------------------------------------------
// Grid arithmetic (core.hpp:19-34) and packed group keys.
// A GroupKey (d-1 chunk indices, lexicographic) is packed mixed-radix with the
// OLDEST index most significant, so numeric order == std::map<GroupKey> order
// and next_group_key (drop oldest, append rank) is (key % M^(d-2)) * M + rank.
// ---------------------------------------------------------------------------
struct Grid {
  std::uint32_t M = 1, d = 1;
  std::uint32_t klen = 0;       // d - 1
  std::uint64_t capacity = 1;   // M^d
  std::uint64_t pow_drop = 1;   // M^(d-2) (1 when d <= 2)

  Grid() = default;
  Grid(std::uint32_t M_, std::uint32_t d_) : M(M_), d(d_) {
    if (M < 1 || d < 1)
      throw std::invalid_argument("GridConfig: M, d, T must all be >= 1");
    klen = d - 1;
    capacity = 1;
    for (std::uint32_t j = 0; j < d; ++j) {
      if (capacity > (UINT64_MAX >> 1) / M)
        throw std::invalid_argument("GridConfig: M^d overflows 63 bits");
      capacity *= M;
    }
    pow_drop = 1;
    for (std::uint32_t j = 0; j + 2 < d; ++j) pow_drop *= M;
  }
  // distinct (d-1)-digit group keys, M^(d-1): a bound on any round's groups
  std::uint64_t lines() const { return capacity / M; }
  // matchmaking.hpp:46-59, packed
  std::uint64_t initial_key(std::uint64_t cell) const {
    std::uint64_t rest = cell / M, key = 0;
    for (std::uint32_t j = 1; j < d; ++j) {
      key = key * M + rest % M;
      rest /= M;
    }
    return key;
  }
  void unpack(std::uint64_t key, std::uint32_t* digits) const {
    for (std::uint32_t i = klen; i-- > 0;) {
      digits[i] = static_cast<std::uint32_t>(key % M);
      key /= M;
    }
  }
};

inline std::uint32_t ceil_div_u32(std::uint64_t a, std::uint64_t b) {
  return static_cast<std::uint32_t>((a + b - 1) / b);
}

// ---------------------------------------------------------------------------
// RAII device / pinned buffers.
// ---------------------------------------------------------------------------
struct DeviceBuffer {
  void* ptr = nullptr;
  std::size_t bytes = 0;
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t b) { resize(b); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  void resize(std::size_t b) {
    if (b <= bytes && ptr) return;
    release();
    MB_CUDA(cudaMalloc(&ptr, b ? b : 16));
    bytes = b;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

struct PinnedBuffer {
  void* ptr = nullptr;
  std::size_t bytes = 0;
  PinnedBuffer() = default;
  PinnedBuffer(const PinnedBuffer&) = delete;
  PinnedBuffer& operator=(const PinnedBuffer&) = delete;
  ~PinnedBuffer() {
    if (ptr) cudaFreeHost(ptr);
  }
  void resize(std::size_t b) {
    if (b <= bytes && ptr) return;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    MB_CUDA(cudaMallocHost(&ptr, b ? b : 16));
    bytes = b;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

// Restores the caller's current device on scope exit (torch and other
// callers keep their own notion of the current device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    MB_CUDA(cudaGetDevice(&prev));
    if (dev >= 0 && dev != prev) MB_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void require_device();  // throws CudaError when no usable device exists

// ---------------------------------------------------------------------------
// Kernel entry points (defined in the .cu files).
// ---------------------------------------------------------------------------

// Kernel 1: group formation over packed keys or digit keys.
struct GroupArgs {
  std::uint32_t n = 0;
  std::uint32_t cap = 0;
  std::uint32_t M = 1;
  std::uint64_t pow_drop = 1;   // next key = (key % pow_drop) * M + rank
  int advance_keys = 0;         // round mode: update keys in place
  int klen_zero = 0;            // d == 1: keys stay empty (0)
  std::uint64_t* keys = nullptr;          // packed keys [n] (round mode)
  const std::uint32_t* digit_keys = nullptr;  // [n*dklen] (standalone mode)
  std::uint32_t dklen = 0;
  const std::uint64_t* ts = nullptr;      // [n] 48-bit priorities
  const std::uint8_t* failed = nullptr;   // [n] or null
  const std::uint32_t* ids = nullptr;     // [n] or null (id = index)
  // outputs
  std::uint32_t* members = nullptr;  // [n]
  std::uint32_t* goff = nullptr;     // [n+1]
  std::uint8_t* gvoid = nullptr;     // [n]
  std::uint32_t* rank = nullptr;     // [n] by input index
  std::uint32_t* act = nullptr;      // [n] non-voided group ids
  std::uint32_t* counts = nullptr;   // [0]=n_groups [1]=n_act [2]=peers in act
  unsigned long long* totals = nullptr;  // [0]+=peers in act (running)
  // global scratch (used when the sort does not fit in shared memory)
  std::uint32_t* sidx = nullptr;  // [pow2(n)]
  std::uint32_t* scs = nullptr;   // [n]
  std::uint32_t* sgi = nullptr;   // [n]
  // trial batching (moshpit_run_moshpit_batch): CTA b works on trial b; every
  // per-peer array above is [batch][n] (goff [batch][n+1], counts [batch][4],
  // sidx [batch][pow2(n)]).  0 = a single trial.
  std::uint32_t batch = 0;
  // Fused narrow round (trial batching, tiny dim): after the tables, the same
  // CTA averages the non-voided groups of its trial's state rows in place --
  // kernel 2's work, same tree, same rounding.  Rows at fuse_x + t*fuse_stride
  // (elements), pitch fuse_ld, fuse_dim columns, fp64 when fuse_f64.
  void* fuse_x = nullptr;
  std::uint64_t fuse_ld = 0, fuse_dim = 0, fuse_stride = 0;
  int fuse_f64 = 0;
};

std::size_t group_smem_bytes(std::uint32_t n, bool packed);
void launch_form_groups(const GroupArgs& a, bool packed, cudaStream_t s);
// Batched kernel 2: trial t (= gridDim.y) reads state + t*state_stride and its
// own tables at members/act + t*n, goff + t*(n+1), counts + t*4.
template <typename T>
void launch_group_mean_batch(T* state, std::uint64_t state_stride, std::uint64_t ld,
                             std::uint64_t dim, std::uint32_t n, std::uint32_t trials,
                             const std::uint32_t* members, const std::uint32_t* goff,
                             const std::uint32_t* act, const std::uint32_t* counts,
                             cudaStream_t s);
void launch_initial_keys(const std::uint64_t* cells, std::uint64_t* keys,
                         std::uint64_t n, std::uint32_t M, std::uint32_t d,
                         cudaStream_t s);

// Kernel 3 prologue: the local SGD step (optimizer.hpp:356-373) applied to
// each member vector as kernel 2 loads it (row index == peer id).
template <typename T>
struct StepPrologue {
  const T* curv = nullptr;  // [ld] curvature (padded with zeros)
  const T* tgt = nullptr;   // [ld] target
  T gamma = 0;
  double coord_std = 0.0;
  int philox = 0;           // device noise (0: sigma == 0)
  std::uint64_t seed = 0, step_no = 0, dim = 0;
  std::uint32_t* nonfinite = nullptr;
  double* noise_partial = nullptr;  // [gridDim] sum of nj^2 per CTA
};

// Kernel 2: segmented group mean over the active groups (with the kernel-3
// step fused into the loads when `step` is non-null).
template <typename T>
void launch_group_mean(T* state, std::uint64_t ld, std::uint64_t dim,
                       const std::uint32_t* members, const std::uint32_t* goff,
                       const std::uint32_t* act, const std::uint32_t* counts,
                       std::uint32_t max_group, int variant, cudaStream_t s,
                       const StepPrologue<T>* step = nullptr);
int group_mean_grid_size(bool f64, bool step);
// Kernel 3 leaf-streamed form (step_kernel.cu), groups of <= 32 members.
template <typename T>
void launch_group_mean_step(T* state, std::uint64_t ld, std::uint64_t dim,
                            const std::uint32_t* members, const std::uint32_t* goff,
                            const std::uint32_t* act, const std::uint32_t* counts,
                            const StepPrologue<T>& sp, cudaStream_t s);
int group_mean_step_grid(bool f64, bool noisy);
// Several rounds in one pass over the state (fused_rounds.cu): the device
// tables of one round (kernel 1's output) ...
struct FusedRound {
  const std::uint32_t* members = nullptr;
  const std::uint32_t* goff = nullptr;
  const std::uint32_t* act = nullptr;
  const std::uint32_t* counts = nullptr;
};
// ... the most rounds one pass can hold for n peers in at most gcap groups a
// round (0: n too large, > ~1800) ...
std::uint32_t fused_rounds_max(std::uint64_t n, std::uint64_t gcap);
// ... and the pass: optional kernel-3 step, then R rounds (rounds_dev: [R]
// tables in device memory), bit-identical to kernel 3 + R - 1 kernel-2 rounds.
template <typename T>
void launch_rounds_fused(T* state, std::uint64_t ld, std::uint64_t dim, std::uint32_t n,
                         std::uint32_t gcap, const FusedRound* rounds_dev, std::uint32_t R,
                         const StepPrologue<T>* step, cudaStream_t s);
// The Moshpit-SGD averaging step with two rounds and no failures in one pass
// (step_kernel.cu): kernel 3's step + round 1 into shared memory, round 2 from
// there, one read and one write of the state; bit-identical to kernel 3 +
// kernel 2.  host_rounds: the two rounds' device tables (host array);
// g1_max >= round 1's group count, <= two_round_max_groups(); groups of <= 32.
std::uint32_t two_round_max_groups();
template <typename T>
void launch_two_round_step(T* state, std::uint64_t ld, std::uint64_t dim, std::uint32_t n,
                           const FusedRound* host_rounds, std::uint32_t g1_max,
                           std::uint32_t* grp1, std::uint32_t* src1, const StepPrologue<T>& sp,
                           cudaStream_t s);
// Kernel-2 grid cap for launches from the calling thread (0 = every SM).
void set_k2_grid_sms(int sms);
// fp32 LogisticRegression step on the tensor cores (tc_logit.cu: tcgen05
// kind::tf32, 3xTF32).  MOSHPIT_LOGIT_TC=0 keeps the fp64 SIMT kernels.
bool logit_tc_enabled(std::uint64_t dim, std::uint64_t samples);
void logit_tc_prepare(const double* xs, std::uint64_t S, std::uint64_t dim, float* x_hi,
                      float* x_lo, float* xt_hi, float* xt_lo, cudaStream_t s);
void logit_tc_step(float* theta, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                   std::uint64_t S, const float* x_hi, const float* x_lo, const float* xt_hi,
                   const float* xt_lo, const double* ys, double l2, float gamma,
                   const float* noise, double coord_std, int philox, std::uint64_t seed,
                   std::uint64_t step, std::uint32_t* nonfinite, double* nsq_out, float* th_hi,
                   float* th_lo, float* c_hi, float* c_lo, cudaStream_t s);

// Diagnostics and helpers.
// Representative rows of a round: after averaging, every member of a
// non-voided group holds the identical group mean, so per-row diagnostics
// need to read only one row per such group (plus every voided row).  rep[i]
// = the representative of row i; list[0 .. *count) = the representatives.
// Results are bit-identical to reading every row (the values are the same).
struct RepRows {
  const std::uint32_t* rep = nullptr;
  const std::uint32_t* list = nullptr;
  const std::uint32_t* count = nullptr;
};
// Noise-free Moshpit-SGD local step fused into hat theta (diag_kernel.cu):
// steps every row in place (the standalone step kernel's arithmetic) and
// writes mean_of(post) to hat.  False (nothing launched) with device noise,
// or unless n = 8 * 2^K (32 .. 4096) with 16-byte rows.
template <typename T>
bool launch_step_colmean(T* x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                         const T* curv, const T* tgt, T gamma, double coord_std, int philox,
                         std::uint64_t seed, std::uint64_t step_no, std::uint32_t* nonfinite,
                         double* noise_partial, std::uint64_t partial_slots, double* hat,
                         cudaStream_t s);
// list_voided = 0: only the averaged groups' representatives are listed
// (the voided rows are unchanged; see launch_distortion_fast_cached)
void launch_build_reps(const std::uint32_t* members, const std::uint32_t* goff,
                       const std::uint8_t* gvoid, const std::uint32_t* counts, std::uint64_t n,
                       std::uint32_t* rep, std::uint32_t* list, std::uint32_t* count,
                       cudaStream_t s, int list_voided = 1);
template <typename T, typename Acc>
void launch_colmean(const T* x, std::uint64_t n, std::uint64_t ld,
                    std::uint64_t dim, const std::uint32_t* rows, Acc* out,
                    cudaStream_t s, bool rows_optional = false);
// fp32 column means over the representative map by exact sums of the distinct
// rows (bit-identical to the tree when the column's exponent range allows,
// the tree for the other columns); false = not applicable, nothing launched.
std::size_t colsum_scratch_bytes(std::uint64_t n, std::uint64_t dim);
bool launch_colmean_exactsum(const float* x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                             const std::uint32_t* rep, double* out, void* scratch,
                             cudaStream_t s);
template <typename T>
void launch_distortion(const T* x, std::uint64_t n, std::uint64_t ld,
                       std::uint64_t dim, const double* ref, double* sq_scratch,
                       double* partial_scratch, double* out, int exact,
                       cudaStream_t s, const RepRows* reps = nullptr);
template <typename T>
void launch_distortion_fast_cached(const T* x, std::uint64_t n, std::uint64_t ld,
                                   std::uint64_t dim, const double* ref, double* sq,
                                   double* partial, double* out, cudaStream_t s,
                                   const RepRows& reps);
void launch_drift(const double* mean, const double* ref, std::uint64_t dim,
                  double* partial_scratch, double* out, int exact,
                  cudaStream_t s);
std::size_t diag_partial_elems(std::uint64_t n, std::uint64_t dim);
std::uint64_t diag_chunk();
// Slab-streamed diagnostics: j-sums that continue across D-slabs (EXACT:
// per-peer / scalar running accumulators; FAST: chunk partials at global
// chunk offset c0), then one finishing pass.
template <typename T>
void launch_dist_slab(const T* x, std::uint64_t n, std::uint64_t ld, std::uint64_t dim,
                      const double* ref, int exact, double* acc, double* partial,
                      std::uint64_t nch_total, std::uint64_t c0, cudaStream_t s,
                      const RepRows* reps = nullptr);
void launch_drift_slab(const double* mean, const double* ref, std::uint64_t dim, int exact,
                       double* acc2, double* partial, std::uint64_t c0, cudaStream_t s);
void launch_diag_finish(std::uint64_t n, std::uint64_t nch_total, int exact, double* acc,
                        double* row_partial, double* acc2, double* drift_partial,
                        double* dist_out, double* drift_out, cudaStream_t s,
                        const std::uint32_t* rep = nullptr);
template <typename T>
void launch_fill_synthetic(T* x, std::uint64_t n, std::uint64_t dim,
                           std::uint64_t ld, std::uint64_t seed,
                           std::uint64_t col0, cudaStream_t s);
template <typename T>
void launch_broadcast_rows(T* dst, std::uint64_t ld, const T* row,
                           std::uint64_t n, std::uint64_t dim, cudaStream_t s);

}  // namespace mb200
