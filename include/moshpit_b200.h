/*
 * moshpit_b200.h -- C ABI of the B200-native Moshpit averaging engine.
 *
 * The reference (arXiv 2103.03239 "moshpit-lab", proj/include/moshpit/) is a
 * header-only C++20 library with no FFI: its drop-in boundary is the header
 * API.  Each entry point below replaces one reference function (cited
 * file:line, relative to proj/include/moshpit/); the C++ header
 * include/moshpit_b200/moshpit.hpp re-exposes them under the reference's own
 * namespaces, signatures and exception types, and INTEGRATION.md shows the
 * bindings (C++ header swap, Python ctypes) a maintainer would add.
 *
 * Conventions
 *  - plain pointers and sizes only; no torch / CUDA types in signatures
 *    (CUDA streams travel as `void*` = cudaStream_t, device buffers as void*);
 *  - every function returns MOSHPIT_OK (0) or a negative status whose class
 *    maps 1:1 onto the reference's exception types; moshpit_last_error()
 *    returns the message (thread-local);
 *  - reentrant: no global mutable state besides the thread-local message;
 *    one moshpit_engine per calling thread;
 *  - compute entry points run on the GPU (sm_100a kernels).  There is no CPU
 *    fallback: without a usable device they return MOSHPIT_ERR_CUDA.
 *    Pure-host helpers (rng, key arithmetic) are marked [host].
 */
#ifndef MOSHPIT_B200_H
#define MOSHPIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOSHPIT_OK 0
#define MOSHPIT_ERR_INVALID_ARGUMENT (-1) /* std::invalid_argument */
#define MOSHPIT_ERR_OUT_OF_RANGE (-2)     /* std::out_of_range */
#define MOSHPIT_ERR_RUNTIME (-3)          /* std::runtime_error */
#define MOSHPIT_ERR_CUDA (-4)             /* device / driver failure */

#define MOSHPIT_F32 0 /* peer state in float (performance path) */
#define MOSHPIT_F64 1 /* peer state in double (bit parity with the reference) */

/* TrialReport diagnostics (protocols.hpp:68-84 record_round). */
#define MOSHPIT_DIAG_NONE 0  /* skip: the averaging round alone */
#define MOSHPIT_DIAG_FAST 1  /* fixed-order blocked fp64 sums (tolerance) */
#define MOSHPIT_DIAG_EXACT 2 /* the reference's summation order (bit parity) */

/* Group-mean kernel variants. */
#define MOSHPIT_KERNEL_AUTO 0
#define MOSHPIT_KERNEL_REGISTER 1 /* 128-bit LDG/STG, tree in registers */
#define MOSHPIT_KERNEL_BULK 2     /* cp.async.bulk (TMA) ring through smem */

const char* moshpit_last_error(void);
const char* moshpit_version(void);
/* Number of visible CUDA devices (0 when none). [host] */
int moshpit_device_count(int* out);

/* ---- RNG: rng.hpp:31-127 (xoshiro256**, splitmix64 seeding, fnv1a names) */
typedef struct {
  uint64_t s[4];
  int32_t have_spare;
  double spare;
} moshpit_rng_state;

/* Rng(root).stream(name) (rng.hpp:118-121) or .stream(name, index)
 * (rng.hpp:123-127) when index >= 0. [host] */
int moshpit_rng_stream(uint64_t root, const char* name, int64_t index,
                       moshpit_rng_state* out);
/* RngStream(seed) (rng.hpp:35-38): four splitmix64 words of `seed`. [host] */
int moshpit_rng_seeded(uint64_t seed, moshpit_rng_state* out);
/* n draws: kind 0=operator() (u64) 1=uniform (f64) 2=below(arg) (u64)
 * 3=normal (f64) 4=bernoulli(p) (u8).  rng.hpp:43-91. [host] */
int moshpit_rng_draws(moshpit_rng_state* st, int kind, uint64_t arg, double p,
                      uint64_t n, void* out);

/* ---- grid and keys: core.hpp:19-34, matchmaking.hpp:46-71 [host] ------ */
int moshpit_grid_validate(uint32_t M, uint32_t d, uint32_t T);
uint64_t moshpit_grid_capacity(uint32_t M, uint32_t d);
/* matchmaking.hpp:46 initial_index; key_out has d-1 entries. */
int moshpit_initial_index(uint64_t cell, uint32_t M, uint32_t d,
                          uint32_t* key_out);
/* matchmaking.hpp:62 next_group_key. */
int moshpit_next_group_key(const uint32_t* key, uint32_t klen, uint32_t chunk,
                           uint32_t M, uint32_t* key_out);
/* allreduce.hpp:46-66 chunk_sizes (largest remainder). */
int moshpit_chunk_sizes(uint64_t dim, const double* weights, uint64_t n,
                        uint64_t* sizes_out);
/* theory.hpp:149-155 complexity_estimate. */
double moshpit_complexity_estimate(uint32_t t, uint32_t n, uint32_t m,
                                   uint32_t dim);

/* ---- matchmaking.hpp:300-323 form_groups_uncontested  [GPU kernel 1] ----
 * Peers: ids[n], keys[n*klen] (GroupKey digits, lexicographic), timestamps[n].
 * Output: members_out[n] (peer ids in group order), group_off_out[g..g+1]
 * bounds group g (n+1 entries reserved), *n_groups_out. */
int moshpit_form_groups_uncontested(uint64_t n, const uint32_t* ids,
                                    const uint32_t* keys, uint32_t klen,
                                    const uint64_t* timestamps, uint32_t cap,
                                    uint32_t* members_out,
                                    uint32_t* group_off_out,
                                    uint64_t* n_groups_out);

/* ---- numerics on host buffers  [GPU kernel 2 and diagnostics] ---------- */
/* core.hpp:91-106 group_mean over rows[members[k]] (members NULL = 0..n-1). */
int moshpit_group_mean(int dtype, const void* rows, uint64_t n_rows,
                       uint64_t dim, const uint32_t* members, uint64_t n,
                       void* mean_out);
/* allreduce.hpp:79-121 butterfly_allreduce (weights only validated: the
 * mean is partition-invariant, allreduce.hpp:104-105). */
int moshpit_butterfly_allreduce(int dtype, const void* inputs, uint64_t n,
                                uint64_t dim, const double* weights,
                                uint64_t n_weights, const uint8_t* failed,
                                void* vectors_out, uint32_t* chunks_out,
                                int32_t* completed_out);
/* core.hpp:111-126 distortion (ref in double), core.hpp:128-133 mean_of. */
int moshpit_distortion(int dtype, const void* peers, uint64_t n, uint64_t dim,
                       const double* reference_mean, double* out);
int moshpit_mean_of(int dtype, const void* peers, uint64_t n, uint64_t dim,
                    void* mean_out);

/* ---- protocols.hpp:108-179 run_moshpit  [GPU, host buffers] ------------
 * initial: n*dim (dtype).  Report arrays have `rounds` entries.  final_out
 * (nullable) receives the vectors after the last round (run_moshpit itself
 * never returns them).  diag: MOSHPIT_DIAG_*.  T is GridConfig::rounds. */
int moshpit_run_moshpit(int dtype, uint32_t M, uint32_t d, uint32_t T,
                        const void* initial, uint64_t n, uint64_t dim,
                        double p_round, uint64_t seed, uint32_t rounds,
                        int diag, double* initial_distortion,
                        double* distortion, double* mean_drift,
                        uint32_t* active_counts, double* cost_units,
                        void* final_out);
/* The same with the initial state given as n row pointers (each `dim`
 * elements, e.g. the data() of a std::vector<ParamVector>): no flattened copy;
 * large states are packed slab by slab into a pinned staging ring by host
 * threads (MOSHPIT_HOST_THREADS, default all cores) while the GPU runs the
 * previous slab.  Returns the report only, as protocols::run_moshpit does.
 * [GPU, host buffers] */
int moshpit_run_moshpit_rows(int dtype, uint32_t M, uint32_t d, uint32_t T,
                             const void* const* rows, uint64_t n, uint64_t dim,
                             double p_round, uint64_t seed, uint32_t rounds,
                             int diag, double* initial_distortion,
                             double* distortion, double* mean_drift,
                             uint32_t* active_counts, double* cost_units);
/* run_moshpit keeps a grow-only per-thread device workspace (slab ring of up
 * to 3 x 256 MB, round tables, diagnostics buffers, streams) so repeated calls
 * from one thread allocate nothing.  This frees the CALLING thread's
 * workspace; call it before a long-lived worker thread goes idle. [GPU] */
int moshpit_release_workspace(void);

/* ---- one round over an externally formed group table  [GPU] -------------
 * For callers that form groups themselves, e.g. the reference's contested
 * matchmaking::form_groups / GroupFormation with FailStop injections
 * (matchmaking.hpp:104-294, 325-333), which stays on the CPU: group g is
 * members[group_off[g] .. group_off[g+1]) (row indices in the group's
 * priority order = the reference's SealedGroup::members), void_flags[g] != 0
 * voids it (inputs kept, allreduce.hpp:95-102); every other group's rows get
 * the butterfly_allreduce mean (reference pairwise tree, allreduce.hpp:79-121).
 * Groups must be non-empty and disjoint.  The device form is async on
 * `stream` (state: n_rows x ld, 16-byte aligned); the host form copies in and
 * out and synchronises. */
int moshpit_round_from_groups(int dtype, void* state, uint64_t n_rows, uint64_t dim,
                              uint64_t ld, const uint32_t* members,
                              const uint32_t* group_off, uint64_t n_groups,
                              const uint8_t* void_flags, void* stream);
int moshpit_round_from_groups_host(int dtype, void* vectors, uint64_t n_rows,
                                   uint64_t dim, const uint32_t* members,
                                   const uint32_t* group_off, uint64_t n_groups,
                                   const uint8_t* void_flags);

/* ---- trial-batched run_moshpit (harness.hpp:157-280 sweeps)  [GPU] ------
 * `trials` independent protocols::run_moshpit calls in one batch: trial t
 * uses initial + t*n*dim and Rng(seeds[t]); reports are [trials] and
 * [trials][rounds]; diagnostics in the reference order unless DIAG_NONE.
 * n <= 8192, trials <= 65535. */
int moshpit_run_moshpit_batch(int dtype, uint32_t M, uint32_t d, uint32_t T,
                              uint32_t trials, const void* initial, uint64_t n,
                              uint64_t dim, double p_round, const uint64_t* seeds,
                              uint32_t rounds, int diag, double* initial_distortion,
                              double* distortion, double* mean_drift,
                              uint32_t* active_counts, double* cost_units,
                              void* final_out);
/* harness.hpp:145-155 trial_rng: root seed of trial `seed_index` of a sweep
 * cell (protocol name as protocols::to_string). [host] */
uint64_t moshpit_trial_seed(uint64_t seed_base, const char* protocol, uint32_t n,
                            double p, uint32_t seed_index);

/* ---- optimizer.hpp:249-284 detail::moshpit_average  [GPU, host buffers]
 * thetas (n*dim, dtype) averaged in place; *stream advanced exactly as the
 * reference advances its RngStream. */
int moshpit_moshpit_average(int dtype, void* thetas, uint64_t n, uint64_t dim,
                            uint32_t M, uint32_t d, uint32_t rounds,
                            moshpit_rng_state* stream);

/* ---- optimizer.hpp:231-242 local_step, Quadratic objective  [GPU] --------
 * Quadratic(dim, L, mu, target) (optimizer.hpp:31-72); the noise is drawn
 * from *noise exactly as the reference draws it; theta (host, dtype) is
 * updated in place.  runtime_error on a non-finite gradient. */
int moshpit_local_step_quadratic(int dtype, void* theta, uint64_t dim, double L,
                                 double mu, const double* target, double gamma,
                                 double sigma, moshpit_rng_state* noise);

/* ---- optimizer.hpp:297-439 run_moshpit_sgd, Quadratic objective [GPU] ----
 * Schedule: n_events MembershipEvent{ev_step[e], ev_delta[e]}.  diag:
 * MOSHPIT_DIAG_EXACT (reference summation order) or MOSHPIT_DIAG_FAST.
 * noise_mode 0: the reference's "noise" stream (host draws, bit-exact);
 * 1: device Philox4x32-10 normals (statistical parity, the fast path).
 * Outputs: f_gap, grad_norm_sq, f_gap_weighted, dispersion [steps];
 * final_mean [dim]; diag6 = {delta_aq_hat, sigma_hat, delta_pv1_hat,
 * delta_pv2_hat, n_min, n_final}; final_thetas (nullable, n_final*dim).
 * MOSHPIT_DIAG_NONE runs kernel 3 (the step fused into averaging round 1)
 * and reports NaN diagnostics. */
int moshpit_run_moshpit_sgd_quadratic(
    int dtype, uint32_t M, uint32_t d, uint32_t T, uint32_t n_peers,
    uint64_t dim, double L, double mu, const double* target,
    const double* theta0, double gamma, uint32_t tau, uint32_t steps,
    double sigma, uint32_t inner_rounds, uint64_t seed, const uint32_t* ev_step,
    const int32_t* ev_delta, uint64_t n_events, int diag, int noise_mode,
    double* f_gap, double* grad_norm_sq, double* f_gap_weighted,
    double* dispersion, double* final_mean, double* diag6, void* final_thetas,
    double* loop_ms);
/* loop_ms (nullable): device time of the step loop (CUDA events on the call's
 * stream; excludes setup and the final copies). */

/* ---- optimizer.hpp:75-146 LogisticRegression ----------------------------
 * Dataset: xs [samples x dim] row-major fp64, ys [samples] in {-1, +1}.
 * moshpit_logistic_synthetic replaces LogisticRegression::synthetic
 * (optimizer.hpp:89-104): draws from *stream exactly as the reference (host).
 * moshpit_logistic_eval replaces value()/gradient()/smoothness()
 * (optimizer.hpp:106-140) [GPU; value and gradient in the reference's
 * summation orders, exp/log1p from CUDA's libdevice -- see DESIGN.md]. */
int moshpit_logistic_synthetic(uint64_t dim, uint64_t samples,
                               moshpit_rng_state* stream, double* xs, double* ys);
int moshpit_logistic_eval(const double* xs, const double* ys, uint64_t samples,
                          uint64_t dim, double l2, const double* theta,
                          double* value, double* grad, double* smoothness);
/* optimizer.hpp:231-242 local_step with LogisticRegression [GPU]. */
int moshpit_local_step_logistic(int dtype, void* theta, uint64_t dim,
                                const double* xs, const double* ys,
                                uint64_t samples, double l2, double gamma,
                                double sigma, moshpit_rng_state* noise);
/* optimizer.hpp:297-439 run_moshpit_sgd with LogisticRegression(xs, ys, l2)
 * [GPU]: arguments and outputs as moshpit_run_moshpit_sgd_quadratic.  diag
 * NONE skips the per-step diagnostics (NaN); EXACT evaluates all of them in
 * the reference's order; FAST differs only in the dispersion V_k (fixed-order
 * block partials).  mu = l2 (strong_convexity, :141). */
int moshpit_run_moshpit_sgd_logistic(
    int dtype, uint32_t M, uint32_t d, uint32_t T, uint32_t n_peers,
    uint64_t dim, const double* xs, const double* ys, uint64_t samples,
    double l2, const double* theta0, double gamma, uint32_t tau,
    uint32_t steps, double sigma, uint32_t inner_rounds, uint64_t seed,
    const uint32_t* ev_step, const int32_t* ev_delta, uint64_t n_events,
    int diag, int noise_mode, double* f_gap, double* grad_norm_sq,
    double* f_gap_weighted, double* dispersion, double* final_mean,
    double* diag6, void* final_thetas, double* loop_ms);

/* ---- device-resident engine (the performance boundary) -----------------
 * One engine = one trial's integer plane (grid, keys, rng streams, group
 * tables) resident on `device`.  The peer state is caller-owned device
 * memory: n rows of `ld` elements (ld >= dim, ld*elem % 16 == 0, base 16-byte
 * aligned); columns [dim, round_up(dim, 16/elem)) are scratch. */
typedef struct moshpit_engine moshpit_engine;

/* Protocol mode: streams "cells", "failures", "priorities" of Rng(seed),
 * exactly as run_moshpit (protocols.hpp:123-140). */
int moshpit_engine_create(uint32_t M, uint32_t d, uint64_t n, double p_round,
                          uint64_t seed, int device, moshpit_engine** out);
int moshpit_engine_destroy(moshpit_engine* e);
/* Select MOSHPIT_KERNEL_* for the group mean. */
int moshpit_engine_set_kernel(moshpit_engine* e, int variant);
/* Enqueue one round on `stream` (cudaStream_t; NULL = legacy default):
 * draw failures + priorities on the host, group on the GPU (kernel 1),
 * average non-voided groups in place (kernel 2), advance keys.  Does not
 * synchronise.  *active_out (nullable) = peers that did not fail. */
int moshpit_engine_round(moshpit_engine* e, int dtype, void* state,
                         uint64_t dim, uint64_t ld, void* stream,
                         uint32_t* active_out);
/* `rounds` rounds in ONE pass over the state (temporal blocking over column
 * tiles; n <= 1800 peers): the same draws, groups and bits as `rounds` calls
 * of moshpit_engine_round, 2 * n * dim * elem bytes of HBM traffic per pass
 * of up to ~12 rounds (n = 1024) instead of per round -- a separate mode,
 * not the per-round path.  active_out (nullable) = [rounds] non-failed
 * peers.  Enqueued on `stream`, no synchronisation. */
int moshpit_engine_rounds_fused(moshpit_engine* e, int dtype, void* state,
                                uint64_t dim, uint64_t ld, uint32_t rounds,
                                void* stream, uint32_t* active_out);
/* Synchronise the engine's last stream and report how many rounds ran and
 * how many peer rows sat in non-voided groups, summed over those rounds.
 * Algorithmic HBM bytes of kernel 2 = 2 * elem * dim * active_rows_total. */
int moshpit_engine_stats(moshpit_engine* e, uint64_t* rounds,
                         uint64_t* active_rows_total);
/* Bracket every kernel-2 launch with CUDA events on its launch stream
 * (enable=1), and read back the summed device time of the bracketed launches
 * since the last read (synchronises on the events). */
int moshpit_engine_set_timing(moshpit_engine* e, int enable);
int moshpit_engine_kernel_time(moshpit_engine* e, double* total_ms,
                               uint64_t* launches);
/* Device-resident record_round (protocols.hpp:68-84) for engine callers.
 * set_reference: reference = mean_of(state) in fp64 (protocols.hpp:119) and
 * the initial distortion, diag = MOSHPIT_DIAG_FAST or _EXACT (NONE disables).
 * record: after a round, append (distortion, mean_drift) to an engine-owned
 * device log; the distortion and colmean + drift run on two streams.  Both
 * are async on `stream`.  report: copy the log out (synchronises); count =
 * records so far. */
int moshpit_engine_set_reference(moshpit_engine* e, int dtype, const void* state,
                                 uint64_t dim, uint64_t ld, int diag, void* stream);
int moshpit_engine_record(moshpit_engine* e, int dtype, const void* state,
                          uint64_t dim, uint64_t ld, void* stream);
/* A round and its record_round in one call: the diagnostics then read one
 * representative row per averaged group (all its members hold the same
 * mean) -- the same bits as moshpit_engine_round + moshpit_engine_record,
 * fewer HBM bytes. */
int moshpit_engine_round_record(moshpit_engine* e, int dtype, void* state,
                                uint64_t dim, uint64_t ld, void* stream,
                                uint32_t* active_out);
/* `rounds` x (round + record_round) in one call on device-resident state
 * (the protocols::run_moshpit loop, protocols.hpp:142-173).  Nothing else
 * touches the state between the rounds of one call, so with
 * MOSHPIT_DIAG_FAST the voided groups' rows keep their cached FAST row
 * partials and only the averaged groups' representative rows are re-read;
 * the TrialReport bits equal `rounds` moshpit_engine_round_record calls.
 * active_out: [rounds] non-failed peers per round (optional). */
int moshpit_engine_rounds_record(moshpit_engine* e, int dtype, void* state,
                                 uint64_t dim, uint64_t ld, uint32_t rounds,
                                 void* stream, uint32_t* active_out);
int moshpit_engine_report(moshpit_engine* e, double* initial_distortion,
                          double* distortion, double* mean_drift, uint64_t cap,
                          uint64_t* count);
/* Copy the last round's group tables to host (synchronises the engine's
 * last stream): members[n], group_off[n+1], *n_groups, void_flags[n] (per
 * group), ranks[n] (per peer), keys[n*(d-1)] (keys after the round). */
int moshpit_engine_tables(moshpit_engine* e, uint32_t* members,
                          uint32_t* group_off, uint32_t* n_groups,
                          uint8_t* void_flags, uint32_t* ranks, uint32_t* keys);

/* ---- peer-sharded multi-GPU rounds ---------------------------
 * One rank per GPU (or, with emulate=1, all `world` ranks as separate pools
 * on the current device -- a 1-GPU test harness for the same data plane).
 * Peers sit cell-major with grid digit d-1 split across ranks; rounds on axes
 * 0..d-2 are GPU-local, the axis-(d-1) round runs one fused kernel that reads
 * and writes member rows in peer HBM over NVLink.  Requires a full grid
 * (N == M^d), world | M, M <= 32.  Every rank makes the same host draws and
 * computes the same tables (no metadata exchange). */
typedef struct moshpit_shard moshpit_shard;
int moshpit_shard_create(int dtype, uint32_t M, uint32_t d, uint64_t n,
                         double p_round, uint64_t seed, uint64_t dim,
                         int32_t rank, int32_t world, int32_t emulate,
                         int32_t device, moshpit_shard** out);
/* General form: this process hosts ranks [first_rank, first_rank+ranks_here)
 * (ranks_here | world, aligned; 1 = one rank per GPU, world = the 1-GPU
 * emulation), and the columns run as `slabs` (1..8) pipelined slabs one round
 * apart on separate streams, so cross rounds (NVLink) of one slab overlap
 * local rounds (HBM) of the others; results are bit-identical to slabs = 1. */
int moshpit_shard_create_ex(int dtype, uint32_t M, uint32_t d, uint64_t n,
                            double p_round, uint64_t seed, uint64_t dim,
                            int32_t first_rank, int32_t ranks_here, int32_t world,
                            int32_t slabs, int32_t device, moshpit_shard** out);
int moshpit_shard_destroy(moshpit_shard* s);
/* ranks_here * 128 bytes: per hosted rank, the cudaIpcMemHandle_t of its row
 * pool and of this process's barrier flags. */
int moshpit_shard_ipc_handles(moshpit_shard* s, void* out);
/* world*128 bytes gathered in rank order; maps every peer's pool/flags. */
int moshpit_shard_open_peers(moshpit_shard* s, const void* all_handles);
/* PROFILING ONLY: take the other ranks' pools as device pointers of this
 * process (peer access enabled) and disable the inter-rank barriers, so one
 * process can run one rank's cross-round kernels under ncu (NVLink counters)
 * without waiting on other GPUs.  The averages are not valid. */
int moshpit_shard_probe_peers(moshpit_shard* s, void* const* pools_by_rank);
/* slabs > 1: finish the lagging slabs' rounds and order `stream` after them
 * (the state is complete only after a flush; read() flushes). */
int moshpit_shard_flush(moshpit_shard* s, void* stream);
/* Synthetic init of the resident peers' rows (x(peer, j), as fill_synthetic). */
int moshpit_shard_fill_synthetic(moshpit_shard* s, uint64_t seed, void* stream);
/* Enqueue one round (all ranks must call it the same number of times). */
int moshpit_shard_round(moshpit_shard* s, void* stream, uint32_t* active_out,
                        int32_t* crossed_out);
/* Resident peers' vectors -> out[n*dim] by peer id, mask[p]=1 where written. */
int moshpit_shard_read(moshpit_shard* s, void* out, uint8_t* mask);
/* Cross-round summation (rounds enqueued after the call):
 * MOSHPIT_CROSS_EXACT (default) evaluates the reference tree
 * (allreduce.hpp:79-121 over core.hpp:72-81) on the members' raw chunks,
 * pulled over NVLink -- bit-exact; MOSHPIT_CROSS_PARTIAL sums each GPU's
 * members first and moves one partial row per GPU and group (2(w-1)/w rows
 * of NVLink ingress per group instead of ((M-Mg)+(w-1))/w), combined in a
 * fixed rank order in fp64 -- deterministic, within 1e-6 relative of the
 * reference order in fp32 (north_star's tolerance where the summation order
 * is not matched).  Group formation, failures and placement are unchanged. */
#define MOSHPIT_CROSS_EXACT 0
#define MOSHPIT_CROSS_PARTIAL 1
int moshpit_shard_set_cross_mode(moshpit_shard* s, int32_t mode);
int moshpit_shard_set_timing(moshpit_shard* s, int32_t enable);
int moshpit_shard_kernel_time(moshpit_shard* s, double* local_ms,
                              uint64_t* local_n, double* cross_ms,
                              uint64_t* cross_n);
/* Cumulative counters (synchronises): cross rounds run, non-voided groups
 * summed over cross rounds, rows in non-voided local groups on rank k (own
 * rank in real mode) -- the algorithmic-byte accounting of the bench. */
int moshpit_shard_stats(moshpit_shard* s, int32_t k, uint64_t* cross_rounds,
                        uint64_t* cross_active_groups,
                        uint64_t* local_active_rows);
int moshpit_shard_pool(moshpit_shard* s, int32_t k, void** ptr, uint64_t* rows,
                       uint64_t* ld);
/* Host I/O of hosted rank k's pool (its R resident rows of dim elements):
 * peer_of_row[R] = the peer each row holds (0xffffffff: none; synchronises),
 * and host <-> pool copies of the R rows (host rows host_ld_bytes apart;
 * pinned host memory for full PCIe rate), after the prior work on `stream`.
 * With the slab pipeline (slabs > 1) each column slab moves on its own
 * stream: a load overlaps the first slabs' rounds (the shard's later rounds,
 * stores and reads are ordered after it; `stream` itself passes it at the
 * next flush / store_rows), a store finishes the lagging slabs' rounds and
 * lets each slab's columns leave as soon as its rounds are done; `stream`
 * waits for the whole store.  The multi-GPU end-to-end path: each process
 * loads its own peers, runs the rounds, stores them back. */
int moshpit_shard_row_peers(moshpit_shard* s, int32_t k, uint32_t* peer_of_row);
int moshpit_shard_load_rows(moshpit_shard* s, int32_t k, const void* host,
                            uint64_t host_ld_bytes, void* stream);
int moshpit_shard_store_rows(moshpit_shard* s, int32_t k, void* host,
                             uint64_t host_ld_bytes, void* stream);
/* Cross-round detail (synchronises): device ms of phase A (chunk means +
 * voided-row pulls) and phase B (mean-chunk pulls + voided-row writes) as
 * split by the last moshpit_shard_kernel_time call, and the cumulative
 * number of voided-group rows that moved INTO rank k (each one row of dim
 * elements over NVLink -- part of the cross round's minimal traffic). */
int moshpit_shard_cross_detail(moshpit_shard* s, int32_t k, double* phase_a_ms,
                               double* phase_b_ms, uint64_t* moved_rows_in);

/* Counter-based synthetic init (bench / tests):
 * x(i,j) = (splitmix64(seed ^ (i<<32) ^ (col0+j)) >> 40) * 2^-24. */
int moshpit_fill_synthetic(int dtype, void* state, uint64_t n, uint64_t dim,
                           uint64_t ld, uint64_t seed, uint64_t col0,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOSHPIT_B200_H */
