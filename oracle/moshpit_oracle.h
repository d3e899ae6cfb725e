/*
 * moshpit_oracle.h -- CPU restatement of the reference Moshpit averaging path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product path (paper_2103_03239_b200/,
 * libmoshpit_b200.so) never links or calls anything under oracle/.
 *
 * Every function restates the reference algorithm at the cited file:line
 * (paths relative to the reference's proj/include/moshpit/).  Parity is
 * pinned against the unmodified reference compiled by oracle/Makefile into
 * oracle/_ref/ (tests/test_oracle_*.py) and against the committed golden
 * vectors in tests/golden/ (generated from oracle/_ref by
 * tests/golden/gen_golden.py).
 *
 * Real-valued routines come in two instantiations: _f64 (bit-identical to the
 * reference, which is double throughout) and _f32 (same tree, same order, in
 * float: the bit-exact twin of the GPU fp32 path).
 */
#ifndef MOSHPIT_ORACLE_H
#define MOSHPIT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_OK 0
#define ORC_INVALID_ARGUMENT (-1)
#define ORC_OUT_OF_RANGE (-2)
#define ORC_RUNTIME_ERROR (-3)

/* ---- rng.hpp:12-127 ---------------------------------------------------- */
typedef struct {
  uint64_t s[4];
  int have_spare;
  double spare;
} orc_rng;

uint64_t orc_splitmix64(uint64_t* state);              /* rng.hpp:12-17 */
uint64_t orc_fnv1a(const char* s);                     /* rng.hpp:19-26 */
void orc_rng_seed(orc_rng* r, uint64_t seed);          /* rng.hpp:35-38 */
void orc_rng_stream(orc_rng* r, uint64_t root, const char* name); /* rng.hpp:118-121 */
void orc_rng_stream_idx(orc_rng* r, uint64_t root, const char* name,
                        uint64_t index);               /* rng.hpp:123-127 */
uint64_t orc_rng_next(orc_rng* r);                     /* rng.hpp:43-53 */
double orc_rng_uniform(orc_rng* r);                    /* rng.hpp:56 */
uint64_t orc_rng_below(orc_rng* r, uint64_t n);        /* rng.hpp:59-66 */
double orc_rng_normal(orc_rng* r);                     /* rng.hpp:68-83 */
int orc_rng_bernoulli(orc_rng* r, double p);           /* rng.hpp:91 */

/* Batch draws for tests: kind 0=next 1=uniform(as f64) 2=below(arg) 3=normal
 * 4=bernoulli(p=arg_f).  index < 0 selects Rng::stream(name). */
void orc_stream_draws(uint64_t root, const char* name, int64_t index, int kind,
                      uint64_t arg, double arg_f, uint64_t n, void* out);

/* counter-based synthetic init used by bench and parity tests:
 * x(i,j) = (splitmix64(seed ^ (i<<32) ^ j) >> 40) * 2^-24, exact in fp32. */
double orc_init_value(uint64_t seed, uint64_t i, uint64_t j);

/* ---- core.hpp:19-34, matchmaking.hpp:46-71 ----------------------------- */
int orc_grid_validate(uint32_t M, uint32_t d, uint32_t T);
uint64_t orc_grid_capacity(uint32_t M, uint32_t d);
int orc_initial_index(uint64_t cell, uint32_t M, uint32_t d, uint32_t* key);
int orc_next_group_key(const uint32_t* key, uint32_t klen, uint32_t chunk,
                       uint32_t M, uint32_t* out);

/* ---- matchmaking.hpp:300-323 -------------------------------------------
 * peers: ids[n], keys[n*klen] (lexicographic), ts[n].  Output members[n] in
 * group order, group_off[n_groups+1]; returns n_groups. */
int64_t orc_form_groups_uncontested(uint64_t n, const uint32_t* ids,
                                    const uint32_t* keys, uint32_t klen,
                                    const uint64_t* ts, uint32_t cap,
                                    uint32_t* members, uint32_t* group_off);

/* ---- allreduce.hpp:46-66 ----------------------------------------------- */
int orc_chunk_sizes(uint64_t dim, const double* w, uint64_t n, uint64_t* sizes);

/* ---- theory.hpp:149-155 ------------------------------------------------- */
double orc_complexity_estimate(uint32_t t, uint32_t n, uint32_t m, uint32_t dim);

/* Per-round integer trace of run_moshpit (protocols.hpp:123-170): for each
 * round r, members[r*n..], group_off[r*(n+1)..], n_groups[r], void_flag[r*n..]
 * (per group), rank[r*n..] (per peer), active[r].  keys_final[n*(d-1)]. */
int orc_moshpit_trace(uint32_t M, uint32_t d, uint64_t n, double p,
                      uint64_t seed, uint32_t rounds, uint32_t* members,
                      uint32_t* group_off, uint32_t* n_groups,
                      uint8_t* void_flag, uint32_t* rank, uint32_t* active,
                      uint32_t* keys_final, uint64_t* cells);

/* ---- real-valued routines (core.hpp, allreduce.hpp, protocols.hpp,
 *      optimizer.hpp) in two precisions. ------------------------------- */
#define ORC_DECLARE_REAL(R, SFX)                                               \
  R orc_pairwise_sum_##SFX(const R* xs, uint64_t n);                           \
  int orc_group_mean_##SFX(const R* rows, uint64_t n, uint64_t dim,            \
                           const uint32_t* members, R* out);                   \
  int orc_butterfly_##SFX(const R* inputs, uint64_t n, uint64_t dim,           \
                          const uint8_t* failed, R* out, int* completed);      \
  double orc_distortion_##SFX(const R* peers, uint64_t n, uint64_t dim,        \
                              const double* ref);                              \
  int orc_mean_of_##SFX(const R* peers, uint64_t n, uint64_t dim, R* out);     \
  int orc_run_moshpit_##SFX(uint32_t M, uint32_t d, uint32_t T,                \
                            const R* initial, uint64_t n, uint64_t dim,        \
                            double p, uint64_t seed, uint32_t rounds,          \
                            double* initial_distortion, double* distortion,    \
                            double* mean_drift, uint32_t* active,              \
                            double* cost_units, R* final_vectors);             \
  int orc_moshpit_average_##SFX(R* thetas, uint64_t n, uint64_t dim,           \
                                uint32_t M, uint32_t d, uint32_t rounds,       \
                                orc_rng* stream);                               \
  int orc_sgd_quadratic_##SFX(                                                 \
      uint32_t M, uint32_t d, uint32_t T, uint32_t n_peers, uint64_t dim,      \
      double L, double mu, const double* target, const double* theta0,         \
      double gamma, uint32_t tau, uint32_t steps, double sigma,                \
      uint32_t inner_rounds, uint64_t seed, const uint32_t* ev_step,           \
      const int32_t* ev_delta, uint64_t n_events, double* f_gap,               \
      double* grad_norm_sq, double* f_gap_weighted, double* dispersion,        \
      double* final_mean, double* diag6, R* final_thetas);

ORC_DECLARE_REAL(double, f64)
ORC_DECLARE_REAL(float, f32)

/* ---- LogisticRegression (optimizer.hpp:75-146), fp64 ---------------- */
void orc_logistic_synthetic(uint64_t dim, uint64_t samples, orc_rng* st, double* xs,
                            double* ys);
double orc_logistic_value(const double* xs, const double* ys, uint64_t samples, uint64_t dim,
                          double l2, const double* th);
void orc_logistic_gradient(const double* xs, const double* ys, uint64_t samples, uint64_t dim,
                           double l2, const double* th, double* g);
double orc_logistic_smoothness(const double* xs, uint64_t samples, uint64_t dim, double l2);
int orc_sgd_logistic_f64(uint32_t M, uint32_t d, uint32_t T, uint32_t n_peers, uint64_t dim,
                         const double* xs, const double* ys, uint64_t samples, double l2,
                         const double* theta0, double gamma, uint32_t tau, uint32_t steps,
                         double sigma, uint32_t inner_rounds, uint64_t seed,
                         double* f_gap, double* grad_norm_sq, double* f_gap_weighted,
                         double* dispersion, double* final_mean, double* diag6,
                         double* final_thetas);

#ifdef __cplusplus
}
#endif
#endif
