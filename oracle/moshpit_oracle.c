/*
 * moshpit_oracle.c -- CPU restatement of the reference Moshpit averaging path.
 * TEST INFRASTRUCTURE ONLY (see moshpit_oracle.h).  File:line citations are
 * relative to the reference's proj/include/moshpit/.
 *
 * Built with -ffp-contract=off so that every a*b+c stays two roundings, as in
 * the reference compiled for baseline x86-64 (no FMA).
 */
#include "moshpit_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* RNG: rng.hpp                                                              */
/* ------------------------------------------------------------------------ */

/* rng.hpp:12-17 */
uint64_t orc_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* rng.hpp:19-26 */
uint64_t orc_fnv1a(const char* s) {
  uint64_t h = 0xCBF29CE484222325ULL;
  for (const unsigned char* c = (const unsigned char*)s; *c; ++c) {
    h ^= *c;
    h *= 0x100000001B3ULL;
  }
  return h;
}

/* rng.hpp:35-38: four splitmix64 draws seed the xoshiro state */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  uint64_t sm = seed;
  for (int k = 0; k < 4; ++k) r->s[k] = orc_splitmix64(&sm);
  r->have_spare = 0;
  r->spare = 0.0;
}

/* rng.hpp:118-121 */
void orc_rng_stream(orc_rng* r, uint64_t root, const char* name) {
  uint64_t mix = root ^ orc_fnv1a(name);
  orc_rng_seed(r, orc_splitmix64(&mix));
}

/* rng.hpp:123-127 */
void orc_rng_stream_idx(orc_rng* r, uint64_t root, const char* name,
                        uint64_t index) {
  uint64_t mix = root ^ orc_fnv1a(name);
  mix = orc_splitmix64(&mix) ^ (0x9E3779B97F4A7C15ULL * (index + 1));
  orc_rng_seed(r, orc_splitmix64(&mix));
}

static inline uint64_t rotl64(uint64_t x, int k) {
  return (x << k) | (x >> (64 - k));
}

/* rng.hpp:43-53, xoshiro256** */
uint64_t orc_rng_next(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

/* rng.hpp:56 */
double orc_rng_uniform(orc_rng* r) {
  return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:59-66: rejection threshold (2^64 - n) mod n */
uint64_t orc_rng_below(orc_rng* r, uint64_t n) {
  const uint64_t threshold = (~n + 1) % n;
  for (;;) {
    const uint64_t x = orc_rng_next(r);
    if (x >= threshold) return x % n;
  }
}

/* rng.hpp:68-83, polar method with one spare */
double orc_rng_normal(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u, v, r2;
  do {
    u = 2.0 * orc_rng_uniform(r) - 1.0;
    v = 2.0 * orc_rng_uniform(r) - 1.0;
    r2 = u * u + v * v;
  } while (r2 >= 1.0 || r2 == 0.0);
  const double f = sqrt(-2.0 * log(r2) / r2);
  r->spare = v * f;
  r->have_spare = 1;
  return u * f;
}

/* rng.hpp:91 */
int orc_rng_bernoulli(orc_rng* r, double p) { return orc_rng_uniform(r) < p; }

void orc_stream_draws(uint64_t root, const char* name, int64_t index, int kind,
                      uint64_t arg, double arg_f, uint64_t n, void* out) {
  orc_rng r;
  if (index < 0)
    orc_rng_stream(&r, root, name);
  else
    orc_rng_stream_idx(&r, root, name, (uint64_t)index);
  for (uint64_t i = 0; i < n; ++i) {
    switch (kind) {
      case 0: ((uint64_t*)out)[i] = orc_rng_next(&r); break;
      case 1: ((double*)out)[i] = orc_rng_uniform(&r); break;
      case 2: ((uint64_t*)out)[i] = orc_rng_below(&r, arg); break;
      case 3: ((double*)out)[i] = orc_rng_normal(&r); break;
      default: ((uint8_t*)out)[i] = (uint8_t)orc_rng_bernoulli(&r, arg_f); break;
    }
  }
}

double orc_init_value(uint64_t seed, uint64_t i, uint64_t j) {
  uint64_t s = seed ^ (i << 32) ^ j;
  return (double)(orc_splitmix64(&s) >> 40) * 0x1.0p-24;
}

/* ------------------------------------------------------------------------ */
/* Grid and keys: core.hpp:19-34, matchmaking.hpp:46-71                      */
/* ------------------------------------------------------------------------ */

int orc_grid_validate(uint32_t M, uint32_t d, uint32_t T) {
  return (M < 1 || d < 1 || T < 1) ? ORC_INVALID_ARGUMENT : ORC_OK;
}

uint64_t orc_grid_capacity(uint32_t M, uint32_t d) {
  uint64_t cap = 1;
  for (uint32_t j = 0; j < d; ++j) cap *= M;
  return cap;
}

/* matchmaking.hpp:46-59: key[j-1] = floor(cell / M^j) mod M, j = 1..d-1 */
int orc_initial_index(uint64_t cell, uint32_t M, uint32_t d, uint32_t* key) {
  if (orc_grid_validate(M, d, 1)) return ORC_INVALID_ARGUMENT;
  if (cell >= orc_grid_capacity(M, d)) return ORC_OUT_OF_RANGE;
  uint64_t rest = cell / M;
  for (uint32_t j = 1; j < d; ++j) {
    key[j - 1] = (uint32_t)(rest % M);
    rest /= M;
  }
  return ORC_OK;
}

/* matchmaking.hpp:62-71: drop the oldest index, append the new chunk */
int orc_next_group_key(const uint32_t* key, uint32_t klen, uint32_t chunk,
                       uint32_t M, uint32_t* out) {
  if (chunk >= M) return ORC_OUT_OF_RANGE;
  if (klen == 0) return ORC_OK;
  for (uint32_t i = 0; i + 1 < klen; ++i) out[i] = key[i + 1];
  out[klen - 1] = chunk;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* form_groups_uncontested: matchmaking.hpp:300-323                          */
/* ------------------------------------------------------------------------ */

typedef struct {
  const uint32_t* ids;
  const uint32_t* keys;
  uint32_t klen;
  const uint64_t* ts;
} grp_ctx;

/* std::map<GroupKey> order (lexicographic), then Priority{timestamp, id};
 * input position breaks exact ties deterministically. */
static int grp_less(const grp_ctx* c, uint64_t a, uint64_t b) {
  for (uint32_t k = 0; k < c->klen; ++k) {
    const uint32_t ka = c->keys[a * c->klen + k], kb = c->keys[b * c->klen + k];
    if (ka != kb) return ka < kb;
  }
  if (c->ts[a] != c->ts[b]) return c->ts[a] < c->ts[b];
  if (c->ids[a] != c->ids[b]) return c->ids[a] < c->ids[b];
  return a < b;
}

static int grp_same_key(const grp_ctx* c, uint64_t a, uint64_t b) {
  for (uint32_t k = 0; k < c->klen; ++k)
    if (c->keys[a * c->klen + k] != c->keys[b * c->klen + k]) return 0;
  return 1;
}

static void merge_sort(const grp_ctx* c, uint64_t* v, uint64_t* tmp,
                       uint64_t n) {
  if (n < 2) return;
  const uint64_t h = n / 2;
  merge_sort(c, v, tmp, h);
  merge_sort(c, v + h, tmp, n - h);
  uint64_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = grp_less(c, v[j], v[i]) ? v[j++] : v[i++];
  while (i < h) tmp[k++] = v[i++];
  while (j < n) tmp[k++] = v[j++];
  memcpy(v, tmp, n * sizeof(uint64_t));
}

/* Returns the number of groups; members[] lists peer ids in group order and
 * group_off[g]..group_off[g+1] delimits group g.  Also exposes the sorted
 * input positions through `order` when non-NULL. */
static int64_t form_groups_impl(uint64_t n, const uint32_t* ids,
                                const uint32_t* keys, uint32_t klen,
                                const uint64_t* ts, uint32_t cap,
                                uint32_t* members, uint32_t* group_off,
                                uint64_t* order) {
  if (cap == 0) return ORC_INVALID_ARGUMENT;
  grp_ctx c = {ids, keys, klen, ts};
  uint64_t* v = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  uint64_t* tmp = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) v[i] = i;
  merge_sort(&c, v, tmp, n);
  int64_t g = 0;
  uint64_t cohort_start = 0;
  for (uint64_t p = 0; p < n; ++p) {
    if (p == 0 || !grp_same_key(&c, v[p], v[p - 1])) cohort_start = p;
    if ((p - cohort_start) % cap == 0) group_off[g++] = (uint32_t)p;
    members[p] = ids[v[p]];
    if (order) order[p] = v[p];
  }
  group_off[g] = (uint32_t)n;
  free(v);
  free(tmp);
  return g;
}

int64_t orc_form_groups_uncontested(uint64_t n, const uint32_t* ids,
                                    const uint32_t* keys, uint32_t klen,
                                    const uint64_t* ts, uint32_t cap,
                                    uint32_t* members, uint32_t* group_off) {
  return form_groups_impl(n, ids, keys, klen, ts, cap, members, group_off,
                          NULL);
}

/* ------------------------------------------------------------------------ */
/* allreduce.hpp:46-66 largest-remainder chunking                            */
/* ------------------------------------------------------------------------ */

typedef struct {
  double r;
  uint64_t i;
} rem_t;

static int rem_cmp(const void* pa, const void* pb) {
  /* descending by (remainder, index) -- allreduce.hpp:59-61 */
  const rem_t* a = (const rem_t*)pa;
  const rem_t* b = (const rem_t*)pb;
  if (a->r != b->r) return a->r > b->r ? -1 : 1;
  if (a->i != b->i) return a->i > b->i ? -1 : 1;
  return 0;
}

int orc_chunk_sizes(uint64_t dim, const double* w, uint64_t n, uint64_t* sizes) {
  double total = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    if (w[i] < 0.0) return ORC_INVALID_ARGUMENT;
    total += w[i];
  }
  if (fabs(total - 1.0) > 1e-9) return ORC_INVALID_ARGUMENT;
  rem_t* rem = (rem_t*)malloc((n + 1) * sizeof(rem_t));
  uint64_t assigned = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const double exact = w[i] * (double)dim;
    sizes[i] = (uint64_t)floor(exact);
    assigned += sizes[i];
    rem[i].r = exact - floor(exact);
    rem[i].i = i;
  }
  qsort(rem, n, sizeof(rem_t), rem_cmp);
  for (uint64_t k = 0; assigned < dim; ++k, ++assigned) sizes[rem[k % n].i] += 1;
  free(rem);
  return ORC_OK;
}

/* theory.hpp:149-155 */
double orc_complexity_estimate(uint32_t t, uint32_t n, uint32_t m, uint32_t dim) {
  if (t == 0) return 0.0;
  const double md = m;
  const double s = (double)dim > md ? (double)dim : md;
  return t * (log2((double)n) + md + s * (md - 1.0) / md);
}

/* ------------------------------------------------------------------------ */
/* Shared round scaffolding: protocols.hpp:123-170                           */
/* ------------------------------------------------------------------------ */

/* Distinct random cells by partial Fisher-Yates (protocols.hpp:124-130). */
static void draw_cells(orc_rng* st, uint64_t capacity, uint64_t n,
                       uint64_t* out) {
  uint64_t* cells = (uint64_t*)malloc(capacity * sizeof(uint64_t));
  for (uint64_t i = 0; i < capacity; ++i) cells[i] = i;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t j = i + orc_rng_below(st, capacity - i);
    const uint64_t t = cells[i];
    cells[i] = cells[j];
    cells[j] = t;
  }
  memcpy(out, cells, n * sizeof(uint64_t));
  free(cells);
}

/* protocols.hpp:86-97: no draws at all when p <= 0 */
static void draw_failures(orc_rng* st, uint64_t n, double p, uint8_t* failed) {
  memset(failed, 0, n);
  if (p <= 0.0) return;
  for (uint64_t i = 0; i < n; ++i) failed[i] = (uint8_t)orc_rng_bernoulli(st, p);
}

/* State of one trial's integer plane. */
typedef struct {
  uint32_t M, d, klen;
  uint64_t n;
  uint32_t* keys;  /* n * klen */
  uint32_t* ids;
  uint64_t* ts;
  uint8_t* failed;
  uint32_t* members;
  uint32_t* group_off;
  uint32_t* scratch_key;
  int64_t n_groups;
} plane_t;

static int plane_init(plane_t* pl, uint32_t M, uint32_t d, uint64_t n,
                      orc_rng* cell_stream, uint64_t* cells_out) {
  pl->M = M;
  pl->d = d;
  pl->klen = d - 1;
  pl->n = n;
  pl->keys = (uint32_t*)calloc(n * (pl->klen ? pl->klen : 1), sizeof(uint32_t));
  pl->ids = (uint32_t*)malloc(n * sizeof(uint32_t));
  pl->ts = (uint64_t*)malloc(n * sizeof(uint64_t));
  pl->failed = (uint8_t*)calloc(n, 1);
  pl->members = (uint32_t*)malloc(n * sizeof(uint32_t));
  pl->group_off = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  pl->scratch_key = (uint32_t*)malloc((pl->klen + 1) * sizeof(uint32_t));
  uint64_t* cells = (uint64_t*)malloc(n * sizeof(uint64_t));
  draw_cells(cell_stream, orc_grid_capacity(M, d), n, cells);
  for (uint64_t i = 0; i < n; ++i) {
    pl->ids[i] = (uint32_t)i;
    orc_initial_index(cells[i], M, d, pl->keys + i * pl->klen);
  }
  if (cells_out) memcpy(cells_out, cells, n * sizeof(uint64_t));
  free(cells);
  return ORC_OK;
}

static void plane_free(plane_t* pl) {
  free(pl->keys);
  free(pl->ids);
  free(pl->ts);
  free(pl->failed);
  free(pl->members);
  free(pl->group_off);
  free(pl->scratch_key);
}

/* declare (protocols.hpp:146-150) + form groups (:151) */
static void plane_group(plane_t* pl, orc_rng* clock) {
  for (uint64_t i = 0; i < pl->n; ++i) pl->ts[i] = orc_rng_next(clock) >> 16;
  pl->n_groups = form_groups_impl(pl->n, pl->ids, pl->keys, pl->klen, pl->ts,
                                  pl->M, pl->members, pl->group_off, NULL);
}

/* keys advance for every member, voided or not (protocols.hpp:165-170) */
static void plane_advance(plane_t* pl, uint32_t* rank_out) {
  for (int64_t g = 0; g < pl->n_groups; ++g) {
    for (uint32_t p = pl->group_off[g]; p < pl->group_off[g + 1]; ++p) {
      const uint32_t id = pl->members[p];
      const uint32_t k = p - pl->group_off[g];
      uint32_t* key = pl->keys + (uint64_t)id * pl->klen;
      orc_next_group_key(key, pl->klen, k, pl->M, pl->scratch_key);
      memcpy(key, pl->scratch_key, pl->klen * sizeof(uint32_t));
      if (rank_out) rank_out[id] = k;
    }
  }
}

static int plane_group_void(const plane_t* pl, int64_t g) {
  for (uint32_t p = pl->group_off[g]; p < pl->group_off[g + 1]; ++p)
    if (pl->failed[pl->members[p]]) return 1;
  return 0;
}

int orc_moshpit_trace(uint32_t M, uint32_t d, uint64_t n, double p,
                      uint64_t seed, uint32_t rounds, uint32_t* members,
                      uint32_t* group_off, uint32_t* n_groups,
                      uint8_t* void_flag, uint32_t* rank, uint32_t* active,
                      uint32_t* keys_final, uint64_t* cells) {
  if (orc_grid_validate(M, d, 1) || p < 0.0 || p > 1.0 || n == 0 ||
      n > orc_grid_capacity(M, d))
    return ORC_INVALID_ARGUMENT;
  orc_rng cs, fs, ck;
  orc_rng_stream(&cs, seed, "cells");
  plane_t pl;
  plane_init(&pl, M, d, n, &cs, cells);
  orc_rng_stream(&fs, seed, "failures");
  orc_rng_stream(&ck, seed, "priorities");
  for (uint32_t r = 0; r < rounds; ++r) {
    draw_failures(&fs, n, p, pl.failed);
    plane_group(&pl, &ck);
    memcpy(members + (uint64_t)r * n, pl.members, n * sizeof(uint32_t));
    memcpy(group_off + (uint64_t)r * (n + 1), pl.group_off,
           (pl.n_groups + 1) * sizeof(uint32_t));
    n_groups[r] = (uint32_t)pl.n_groups;
    uint32_t act = 0;
    for (int64_t g = 0; g < pl.n_groups; ++g)
      void_flag[(uint64_t)r * n + g] = (uint8_t)plane_group_void(&pl, g);
    for (uint64_t i = 0; i < n; ++i) act += !pl.failed[i];
    active[r] = act;
    plane_advance(&pl, rank + (uint64_t)r * n);
  }
  if (pl.klen) memcpy(keys_final, pl.keys, n * pl.klen * sizeof(uint32_t));
  plane_free(&pl);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Real-valued routines, instantiated for double and float                   */
/* ------------------------------------------------------------------------ */

#define REAL double
#define SFX f64
#include "oracle_real.inc"
#undef REAL
#undef SFX

#define REAL float
#define SFX f32
#include "oracle_real.inc"
#undef REAL
#undef SFX

/* ------------------------------------------------------------------------ */
/* LogisticRegression (optimizer.hpp:75-146), fp64                          */
/* ------------------------------------------------------------------------ */

/* optimizer.hpp:89-104 synthetic(dim, samples, l2, stream) */
void orc_logistic_synthetic(uint64_t dim, uint64_t samples, orc_rng* st, double* xs,
                            double* ys) {
  double* truth = (double*)malloc((dim ? dim : 1) * sizeof(double));
  for (uint64_t j = 0; j < dim; ++j) truth[j] = orc_rng_normal(st);
  for (uint64_t i = 0; i < samples; ++i) {
    double dot = 0.0;
    for (uint64_t j = 0; j < dim; ++j) {
      xs[i * dim + j] = orc_rng_normal(st);
      dot += xs[i * dim + j] * truth[j];
    }
    ys[i] = dot + 0.1 * orc_rng_normal(st) > 0.0 ? 1.0 : -1.0;
  }
  free(truth);
}

/* optimizer.hpp:106-120 */
double orc_logistic_value(const double* xs, const double* ys, uint64_t samples, uint64_t dim,
                          double l2, const double* th) {
  double f = 0.0;
  for (uint64_t i = 0; i < samples; ++i) {
    double margin = 0.0;
    for (uint64_t j = 0; j < dim; ++j) margin += xs[i * dim + j] * th[j];
    margin *= ys[i];
    f += margin > 0.0 ? log1p(exp(-margin)) : -margin + log1p(exp(margin));
  }
  f /= (double)samples;
  for (uint64_t j = 0; j < dim; ++j) f += 0.5 * l2 * th[j] * th[j];
  return f;
}

/* optimizer.hpp:122-136 */
void orc_logistic_gradient(const double* xs, const double* ys, uint64_t samples, uint64_t dim,
                           double l2, const double* th, double* g) {
  for (uint64_t j = 0; j < dim; ++j) g[j] = 0.0;
  for (uint64_t i = 0; i < samples; ++i) {
    double margin = 0.0;
    for (uint64_t j = 0; j < dim; ++j) margin += xs[i * dim + j] * th[j];
    const double coeff = -ys[i] / (1.0 + exp(ys[i] * margin));
    for (uint64_t j = 0; j < dim; ++j) g[j] += coeff * xs[i * dim + j];
  }
  for (uint64_t j = 0; j < dim; ++j) g[j] = g[j] / (double)samples + l2 * th[j];
}

/* optimizer.hpp:82-86 smoothness L = trace / (4 m) + l2 */
double orc_logistic_smoothness(const double* xs, uint64_t samples, uint64_t dim, double l2) {
  double trace = 0.0;
  for (uint64_t i = 0; i < samples * dim; ++i) trace += xs[i] * xs[i];
  return trace / (4.0 * (double)samples) + l2;
}

/* run_moshpit_sgd (optimizer.hpp:297-439) with LogisticRegression, fp64;
 * same outputs as orc_sgd_quadratic_f64. */
int orc_sgd_logistic_f64(uint32_t M, uint32_t d, uint32_t T, uint32_t n_peers, uint64_t dim,
                         const double* xs, const double* ys, uint64_t samples, double l2,
                         const double* theta0, double gamma, uint32_t tau, uint32_t steps,
                         double sigma, uint32_t inner_rounds, uint64_t seed,
                         double* f_gap, double* grad_norm_sq, double* f_gap_weighted,
                         double* dispersion, double* final_mean, double* diag6,
                         double* final_thetas) {
  if (gamma <= 0.0 || tau < 1 || sigma < 0.0) return ORC_INVALID_ARGUMENT;
  if (orc_grid_validate(M, d, T)) return ORC_INVALID_ARGUMENT;
  if (n_peers < 1 || n_peers > orc_grid_capacity(M, d)) return ORC_INVALID_ARGUMENT;
  const uint32_t inner = inner_rounds == 0 ? d : inner_rounds;
  const uint64_t D = dim ? dim : 1;
  const uint64_t n = n_peers;
  double* th = (double*)malloc(n * D * sizeof(double));
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < dim; ++j) th[i * dim + j] = theta0[j];
  orc_rng noise, avg;
  orc_rng_stream(&noise, seed, "noise");
  orc_rng_stream(&avg, seed, "averaging");
  const double mu = l2;
  double pv_max = 0.0, noise_sq_sum = 0.0, weight_total = 0.0, w_k = 1.0;
  uint64_t noise_count = 0;
  const double w_growth = mu > 0.0 ? 1.0 / (1.0 - gamma * mu) : 1.0;
  double* g = (double*)malloc(D * sizeof(double));
  double* hat = (double*)malloc(D * sizeof(double));
  double* mean = (double*)malloc(D * sizeof(double));
  double* wsum = (double*)calloc(D, sizeof(double));
  double* wtd = (double*)malloc(D * sizeof(double));
  int rc = ORC_OK;
  for (uint32_t k = 0; k < steps && rc == ORC_OK; ++k) {
    const double coord_std = sigma > 0.0 ? sigma / sqrt((double)dim) : 0.0;
    for (uint64_t i = 0; i < n && rc == ORC_OK; ++i) {
      orc_logistic_gradient(xs, ys, samples, dim, l2, th + i * dim, g);
      for (uint64_t j = 0; j < dim; ++j) {
        if (coord_std > 0.0) {
          const double nj = coord_std * orc_rng_normal(&noise);
          noise_sq_sum += nj * nj;
          g[j] += nj;
        }
        if (!isfinite(g[j])) { rc = ORC_RUNTIME_ERROR; break; }
        th[i * dim + j] -= gamma * g[j];
      }
      ++noise_count;
    }
    if (rc != ORC_OK) break;
    colmean_d_f64(th, n, dim, hat);
    if ((k + 1) % tau == 0) orc_moshpit_average_f64(th, n, dim, M, d, inner, &avg);
    colmean_d_f64(th, n, dim, mean);
    double ip = 0.0;
    for (uint64_t j = 0; j < dim; ++j) ip += (mean[j] - hat[j]) * (mean[j] + hat[j]);
    if (ip > pv_max) pv_max = ip;
    double v = 0.0;
    for (uint64_t i = 0; i < n; ++i)
      for (uint64_t j = 0; j < dim; ++j) {
        const double dd = th[i * dim + j] - mean[j];
        v += dd * dd;
      }
    dispersion[k] = v / (double)n;
    f_gap[k] = orc_logistic_value(xs, ys, samples, dim, l2, mean) - 0.0;
    orc_logistic_gradient(xs, ys, samples, dim, l2, mean, g);
    double gn = 0.0;
    for (uint64_t j = 0; j < dim; ++j) gn += g[j] * g[j];
    grad_norm_sq[k] = gn;
    w_k *= w_growth;
    for (uint64_t j = 0; j < dim; ++j) wsum[j] += w_k * mean[j];
    weight_total += w_k;
    for (uint64_t j = 0; j < dim; ++j) wtd[j] = wsum[j] / weight_total;
    f_gap_weighted[k] = orc_logistic_value(xs, ys, samples, dim, l2, wtd) - 0.0;
    memcpy(final_mean, mean, dim * sizeof(double));
  }
  if (rc == ORC_OK) {
    double v_sync_max = 0.0;
    for (uint32_t k = tau - 1; k < steps; k += tau)
      if (dispersion[k] > v_sync_max) v_sync_max = dispersion[k];
    diag6[0] = sqrt(v_sync_max) / gamma;
    diag6[1] = noise_count > 0 && sigma > 0.0 ? sqrt(noise_sq_sum / (double)noise_count) : 0.0;
    diag6[2] = 0.0;
    diag6[3] = sqrt(pv_max > 0.0 ? pv_max : 0.0) / gamma;
    diag6[4] = (double)n;
    diag6[5] = (double)n;
    if (final_thetas) memcpy(final_thetas, th, n * dim * sizeof(double));
  }
  free(th); free(g); free(hat); free(mean); free(wsum); free(wtd);
  return rc;
}
