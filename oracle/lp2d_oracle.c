/* ORACLE — TEST INFRASTRUCTURE ONLY (header: oracle/lp2d_oracle.h).
 *
 * Plain-C restatement of the reference CPU algorithm for the batch-solve hot
 * path. Each function cites the reference file:line it restates (paths under
 * /root/reference/proj/include/lp2d/). Build: oracle/Makefile, flags
 * -O2 -ffp-contract=off (the reference's dot products are unfused).
 */
#include "lp2d_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:13-18 splitmix64 ---------------------------------------- */
static uint64_t splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static inline uint64_t rotl64(uint64_t x, int k) {
  return (x << k) | (x >> (64 - k));
}

/* ---- rng.hpp:20-60 xoshiro256++ ---------------------------------------- */
typedef struct {
  uint64_t s[4];
} xoshiro;

static void xo_seed(xoshiro* r, uint64_t seed) {
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&sm);
}

static uint64_t xo_next(xoshiro* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

/* rng.hpp:42 unit() = (next() >> 11) * 2^-53 */
static double xo_unit(xoshiro* r) {
  return (double)(xo_next(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:44 in_range */
static double xo_in_range(xoshiro* r, double lo, double hi) {
  return lo + (hi - lo) * xo_unit(r);
}

/* rng.hpp:45-56 below(n): Lemire multiply-shift with rejection. */
static uint64_t xo_below(xoshiro* r, uint64_t n) {
  unsigned __int128 mm = (unsigned __int128)xo_next(r) * n;
  uint64_t lo = (uint64_t)mm;
  if (lo < n) {
    const uint64_t threshold = (0 - n) % n;
    while (lo < threshold) {
      mm = (unsigned __int128)xo_next(r) * n;
      lo = (uint64_t)mm;
    }
  }
  return (uint64_t)(mm >> 64);
}

/* rng.hpp:64-68 derive_seed */
uint64_t lp2d_oracle_derive_seed(uint64_t base, uint64_t stream) {
  uint64_t st = base ^ (0x9e3779b97f4a7c15ull * (stream + 1));
  splitmix64(&st);
  return splitmix64(&st);
}

void lp2d_oracle_xoshiro_first(uint64_t seed, int n, uint64_t* out) {
  xoshiro r;
  xo_seed(&r, seed);
  for (int i = 0; i < n; ++i) out[i] = xo_next(&r);
}

uint64_t lp2d_oracle_below(uint64_t seed, uint64_t n, int draws, uint64_t* out) {
  xoshiro r;
  xo_seed(&r, seed);
  for (int i = 0; i < draws; ++i) out[i] = xo_below(&r, n);
  return draws ? out[draws - 1] : 0;
}

/* serial.hpp:126-146 identity_permutation + shuffle (Fisher-Yates). */
void lp2d_oracle_shuffle(int64_t m, uint64_t seed, uint32_t* order) {
  for (int64_t i = 0; i < m; ++i) order[i] = (uint32_t)i;
  xoshiro r;
  xo_seed(&r, seed);
  for (int64_t i = m; i > 1; --i) {
    const uint64_t j = xo_below(&r, (uint64_t)i);
    const uint32_t tmp = order[i - 1];
    order[i - 1] = order[j];
    order[j] = tmp;
  }
}

/* ---- generate.hpp:60-91 ------------------------------------------------ */
static const double kTwoPi = 2.0 * 3.14159265358979323846; /* 2*numbers::pi */

static void gen_feasible_random(int64_t m, xoshiro* r, double margin,
                                double* ax, double* ay, double* b, double* c,
                                double bound_m, double* witness) {
  const double phi = kTwoPi * xo_unit(r);
  c[0] = cos(phi);
  c[1] = sin(phi);
  const double half = bound_m / 2.0;
  const double ix = xo_in_range(r, -half, half);
  const double iy = xo_in_range(r, -half, half);
  if (witness) {
    witness[0] = ix;
    witness[1] = iy;
  }
  for (int64_t k = 0; k < m; ++k) {
    const double theta = kTwoPi * xo_unit(r);
    const double a0 = cos(theta), a1 = sin(theta);
    const double slack = margin * (1.0 + 9.0 * xo_unit(r));
    ax[k] = a0;
    ay[k] = a1;
    b[k] = (a0 * ix + a1 * iy) + slack;
  }
}

int lp2d_oracle_gen(int64_t m, uint64_t seed, int kind, double margin,
                    double* ax, double* ay, double* b, double* c,
                    double* bound_m, double* witness) {
  xoshiro r;
  xo_seed(&r, seed);
  const double M = 1e7; /* serial.hpp:26 default_bound */
  *bound_m = M;
  if (kind == 0) {
    gen_feasible_random(m, &r, margin, ax, ay, b, c, M, witness);
    return 0;
  }
  if (kind == 1) {
    if (m < 1) return -1;
    gen_feasible_random(m - 1, &r, margin, ax, ay, b, c, M, witness);
    const double theta = kTwoPi * xo_unit(&r);
    const double a0 = cos(theta), a1 = sin(theta);
    const double box_min = -(fabs(a0) + fabs(a1)) * M;
    ax[m - 1] = a0;
    ay[m - 1] = a1;
    b[m - 1] = box_min - 1.0;
    return 0;
  }
  return -1;
}

/* ---- serial.hpp solve: double arithmetic over double or float storage ---- */
#define T double
#define S double
#define SUF d
#define SQRT sqrt
#define FABS fabs
#define FMAX fmax
#define FMIN fmin
#include "oracle_solve_impl.h"
#undef S
#undef SUF

/* fp32 configs: the instance is stored in float; the solve is the
 * reference's double arithmetic on the exactly widened values. */
#define S float
#define SUF f
#include "oracle_solve_impl.h"
#undef T
#undef S
#undef SUF
#undef SQRT
#undef FABS
#undef FMAX
#undef FMIN

/* ---- threaded batch driver (bench.hpp:85-99 timed region analogue) ------ */
typedef struct {
  int is_double;
  int64_t lo, hi;
  const int64_t* offset;
  const int32_t* m;
  const void *ax, *ay, *b, *c, *M;
  const uint32_t* perm;
  double eps_par, eps_feas;
  lp2d_oracle_result* out;
  int rc;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  if (j->is_double) {
    j->rc = serial_batch_d(
        j->hi - j->lo, j->offset + j->lo, j->m + j->lo, (const double*)j->ax,
        (const double*)j->ay, (const double*)j->b, j->perm,
        (const double*)j->c + 2 * j->lo, (const double*)j->M + j->lo,
        j->eps_par, j->eps_feas, j->out + j->lo);
  } else {
    j->rc = serial_batch_f(
        j->hi - j->lo, j->offset + j->lo, j->m + j->lo, (const float*)j->ax,
        (const float*)j->ay, (const float*)j->b, j->perm,
        (const float*)j->c + 2 * j->lo, (const float*)j->M + j->lo,
        j->eps_par, j->eps_feas, j->out + j->lo);
  }
  return NULL;
}

static int run_batch(int is_double, int64_t n, const int64_t* offset,
                     const int32_t* m, const void* ax, const void* ay,
                     const void* b, const uint32_t* perm, const void* c,
                     const void* M, double eps_par, double eps_feas,
                     int threads, lp2d_oracle_result* out) {
  if (threads < 1) threads = 1;
  if (threads > n) threads = (int)(n > 0 ? n : 1);
  batch_job* jobs = (batch_job*)calloc((size_t)threads, sizeof(batch_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  /* interleaved-by-chunk split keeps mixed-size batches balanced enough */
  for (int t = 0; t < threads; ++t) {
    batch_job* j = &jobs[t];
    j->is_double = is_double;
    j->lo = n * t / threads;
    j->hi = n * (t + 1) / threads;
    j->offset = offset;
    j->m = m;
    j->ax = ax;
    j->ay = ay;
    j->b = b;
    j->perm = perm;
    j->c = c;
    j->M = M;
    j->eps_par = eps_par;
    j->eps_feas = eps_feas;
    j->out = out;
  }
  int rc = 0;
  if (threads == 1) {
    batch_worker(&jobs[0]);
    rc = jobs[0].rc;
  } else {
    for (int t = 0; t < threads; ++t)
      pthread_create(&tids[t], NULL, batch_worker, &jobs[t]);
    for (int t = 0; t < threads; ++t) {
      pthread_join(tids[t], NULL);
      if (jobs[t].rc) rc = jobs[t].rc;
    }
  }
  free(jobs);
  free(tids);
  return rc;
}

int lp2d_oracle_solve_batch_d(int64_t n, const int64_t* offset,
                              const int32_t* m, const double* ax,
                              const double* ay, const double* b,
                              const uint32_t* perm, const double* c,
                              const double* M, double eps_par, double eps_feas,
                              int threads, lp2d_oracle_result* out) {
  return run_batch(1, n, offset, m, ax, ay, b, perm, c, M, eps_par, eps_feas,
                   threads, out);
}

int lp2d_oracle_solve_batch_f(int64_t n, const int64_t* offset,
                              const int32_t* m, const float* ax,
                              const float* ay, const float* b,
                              const uint32_t* perm, const float* c,
                              const float* M, double eps_par, double eps_feas,
                              int threads, lp2d_oracle_result* out) {
  return run_batch(0, n, offset, m, ax, ay, b, perm, c, M, eps_par, eps_feas,
                   threads, out);
}

/* ---- oracle.hpp:22-74 solve_bruteforce ------------------------------------ */
int lp2d_oracle_bruteforce(const double* cax, const double* cay,
                           const double* cb, int64_t m, double cx, double cy,
                           double M, double eps_par, double eps_feas,
                           lp2d_oracle_result* out) {
  if (m > 512) return -2;
  const int64_t n = m + 4;
  double* ax = (double*)malloc(sizeof(double) * (size_t)n);
  double* ay = (double*)malloc(sizeof(double) * (size_t)n);
  double* b = (double*)malloc(sizeof(double) * (size_t)n);
  const double bx[4] = {1.0, -1.0, 0.0, 0.0}, by[4] = {0.0, 0.0, 1.0, -1.0};
  for (int k = 0; k < 4; ++k) {
    ax[k] = bx[k];
    ay[k] = by[k];
    b[k] = M;
  }
  memcpy(ax + 4, cax, sizeof(double) * (size_t)m);
  memcpy(ay + 4, cay, sizeof(double) * (size_t)m);
  memcpy(b + 4, cb, sizeof(double) * (size_t)m);
  int have = 0;
  double bpx = 0.0, bpy = 0.0, bv = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = i + 1; j < n; ++j) {
      const double det = ax[i] * ay[j] - ay[i] * ax[j]; /* cross(g.a, h.a) */
      const double ng = sqrt(ax[i] * ax[i] + ay[i] * ay[i]);
      const double nh = sqrt(ax[j] * ax[j] + ay[j] * ay[j]);
      if (fabs(det) <= eps_par * ng * nh) continue;
      const double vx = (b[i] * ay[j] - b[j] * ay[i]) / det;
      const double vy = (ax[i] * b[j] - ax[j] * b[i]) / det;
      int feasible = 1;
      for (int64_t q = 0; q < n; ++q) {
        if (!(ax[q] * vx + ay[q] * vy <= b[q] + eps_feas * (1.0 + fabs(b[q])))) {
          feasible = 0;
          break;
        }
      }
      if (!feasible) continue;
      const double value = cx * vx + cy * vy;
      const int better = !have || value > bv ||
                         (value == bv && (vx < bpx || (vx == bpx && vy < bpy)));
      if (better) {
        have = 1;
        bpx = vx;
        bpy = vy;
        bv = value;
      }
    }
  }
  free(ax);
  free(ay);
  free(b);
  memset(out, 0, sizeof(*out));
  out->pair[0] = out->pair[1] = LP2D_ORACLE_NONE;
  if (!have) {
    out->status = LP2D_ORACLE_INFEASIBLE;
    return 0;
  }
  out->status = LP2D_ORACLE_OPTIMAL;
  out->x = bpx;
  out->y = bpy;
  out->value = bv;
  return 0;
}

/* ---- reduction.hpp:46-129 segmented_extremes --------------------------------
 * Each consecutive group of `contention` values reduced to min and max under
 * the reference's three update disciplines (0 serialized, 1 tree, 2 private
 * partials then merge). fmin/fmax as std::fmin/std::fmax. Returns -1 on the
 * reference's invalid_argument cases. */
int lp2d_oracle_segmented_extremes(const double* in, int64_t n, int64_t contention,
                                   int strategy, double* out_min, double* out_max) {
  if (contention <= 0 || n % contention != 0) return -1;
  const int64_t groups = n / contention;
  const int64_t c = contention;
  double* mn = NULL;
  double* mx = NULL;
  if (strategy == 1 || strategy == 2) {
    mn = (double*)malloc(sizeof(double) * (size_t)(c > 32 ? c : 32));
    mx = (double*)malloc(sizeof(double) * (size_t)(c > 32 ? c : 32));
  }
  for (int64_t g = 0; g < groups; ++g) {
    const double* v = in + g * c;
    if (strategy == 0) { /* serialized shared update, reduction.hpp:66-78 */
      double a = v[0], b = v[0];
      for (int64_t i = 1; i < c; ++i) {
        a = fmin(a, v[i]);
        b = fmax(b, v[i]);
      }
      out_min[g] = a;
      out_max[g] = b;
    } else if (strategy == 1) { /* halving tree, reduction.hpp:80-97 */
      for (int64_t i = 0; i < c; ++i) mn[i] = mx[i] = v[i];
      int64_t s = 1;
      while (s < c) s <<= 1;
      for (s >>= 1; s >= 1; s >>= 1) {
        for (int64_t i = 0; i < s; ++i)
          if (i + s < c) {
            mn[i] = fmin(mn[i], mn[i + s]);
            mx[i] = fmax(mx[i], mx[i + s]);
          }
        if (s == 1) break;
      }
      out_min[g] = mn[0];
      out_max[g] = mx[0];
    } else { /* private partials then merge, reduction.hpp:99-125 */
      const int64_t lanes = c < 32 ? c : 32;
      for (int64_t l = 0; l < lanes; ++l) {
        double a = v[l], b = v[l];
        for (int64_t i = l + lanes; i < c; i += lanes) {
          a = fmin(a, v[i]);
          b = fmax(b, v[i]);
        }
        mn[l] = a;
        mx[l] = b;
      }
      double a = mn[0], b = mx[0];
      for (int64_t l = 1; l < lanes; ++l) {
        a = fmin(a, mn[l]);
        b = fmax(b, mx[l]);
      }
      out_min[g] = a;
      out_max[g] = b;
    }
  }
  free(mn);
  free(mx);
  return 0;
}

/* bench.hpp:256-257: the contention benchmark's inputs,
 * xoshiro256pp(derive_seed(seed, stream)).in_range(lo, hi) drawn n times. */
void lp2d_oracle_uniform(uint64_t seed, uint64_t stream, double lo, double hi, int64_t n,
                         double* out) {
  xoshiro r;
  xo_seed(&r, lp2d_oracle_derive_seed(seed, stream));
  for (int64_t i = 0; i < n; ++i) out[i] = xo_in_range(&r, lo, hi);
}
