/* TEST INFRASTRUCTURE ONLY (oracle/).  See lmshoot_oracle.h for the contract and parity status.
 * Plain-C restatement of /root/reference/proj/include/lmshoot/{shooting,reduction,vec,flow,rng}.hpp
 * for the objective-and-gradient hot path.  Each function cites the reference lines it follows.
 * Built by oracle/Makefile with -O2 -ffp-contract=off (no FMA contraction) so that it reproduces
 * the reference build bit for bit. */
#include "lmshoot_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* parallel.hpp:11-20 / parallel.cpp:134-150: [0,n) in at most `threads` contiguous chunks,
 * chunk c = [n*c/chunks, n*(c+1)/chunks); 0 = hardware concurrency; blocking. */
typedef void (*orc_range_fn)(void* job, size_t begin, size_t end);
typedef struct {
  orc_range_fn fn;
  void* job;
  size_t begin, end;
} OrcChunk;

static void* orc_chunk_main(void* v)
{
  OrcChunk* c = (OrcChunk*)v;
  c->fn(c->job, c->begin, c->end);
  return NULL;
}

static unsigned orc_hardware_threads(void)
{
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n < 1 ? 1u : (unsigned)n;
}

static void orc_parallel_for(size_t n, unsigned threads, orc_range_fn fn, void* job)
{
  if (n == 0) return;
  size_t want = threads == 0 ? orc_hardware_threads() : threads;
  size_t chunks = want < n ? want : n;
  if (chunks <= 1) {
    fn(job, 0, n);
    return;
  }
  OrcChunk* cs = (OrcChunk*)malloc(chunks * sizeof(OrcChunk));
  pthread_t* ts = (pthread_t*)malloc(chunks * sizeof(pthread_t));
  for (size_t c = 0; c < chunks; ++c) {
    cs[c].fn = fn;
    cs[c].job = job;
    cs[c].begin = n * c / chunks;
    cs[c].end = n * (c + 1) / chunks;
  }
  for (size_t c = 1; c < chunks; ++c) pthread_create(&ts[c], NULL, orc_chunk_main, &cs[c]);
  orc_chunk_main(&cs[0]);
  for (size_t c = 1; c < chunks; ++c) pthread_join(ts[c], NULL);
  free(cs);
  free(ts);
}

unsigned orc_hardware_threads_public(void) { return orc_hardware_threads(); }

#define REAL float
#define SFX _f32
#define REAL_EXP expf
#include "lmshoot_oracle_body.inc"
#undef REAL
#undef SFX
#undef REAL_EXP

#define REAL double
#define SFX _f64
#define REAL_EXP exp
#include "lmshoot_oracle_body.inc"
#undef REAL
#undef SFX
#undef REAL_EXP

static _Thread_local int g_bad_step = -1;
int orc_last_diverged_step(void) { return g_bad_step; }

/* ---- rng.hpp: std::mt19937_64 (Matsumoto & Nishimura 2004, the parameters the C++ standard fixes)
 * with the explicit uniform (rng.hpp:19-22) and Box-Muller (rng.hpp:27-41) transforms. ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
  int have_spare;
  double spare;
} OrcRng;

static void rng_seed(OrcRng* r, uint64_t seed)
{
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->have_spare = 0;
  r->spare = 0.0;
}

static uint64_t rng_raw(OrcRng* r)
{
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

static double rng_uniform(OrcRng* r) { return (double)(rng_raw(r) >> 11) * 0x1.0p-53; }

static double rng_normal(OrcRng* r)
{
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = 0.0;
  while (u1 <= 0.0) u1 = rng_uniform(r);
  double u2 = rng_uniform(r);
  double rad = sqrt(-2.0 * log(u1));
  double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
  r->spare = rad * sin(theta);
  r->have_spare = 1;
  return rad * cos(theta);
}

void orc_rng_uniforms(unsigned long long seed, size_t count, double* out)
{
  OrcRng r;
  rng_seed(&r, seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng_uniform(&r);
}

void orc_rng_normals(unsigned long long seed, size_t count, double* out)
{
  OrcRng r;
  rng_seed(&r, seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng_normal(&r);
}

void orc_rng_stream(unsigned long long seed, size_t count, const unsigned char* kinds, double* out)
{
  OrcRng r;
  rng_seed(&r, seed);
  for (size_t i = 0; i < count; ++i) out[i] = kinds[i] ? rng_normal(&r) : rng_uniform(&r);
}

/* shooting.hpp:55-59 */
double orc_gaussian_kernel(int prec, double r_sq, double sigma)
{
  if (prec == 0) {
    float r = (float)r_sq, s = (float)sigma;
    return (double)expf(-r / (2.0f * s * s));
  }
  return exp(-r_sq / (2.0 * sigma * sigma));
}

double orc_kernel_scale(int prec, double sigma)
{
  return prec == 0 ? (double)kscale_f32(sigma) : kscale_f64(sigma);
}

/* reduction.hpp:110-122 */
double orc_tree_sum(int prec, const double* values, size_t n)
{
  if (n == 0) return 0.0;
  if (n == 1) return prec == 0 ? (double)(float)values[0] : values[0];
  size_t m = 1;
  while (m < n) m <<= 1;
  double out;
  if (prec == 0) {
    float* buf = (float*)calloc(m, sizeof(float));
    for (size_t i = 0; i < n; ++i) buf[i] = (float)values[i];
    for (size_t h = m / 2; h >= 1; h >>= 1)
      for (size_t k = 0; k < h; ++k) buf[k] += buf[k + h];
    out = (double)buf[0];
    free(buf);
  } else {
    double* buf = (double*)calloc(m, sizeof(double));
    for (size_t i = 0; i < n; ++i) buf[i] = values[i];
    for (size_t h = m / 2; h >= 1; h >>= 1)
      for (size_t k = 0; k < h; ++k) buf[k] += buf[k + h];
    out = buf[0];
    free(buf);
  }
  return out;
}

static int check_args(int dim, double sigma, size_t block)
{
  if (dim != 2 && dim != 3) return 1; /* ShapeError, shooting.hpp:358 */
  if (!(sigma > 0)) return 3;         /* shooting.hpp:113 */
  if (block < 32 || block > 1024 || (block & (block - 1))) return 3; /* reduction.hpp:51-52 */
  return 0;
}

int orc_hamiltonian(int prec, int dim, size_t n, double sigma, const double* q, const double* p,
                    unsigned threads, double* out)
{
  int rc = check_args(dim, sigma, 256);
  if (rc) return rc;
  size_t nd = n * dim;
  if (prec == 0) {
    float *tq = load_f32(q, nd), *tp = load_f32(p, nd);
    *out = hamiltonian_T_f32(dim, n, sigma, tq, tp, threads);
    free(tq); free(tp);
  } else {
    double *tq = load_f64(q, nd), *tp = load_f64(p, nd);
    *out = hamiltonian_T_f64(dim, n, sigma, tq, tp, threads);
    free(tq); free(tp);
  }
  return 0;
}

int orc_derivatives(int prec, int dim, size_t n, double sigma, const double* q, const double* p,
                    double* hq, double* hp, int strategy, size_t block, unsigned threads)
{
  int rc = check_args(dim, sigma, block);
  if (rc) return rc;
  size_t nd = n * dim;
#define BODY(R, S)                                                                       \
  {                                                                                      \
    R *tq = load##S(q, nd), *tp = load##S(p, nd);                                        \
    R *ohq = (R*)malloc((nd ? nd : 1) * sizeof(R)), *ohp = (R*)malloc((nd ? nd : 1) * sizeof(R)); \
    derivatives_T##S(dim, n, sigma, tq, tp, ohq, ohp, strategy, block, threads);         \
    store##S(ohq, nd, hq); store##S(ohp, nd, hp);                                        \
    free(tq); free(tp); free(ohq); free(ohp);                                            \
  }
  if (prec == 0) BODY(float, _f32) else BODY(double, _f64)
#undef BODY
  return 0;
}

int orc_integrate_forward(int prec, int dim, size_t n, double sigma, int timesteps, const double* q0,
                          const double* p0, double* traj_q, double* traj_p, int strategy, size_t block,
                          unsigned threads)
{
  int rc = check_args(dim, sigma, block);
  if (rc) return rc;
  if (timesteps < 1) return 3; /* shooting.hpp:184 */
  size_t nd = n * dim, total = nd * (size_t)(timesteps + 1);
  g_bad_step = -1;
#define BODY(R, S)                                                                          \
  {                                                                                         \
    R *tq0 = load##S(q0, nd), *tp0 = load##S(p0, nd);                                       \
    R *tq = (R*)calloc(total ? total : 1, sizeof(R)), *tp = (R*)calloc(total ? total : 1, sizeof(R)); \
    int bad = -1;                                                                           \
    rc = integrate_T##S(dim, n, sigma, timesteps, tq0, tp0, tq, tp, strategy, block, threads, &bad); \
    if (rc == 0) { store##S(tq, total, traj_q); store##S(tp, total, traj_p); }              \
    else g_bad_step = bad;                                                                  \
    free(tq0); free(tp0); free(tq); free(tp);                                               \
  }
  if (prec == 0) BODY(float, _f32) else BODY(double, _f64)
#undef BODY
  return rc;
}

int orc_adjoint_step(int prec, int dim, size_t n, double sigma, const double* q, const double* p,
                     const double* alpha, const double* beta, double* d_alpha, double* d_beta,
                     int strategy, size_t block, unsigned threads)
{
  int rc = check_args(dim, sigma, block);
  if (rc) return rc;
  size_t nd = n * dim;
#define BODY(R, S)                                                                        \
  {                                                                                       \
    R *tq = load##S(q, nd), *tp = load##S(p, nd), *ta = load##S(alpha, nd), *tb = load##S(beta, nd); \
    R *da = (R*)malloc((nd ? nd : 1) * sizeof(R)), *db = (R*)malloc((nd ? nd : 1) * sizeof(R)); \
    adjoint_T##S(dim, n, sigma, tq, tp, ta, tb, da, db, strategy, block, threads);        \
    store##S(da, nd, d_alpha); store##S(db, nd, d_beta);                                  \
    free(tq); free(tp); free(ta); free(tb); free(da); free(db);                           \
  }
  if (prec == 0) BODY(float, _f32) else BODY(double, _f64)
#undef BODY
  return 0;
}

int orc_mismatch_sq(int prec, int dim, size_t n, const double* a, const double* b, double* out)
{
  if (dim != 2 && dim != 3) return 1;
  size_t nd = n * dim;
  if (prec == 0) {
    float *ta = load_f32(a, nd), *tb = load_f32(b, nd);
    *out = mismatch_T_f32(dim, n, ta, tb);
    free(ta); free(tb);
  } else {
    double *ta = load_f64(a, nd), *tb = load_f64(b, nd);
    *out = mismatch_T_f64(dim, n, ta, tb);
    free(ta); free(tb);
  }
  return 0;
}

/* landmarks.cpp:148-161 pointwise_dist (double sum of squared coordinate differences, sqrt), :164-171 average_dist
 * (sequential sum over the points / n), :173-179 max_dist (running std::max from 0).  n == 0: the reference divides
 * 0 by 0; callers never pass empty sets (require_paired + registration.cpp:148-150), so {0, 0} is returned. */
int orc_landmark_distances(int dim, size_t n, const double* a, const double* b, double* out)
{
  if (dim != 2 && dim != 3) return 1;
  double sum = 0, best = 0;
  for (size_t i = 0; i < n; ++i) {
    double s = 0;
    for (int c = 0; c < dim; ++c) {
      double d = a[i * dim + c] - b[i * dim + c];
      s += d * d;
    }
    double dist = sqrt(s);
    sum += dist;
    best = best > dist ? best : dist;
  }
  out[0] = n ? sum / (double)n : 0.0;
  out[1] = best;
  return 0;
}

int orc_compute_gradient(int prec, int dim, size_t n, double sigma, double lambda, int timesteps,
                         const double* q0, const double* p0, const double* target, double* scalars,
                         double* grad, int strategy, size_t block, unsigned threads)
{
  int rc = check_args(dim, sigma, block);
  if (rc) return rc;
  if (timesteps < 1) return 3;
  size_t nd = n * dim;
  g_bad_step = -1;
#define BODY(R, S)                                                                          \
  {                                                                                         \
    R *tq = load##S(q0, nd), *tp = load##S(p0, nd), *tt = load##S(target, nd);              \
    R* g = (R*)malloc((nd ? nd : 1) * sizeof(R));                                           \
    int bad = -1;                                                                           \
    rc = gradient_T##S(dim, n, sigma, lambda, timesteps, tq, tp, tt, scalars, g, strategy, block, threads, &bad); \
    if (rc == 0) store##S(g, nd, grad); else g_bad_step = bad;                              \
    free(tq); free(tp); free(tt); free(g);                                                  \
  }
  if (prec == 0) BODY(float, _f32) else BODY(double, _f64)
#undef BODY
  return rc;
}

int orc_velocities(int prec, int dim, size_t n, size_t m, double sigma, const double* q, const double* p,
                   const double* points, double* out, int strategy, size_t block, unsigned threads)
{
  int rc = check_args(dim, sigma, block);
  if (rc) return rc;
  size_t nd = n * dim, md = m * dim;
#define BODY(R, S)                                                                     \
  {                                                                                    \
    R *tq = load##S(q, nd), *tp = load##S(p, nd), *tx = load##S(points, md);           \
    R* v = (R*)malloc((md ? md : 1) * sizeof(R));                                      \
    velocities_T##S(dim, n, m, sigma, tq, tp, tx, v, strategy, block, threads);        \
    store##S(v, md, out);                                                              \
    free(tq); free(tp); free(tx); free(v);                                             \
  }
  if (prec == 0) BODY(float, _f32) else BODY(double, _f64)
#undef BODY
  return 0;
}

/* sums: nrows x 2*dim = (hq | hp) of derivatives, or (d_alpha | d_beta) of adjoint_step when alpha/beta
 * are non-NULL, for the listed rows only. */
int orc_pair_rows(int prec, int dim, size_t n, double sigma, const double* q, const double* p,
                  const double* alpha, const double* beta, size_t nrows, const size_t* rows, double* sums,
                  int strategy, size_t block, unsigned threads)
{
  int rc = check_args(dim, sigma, block);
  if (rc) return rc;
  for (size_t r = 0; r < nrows; ++r)
    if (rows[r] >= n) return 1;
  size_t nd = n * dim;
  const int adjoint = alpha != NULL && beta != NULL;
#define BODY(R, S)                                                                               \
  {                                                                                              \
    R *tq = load##S(q, nd), *tp = load##S(p, nd);                                                \
    R *ta = adjoint ? load##S(alpha, nd) : NULL, *tb = adjoint ? load##S(beta, nd) : NULL;       \
    R* out = (R*)malloc((nrows ? nrows : 1) * 2 * dim * sizeof(R));                              \
    rows_T##S(adjoint, dim, n, sigma, tq, tp, ta, tb, nrows, rows, out, strategy, block, threads); \
    store##S(out, nrows * 2 * dim, sums);                                                        \
    free(tq); free(tp); free(ta); free(tb); free(out);                                           \
  }
  if (prec == 0) BODY(float, _f32) else BODY(double, _f64)
#undef BODY
  return 0;
}

/* flow.hpp:66-81: x += dt * v(x, t) for t = 0..T-1 with the trajectory's own dt = T(1/T). */
int orc_warp_points(int prec, int dim, size_t n, size_t m, double sigma, int timesteps,
                    const double* traj_q, const double* traj_p, const double* points, double* out,
                    int strategy, size_t block, unsigned threads)
{
  int rc = check_args(dim, sigma, block);
  if (rc) return rc;
  if (timesteps < 1) return 3;
  size_t nd = n * dim, md = m * dim, total = nd * (size_t)(timesteps + 1);
  g_bad_step = -1;
#define BODY(R, S)                                                                          \
  {                                                                                         \
    R *tq = load##S(traj_q, total), *tp = load##S(traj_p, total), *x = load##S(points, md); \
    R* v = (R*)malloc((md ? md : 1) * sizeof(R));                                           \
    const R dt = (R)(1.0 / timesteps);                                                      \
    for (int t = 0; t < timesteps && rc == 0; ++t) {                                        \
      velocities_T##S(dim, n, m, sigma, tq + (size_t)t * nd, tp + (size_t)t * nd, x, v, strategy, block, threads); \
      for (size_t e = 0; e < md; ++e) {                                                     \
        x[e] = x[e] + dt * v[e];                                                            \
        if (!isfinite(x[e]) && rc == 0) { rc = 2; g_bad_step = t + 1; }                     \
      }                                                                                     \
    }                                                                                       \
    if (rc == 0) store##S(x, md, out);                                                      \
    free(tq); free(tp); free(x); free(v);                                                   \
  }
  if (prec == 0) BODY(float, _f32) else BODY(double, _f64)
#undef BODY
  return rc;
}
