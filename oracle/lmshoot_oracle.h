/* TEST INFRASTRUCTURE ONLY (oracle/): a plain-C CPU restatement of the reference hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this; the product library (paper_1907_04839_b200/csrc) never does.
 *
 * Parity status: PINNED.  Every function below is checked bit for bit against the unmodified
 * reference compiled in place (oracle/_ref/liblmshoot_ref.so, built by oracle/Makefile from
 * /root/reference/proj) in tests/test_oracle.py, against the analytic known-answer values of
 * /root/reference/SPEC.md:148-216, and against the committed fixtures tests/golden/*.npz that
 * tests/golden/make_golden.py generated from the reference build.
 *
 * Conventions: all arrays are row-major double, n x dim (dim in {2,3}); `prec` 0 = float32,
 * 1 = float64 working precision T (inputs are cast T(x) on entry, outputs double(T) on exit, as
 * the reference's objective closure does, registration.cpp:61-67).  `strategy` follows
 * reduction.hpp:41 (0 sequential, 1 precompute_matrix, 2 blocked_tree).  Return codes:
 * 0 ok, 1 shape, 2 diverged (see orc_last_diverged_step), 3 invalid argument. */
#ifndef LMSHOOT_ORACLE_H
#define LMSHOOT_ORACLE_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

int orc_last_diverged_step(void);
double orc_gaussian_kernel(int prec, double r_sq, double sigma);
double orc_kernel_scale(int prec, double sigma);
double orc_tree_sum(int prec, const double* values, size_t n);
void orc_rng_uniforms(unsigned long long seed, size_t count, double* out);
void orc_rng_normals(unsigned long long seed, size_t count, double* out);
void orc_rng_stream(unsigned long long seed, size_t count, const unsigned char* kinds, double* out);

int orc_hamiltonian(int prec, int dim, size_t n, double sigma, const double* q, const double* p,
                    unsigned threads, double* out);
int orc_derivatives(int prec, int dim, size_t n, double sigma, const double* q, const double* p,
                    double* hq, double* hp, int strategy, size_t block, unsigned threads);
int orc_integrate_forward(int prec, int dim, size_t n, double sigma, int timesteps, const double* q0,
                          const double* p0, double* traj_q, double* traj_p, int strategy, size_t block,
                          unsigned threads);
int orc_adjoint_step(int prec, int dim, size_t n, double sigma, const double* q, const double* p,
                     const double* alpha, const double* beta, double* d_alpha, double* d_beta,
                     int strategy, size_t block, unsigned threads);
int orc_mismatch_sq(int prec, int dim, size_t n, const double* a, const double* b, double* out);
/* average_dist / max_dist between paired double landmark sets (landmarks.cpp:148-179): out = {avg, max}. */
int orc_landmark_distances(int dim, size_t n, const double* a, const double* b, double* out);
int orc_compute_gradient(int prec, int dim, size_t n, double sigma, double lambda, int timesteps,
                         const double* q0, const double* p0, const double* target, double* scalars,
                         double* grad, int strategy, size_t block, unsigned threads);
/* Row subset of derivatives (alpha = beta = NULL: sums = hq|hp) or adjoint_step (sums = d_alpha|d_beta):
 * identical terms and per-row reduction, only the listed rows; pinned against the full calls in
 * tests/test_oracle.py. */
int orc_pair_rows(int prec, int dim, size_t n, double sigma, const double* q, const double* p,
                  const double* alpha, const double* beta, size_t nrows, const size_t* rows, double* sums,
                  int strategy, size_t block, unsigned threads);
int orc_velocities(int prec, int dim, size_t n, size_t m, double sigma, const double* q, const double* p,
                   const double* points, double* out, int strategy, size_t block, unsigned threads);
int orc_warp_points(int prec, int dim, size_t n, size_t m, double sigma, int timesteps,
                    const double* traj_q, const double* traj_p, const double* points, double* out,
                    int strategy, size_t block, unsigned threads);

#ifdef __cplusplus
}
#endif
#endif
