/* lmshoot_b200 — C ABI of the B200-native (sm_100a) landmark-shooting hot path.
 *
 * This is the drop-in boundary for the reference's objective-and-gradient evaluation
 * (arXiv 1907.04839).  Every entry point cites the reference interface it replaces
 * (paths under /root/reference/proj).  Plain pointers and sizes only: no C++ or torch types cross
 * this boundary.  The caller owns all host buffers; the library owns all device memory.
 *
 * Data conventions (reference: registration.cpp:48-52,61-67; vec.hpp:12-16): every point array is
 * row-major `double[n * dim]`, element (i, c) at `i * dim + c`, regardless of the working precision
 * T; values are cast `T(x)` on entry and `double(T)` on exit exactly as the reference's objective
 * closure does.  Pair arithmetic and row sums run in T on the GPU; the three scalars (loss, H,
 * mismatch) are accumulated in double (shooting.hpp:99-103).
 *
 * Threading: one call at a time per handle; different handles may be used concurrently from
 * different host threads.  There is no CPU fallback: creation fails with LMS_ERR_CUDA when no
 * sm_100 device is usable.
 */
#ifndef LMSHOOT_B200_H
#define LMSHOOT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1:1 with the reference's exception taxonomy (errors.hpp:10-77) ---- */
#define LMS_OK 0
#define LMS_ERR_SHAPE 1     /* lmshoot::ShapeError (shooting.hpp:332-338, 358) */
#define LMS_ERR_DIVERGED 2  /* lmshoot::DivergedError(timestep[, point]) (shooting.hpp:185-186,210-211) */
#define LMS_ERR_INVALID 3   /* std::invalid_argument (shooting.hpp:39-42,113,184; lbfgs.hpp:21-26) */
#define LMS_ERR_NUMERICAL 4 /* lmshoot::NumericalError (lbfgs.cpp:197-198) */
#define LMS_ERR_CUDA 5      /* CUDA runtime failure / no usable device */
#define LMS_ERR_STATE 6     /* call order violated (e.g. eval before bind) */
#define LMS_ERR_COMM 7      /* NCCL failure in row-partitioned mode */

#define LMS_PRECISION_F32 0 /* lmshoot::Precision::f32 (shooting.hpp:17) */
#define LMS_PRECISION_F64 1 /* lmshoot::Precision::f64 */

typedef struct lms_system lms_system;

/* Replaces the constructor arguments of HamiltonianSystem<T,D> (shooting.hpp:110-117) plus the
 * runtime (precision, dim) dispatch (shooting.hpp:348-368).  ReduceOptions (reduction.hpp:43-54)
 * has no counterpart: the GPU row reduction is register accumulation in a fixed order. */
typedef struct lms_config {
  int precision;     /* LMS_PRECISION_F32 | LMS_PRECISION_F64 */
  int dim;           /* 2 | 3 */
  size_t n;          /* landmarks */
  double sigma;      /* Gaussian kernel std, > 0 */
  int max_timesteps; /* capacity of the device-resident trajectory (T + 1 snapshots are stored) */
  int device;        /* CUDA device ordinal */
  int variant;       /* kernel variant: 0 = library default (by problem size); see lms_variant_name() */
  int flags;         /* 0, or LMS_FLAG_* bits */
} lms_config;

/* Single problems of up to 8192 landmarks in fp32 (3400 in fp64) run the whole evaluation as one persistent
 * cooperative kernel (csrc/small_kernels.cuh); this bit pins the tiled multi-launch path instead (A/B and tests). */
#define LMS_FLAG_TILED_ONLY 1

int lms_system_create(const lms_config* cfg, lms_system** out);
void lms_system_destroy(lms_system* sys);

/* Last error detail for this handle: DivergedError's timestep / point (point = -1 when unknown),
 * and a static message. */
int lms_last_diverged_step(const lms_system* sys);
long long lms_last_diverged_point(const lms_system* sys);
const char* lms_last_error_message(const lms_system* sys);
const char* lms_status_string(int status);
const char* lms_variant_name(int precision, int variant);
/* "<forward kernel> / <adjoint kernel>" this handle launches (variant 0 chooses the shapes by problem size). */
const char* lms_system_kernel_names(const lms_system* sys);

/* ---- HamiltonianSystem members, one call each (parity-test surface) ---- */

/* hamiltonian(q, p) — shooting.hpp:123-142.  out = 1/2 sum_ij (p_i . p_j) K_ij in double. */
int lms_hamiltonian(lms_system* sys, const double* q, const double* p, double* out);

/* derivatives(q, p, hq, hp) — shooting.hpp:147-176. */
int lms_derivatives(lms_system* sys, const double* q, const double* p, double* hq, double* hp);

/* integrate_forward(q0, p0, timesteps) — shooting.hpp:180-214.  traj_q / traj_p receive the
 * (timesteps + 1) x n x dim snapshots (either may be NULL).  The trajectory also stays
 * device-resident for lms_warp_points_stored().  LMS_ERR_DIVERGED carries the first bad step. */
int lms_integrate_forward(lms_system* sys, const double* q0, const double* p0, int timesteps,
                          double* traj_q, double* traj_p);

/* adjoint_step(q, p, adj, d_alpha, d_beta) — shooting.hpp:233-271. */
int lms_adjoint_step(lms_system* sys, const double* q, const double* p, const double* alpha,
                     const double* beta, double* d_alpha, double* d_beta);

/* mismatch_sq(a, b) — shooting.hpp:318-329. */
int lms_mismatch_sq(lms_system* sys, const double* a, const double* b, double* out);

/* compute_gradient(q0, p0, target, lambda, timesteps) — shooting.hpp:277-315.
 * scalars[3] = {loss, kinetic, mismatch} (GradientResult, shooting.hpp:91-97). */
int lms_compute_gradient(lms_system* sys, const double* q0, const double* p0, const double* target,
                         double lambda, int timesteps, double* scalars, double* grad);

/* ---- the objective closure (registration.cpp:58-74) ---- */

/* Captures what the closure captures (registration.cpp:43-45: q0, target, lambda, timesteps):
 * uploaded once, device-resident across evaluations. */
int lms_bind_registration(lms_system* sys, const double* q0, const double* target, double lambda,
                          int timesteps);

/* One objective evaluation = lmshoot::Objective::operator() (lbfgs.hpp:48-50) for the closure at
 * registration.cpp:58-74: x = flat p0, grad fully overwritten, returns the loss through *loss.
 * kinetic / mismatch (may be NULL) feed the verbose line at registration.cpp:70-72.
 * Host buffers; blocking. */
int lms_objective_eval(lms_system* sys, const double* x, double* grad, double* loss, double* kinetic,
                       double* mismatch);

/* Same evaluation with x and grad already in device memory (double[n*dim] on cfg.device); the
 * three scalars come back through host pointers.  Blocking. */
int lms_objective_eval_device(lms_system* sys, const double* d_x, double* d_grad, double* scalars);

/* q(1) of the last evaluation (the warped landmarks; saves the re-integration at
 * registration.cpp:85-93). */
int lms_objective_final_q(lms_system* sys, double* out);

/* Registration metrics on the device (registration.cpp:39-40,95-96 -> landmarks.cpp:164-179 average_dist, max_dist):
 * out[4] = {avg_before, max_before, avg_after, max_after}: template vs target as bound, and the warped landmarks
 * q(1) of the last evaluation (widened to double as registration.cpp:88-92 does) vs target.  Per-point distances in
 * double, the average as the reference's sequential sum: bit-identical to the reference's loops. */
int lms_registration_metrics(lms_system* sys, double* out);

/* Device time (ms, CUDA events on the library stream) of the compute part of the last evaluation
 * and the number of kernels it launched. */
double lms_last_eval_device_ms(const lms_system* sys);
int lms_last_eval_kernel_launches(const lms_system* sys);
/* Average device time (ms) of one launch of the dominant kernel class in the last evaluation:
 * which = 0 forward pair kernel, 1 adjoint pair kernel.  Requires lms_set_kernel_timing(sys, 1),
 * which runs evaluations as individually timed launches instead of one CUDA graph. */
int lms_set_kernel_timing(lms_system* sys, int enabled);
double lms_last_kernel_ms(const lms_system* sys, int which);

/* ---- flow / warp (flow.hpp) ---- */

/* detail::velocities_at_step — flow.hpp:26-48: v[m] = sum_l K(|x_m - q_l|^2) p_l for m points
 * against one snapshot (q, p) of the n landmarks. */
int lms_velocities(lms_system* sys, const double* q, const double* p, size_t m, const double* points,
                   double* out);

/* warp_points — flow.hpp:66-81, through the trajectory stored by the last lms_integrate_forward /
 * lms_objective_eval on this handle. */
int lms_warp_points_stored(lms_system* sys, size_t m, const double* points, double* out);

/* ---- optimiser: L-BFGS + strong-Wolfe line search (lbfgs.hpp:11-82, lbfgs.cpp:186-282) ---- */

typedef double (*lms_objective_fn)(void* user, const double* x, double* grad, size_t n);

typedef struct lms_lbfgs_params { /* LbfgsParams, lbfgs.hpp:11-27 */
  int memory;
  int max_iter;
  double grad_tol;
  double c1;
  double c2;
  int max_line_search;
} lms_lbfgs_params;

typedef struct lms_minimize_result { /* MinimizeResult + OptimHistory, lbfgs.hpp:33-46,71-76 */
  double loss;
  double initial_loss;
  double initial_grad_inf_norm;
  int evaluations;
  int iterations; /* accepted iterates */
  int reason;     /* 0 gradient_tolerance, 1 max_iterations, 2 line_search_failure */
} lms_minimize_result;

void lms_lbfgs_default_params(lms_lbfgs_params* p);

/* minimize(objective, x0, params) — lbfgs.hpp:81-82.  hist_* (each may be NULL) receive one
 * IterationRecord (lbfgs.hpp:33-38) per accepted iterate, capacity params->max_iter. */
int lms_minimize(lms_objective_fn fn, void* user, size_t n, const double* x0,
                 const lms_lbfgs_params* params, double* x_out, double* grad_out,
                 lms_minimize_result* result, double* hist_loss, double* hist_grad_inf_norm,
                 double* hist_step, int* hist_evals);

/* register_impl core — registration.cpp:43-93: x0 = (target - q0)/T, minimize over the bound
 * objective, momenta_out = p0*, warped_out = q(1) under p0*.  Requires lms_bind_registration. */
int lms_register(lms_system* sys, const lms_lbfgs_params* params, double* momenta_out,
                 double* warped_out, lms_minimize_result* result, double* hist_loss);

/* The same registration with the optimiser's vectors resident in HBM: x, g, d, the trial
 * point and the curvature pairs never leave the device, dot products come back as one double each, and the
 * objective runs through lms_objective_eval_device.  Same decision logic as lms_minimize / lbfgs.cpp:186-282;
 * sums are deterministic but not in the reference's sequential order, so iterates agree with lms_register to
 * rounding, not bit for bit. */
int lms_register_device(lms_system* sys, const lms_lbfgs_params* params, double* momenta_out,
                        double* warped_out, lms_minimize_result* result, double* hist_loss);

/* ---- population batches (BASELINE configs[3]; no counterpart in the single-problem reference) ---- */

/* A handle that holds `batch` independent registrations of cfg->n landmarks each (same sigma, dim,
 * precision, lambda, timesteps).  Every O(N^2) launch covers all requested problems at once, so many
 * small problems fill the GPU.  Arrays are batch-major: problem b occupies [b*n*dim, (b+1)*n*dim).
 * lms_bind_registration() on such a handle takes batch x n x dim templates and targets. */
int lms_batch_create(const lms_config* cfg, size_t batch, lms_system** out);
size_t lms_batch_size(const lms_system* sys);

/* One objective evaluation (registration.cpp:58-74) for `count` problems listed in ids (all problems
 * when ids == NULL).  x, grad: batch x n x dim; scalars: batch x 3 = {loss, kinetic, mismatch};
 * diverged_step (may be NULL): batch entries, -1 = finite, else DivergedError's timestep.  Only the
 * listed problems' entries are read and written. */
int lms_batch_eval(lms_system* sys, size_t count, const int* ids, const double* x, double* grad, double* scalars,
                   int* diverged_step);

/* q(1) of every problem after the last evaluation: batch x n x dim. */
int lms_batch_final_q(lms_system* sys, double* out);

/* register_impl core (registration.cpp:43-93) for every problem of the batch: each problem runs its own
 * minimize (lbfgs.hpp:81-82) on a host thread; concurrent objective calls are coalesced into one batched
 * device evaluation per round.  momenta_out / warped_out: batch x n x dim; results / status: batch entries
 * (status = LMS_OK, LMS_ERR_DIVERGED or LMS_ERR_NUMERICAL per problem).  At most LMS_BATCH_REGISTER_MAX problems
 * per call (LMS_ERR_INVALID beyond).  From 32 problems on the population is evaluated in two alternating groups, so
 * that the host-side L-BFGS arithmetic of one group overlaps the device evaluation of the other (LMS_BATCH_GROUPS in
 * the environment overrides the group count); *rounds_out counts the batched device evaluations of all groups. */
#define LMS_BATCH_REGISTER_MAX 4096 /* problems per lms_batch_register call (one host thread each) */
int lms_batch_register(lms_system* sys, const lms_lbfgs_params* params, double* momenta_out, double* warped_out,
                       lms_minimize_result* results, int* status, int* rounds_out);

/* ---- multi-GPU row partition (no counterpart in the single-process reference) ---- */

/* Rank `rank` of `world` owns the contiguous row block [n*rank/world, n*(rank+1)/world) rounded to
 * row tiles (the chunk formula of parallel.cpp:145-146) and all-gathers its slice of the updated
 * state after every time step over NCCL.  unique_id is the 128-byte ncclUniqueId produced by
 * lms_comm_unique_id() on rank 0 and broadcast by the caller. */
int lms_comm_unique_id(unsigned char id[128]);
/* The partition itself (host arithmetic, no device needed): every rank owns `slice` rows of a plane padded
 * to `stride` = slice * world; the live rows of `rank` are [row_begin, row_end). */
int lms_row_partition(size_t n, int world, int rank, long long* slice, long long* stride, long long* row_begin,
                      long long* row_end);
int lms_system_comm_init(lms_system* sys, const unsigned char id[128], int rank, int world);

/* Loopback transport for the same row partition: `world` ranks are handles in ONE process (one host thread
 * each, typically on one GPU); the per-step exchange is a rendezvous plus device-to-device copies instead of
 * NCCL.  Same schedule, same slice layout; it lets a single-GPU machine run the partitioned evaluation with
 * world > 1.  Every rank must call lms_objective_eval concurrently from its own thread. */
typedef struct lms_local_group lms_local_group;
int lms_local_group_create(int world, lms_local_group** out);
void lms_local_group_destroy(lms_local_group* group);
int lms_system_join_local_group(lms_system* sys, lms_local_group* group, int rank);

/* Peer-push transport for the same row partition: instead of an all-gather after every time step, the kernels'
 * epilogues store each updated row straight into every peer's memory (NVLink peer stores between GPUs; CUDA IPC
 * mappings between processes) while the rest of the step is still being computed, and only a 4-byte arrival flag
 * per peer is exchanged in stream order (cuStreamWriteValue32 / cuStreamWaitValue32).  Up to 8 ranks.
 *   1. every rank:  lms_p2p_export(sys, rank, world, blob)      -- lays the handle out for `world` ranks
 *   2. the application all-gathers the `world` blobs (rank-major, LMS_P2P_BLOB_BYTES each)
 *   3. every rank:  lms_p2p_connect(sys, blobs)                 -- then lms_bind_registration / lms_objective_eval
 * Ranks may be processes (one per GPU, or several on one GPU) or handles of one process. */
#define LMS_P2P_BLOB_BYTES 128
int lms_p2p_export(lms_system* sys, int rank, int world, unsigned char blob[LMS_P2P_BLOB_BYTES]);
int lms_p2p_connect(lms_system* sys, const unsigned char* blobs);

/* ---- synthetic inputs (synth.hpp:15-43, rng.hpp) ---- */

/* Rng(seed).normal() / uniform() streams (rng.hpp:19-41; std::mt19937_64). */
void lms_rng_normals(uint64_t seed, size_t count, double* out);
void lms_rng_uniforms(uint64_t seed, size_t count, double* out);
/* Fibonacci-sphere template of diameter `extent` (synth.hpp:20,33-35; formula: SURVEY.md §8d). */
void lms_synth_sphere(size_t n, double extent, double* out /* n x 3 */);

#ifdef __cplusplus
}
#endif
#endif /* LMSHOOT_B200_H */
