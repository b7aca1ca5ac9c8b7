// extern "C" surface of liblmshoot_b200.so (include/lmshoot_b200.h).  Exceptions never cross it.
#include <cuda_runtime.h>

#include <condition_variable>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <random>
#include <thread>

#include "system.cuh"

struct lms_system {  // layout shared with device_lbfgs.cu
  lms::SystemBase* impl = nullptr;
  int device = 0;
};

namespace {

template <class Fn>
int guarded(lms_system* sys, Fn&& fn)
{
  if (!sys || !sys->impl) return LMS_ERR_STATE;
  lms::SystemBase* s = sys->impl;
  s->last_diverged_step = -1;
  s->last_diverged_point = -1;
  s->last_message.clear();
  try {
    cudaError_t e = cudaSetDevice(sys->device);
    if (e != cudaSuccess) throw lms::CudaFailure{e, "cudaSetDevice", __LINE__};
    fn(s);
    return LMS_OK;
  } catch (const lms::StatusError& e) {
    s->last_message = e.msg;
    return e.code;
  } catch (const lms::CudaFailure& e) {
    s->last_message = std::string(cudaGetErrorString(e.err)) + " in " + e.what;
    cudaGetLastError();
    return LMS_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    s->last_message = "host allocation failed";
    return LMS_ERR_CUDA;
  } catch (...) {
    s->last_message = "unexpected exception";
    return LMS_ERR_CUDA;
  }
}

}  // namespace

extern "C" {

const char* lms_status_string(int status)
{
  switch (status) {
    case LMS_OK: return "ok";
    case LMS_ERR_SHAPE: return "shape mismatch (lmshoot::ShapeError)";
    case LMS_ERR_DIVERGED: return "non-finite state (lmshoot::DivergedError)";
    case LMS_ERR_INVALID: return "invalid argument (std::invalid_argument)";
    case LMS_ERR_NUMERICAL: return "non-finite objective (lmshoot::NumericalError)";
    case LMS_ERR_CUDA: return "CUDA failure";
    case LMS_ERR_STATE: return "call order violated";
    case LMS_ERR_COMM: return "NCCL failure";
  }
  return "unknown status";
}

const char* lms_variant_name(int precision, int variant)
{
  return lms::variant_name(precision, variant);
}

const char* lms_system_kernel_names(const lms_system* sys)
{
  return sys && sys->impl ? sys->impl->kernel_names_.c_str() : "";
}

int lms_system_create(const lms_config* cfg, lms_system** out)
{
  if (!cfg || !out) return LMS_ERR_INVALID;
  *out = nullptr;
  if (cfg->dim != 2 && cfg->dim != 3) return LMS_ERR_SHAPE;  // shooting.hpp:358
  if (!(cfg->sigma > 0)) return LMS_ERR_INVALID;             // shooting.hpp:113
  if (cfg->precision != LMS_PRECISION_F32 && cfg->precision != LMS_PRECISION_F64) return LMS_ERR_INVALID;
  if (cfg->max_timesteps < 1) return LMS_ERR_INVALID;
  if (cfg->n > (size_t)0x7fffffff - 1024) return LMS_ERR_INVALID;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || cfg->device < 0 || cfg->device >= count) {
    cudaGetLastError();
    return LMS_ERR_CUDA;
  }
  lms_system* h = new (std::nothrow) lms_system;
  if (!h) return LMS_ERR_CUDA;
  h->device = cfg->device;
  try {
    h->impl = lms::create_system(*cfg);
  } catch (const lms::StatusError& e) {
    delete h;
    return e.code;
  } catch (...) {
    cudaGetLastError();
    delete h;
    return LMS_ERR_CUDA;
  }
  *out = h;
  return LMS_OK;
}

int lms_batch_create(const lms_config* cfg, size_t batch, lms_system** out)
{
  if (!cfg || !out || batch < 1 || batch > (size_t)1 << 20) return LMS_ERR_INVALID;
  *out = nullptr;
  if (cfg->dim != 2 && cfg->dim != 3) return LMS_ERR_SHAPE;
  if (!(cfg->sigma > 0)) return LMS_ERR_INVALID;
  if (cfg->precision != LMS_PRECISION_F32 && cfg->precision != LMS_PRECISION_F64) return LMS_ERR_INVALID;
  if (cfg->max_timesteps < 1) return LMS_ERR_INVALID;
  if (cfg->n * batch > (size_t)0x7fffffff - 1024) return LMS_ERR_INVALID;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || cfg->device < 0 || cfg->device >= count) {
    cudaGetLastError();
    return LMS_ERR_CUDA;
  }
  lms_system* h = new (std::nothrow) lms_system;
  if (!h) return LMS_ERR_CUDA;
  h->device = cfg->device;
  try {
    h->impl = lms::create_system(*cfg, (int)batch);
  } catch (const lms::StatusError& e) {
    delete h;
    return e.code;
  } catch (...) {
    cudaGetLastError();
    delete h;
    return LMS_ERR_CUDA;
  }
  *out = h;
  return LMS_OK;
}

size_t lms_batch_size(const lms_system* sys) { return sys && sys->impl ? (size_t)sys->impl->batch : 0; }

int lms_batch_eval(lms_system* sys, size_t count, const int* ids, const double* x, double* grad, double* scalars,
                   int* diverged_step)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->eval_batch(x, grad, scalars, diverged_step, (int)count, ids); });
}

int lms_batch_final_q(lms_system* sys, double* out)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->final_q_batch(out); });
}

void lms_system_destroy(lms_system* sys)
{
  if (!sys) return;
  delete sys->impl;
  delete sys;
}

int lms_last_diverged_step(const lms_system* sys) { return sys && sys->impl ? sys->impl->last_diverged_step : -1; }
long long lms_last_diverged_point(const lms_system* sys)
{
  return sys && sys->impl ? sys->impl->last_diverged_point : -1;
}
const char* lms_last_error_message(const lms_system* sys)
{
  return sys && sys->impl ? sys->impl->last_message.c_str() : "";
}

int lms_hamiltonian(lms_system* sys, const double* q, const double* p, double* out)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->hamiltonian(q, p, out); });
}

int lms_derivatives(lms_system* sys, const double* q, const double* p, double* hq, double* hp)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->derivatives(q, p, hq, hp); });
}

int lms_integrate_forward(lms_system* sys, const double* q0, const double* p0, int timesteps, double* traj_q,
                          double* traj_p)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->integrate_forward(q0, p0, timesteps, traj_q, traj_p); });
}

int lms_adjoint_step(lms_system* sys, const double* q, const double* p, const double* alpha, const double* beta,
                     double* d_alpha, double* d_beta)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->adjoint_step(q, p, alpha, beta, d_alpha, d_beta); });
}

int lms_mismatch_sq(lms_system* sys, const double* a, const double* b, double* out)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->mismatch_sq(a, b, out); });
}

int lms_bind_registration(lms_system* sys, const double* q0, const double* target, double lambda, int timesteps)
{
  return guarded(sys, [&](lms::SystemBase* s) {
    s->bind(q0, target, lambda, timesteps);
    // the device-resident optimiser's workspace (lms_register_device): allocated and warmed once per handle here,
    // not inside the first registration
    lms::prepare_device_lbfgs(s, 10 /* LbfgsParams::memory default, lbfgs.hpp:12 */);
  });
}

int lms_objective_eval(lms_system* sys, const double* x, double* grad, double* loss, double* kinetic,
                       double* mismatch)
{
  double sc[3] = {0, 0, 0};
  int rc = guarded(sys, [&](lms::SystemBase* s) { s->eval(x, grad, sc, false); });
  if (rc == LMS_OK) {
    if (loss) *loss = sc[0];
    if (kinetic) *kinetic = sc[1];
    if (mismatch) *mismatch = sc[2];
  }
  return rc;
}

int lms_objective_eval_device(lms_system* sys, const double* d_x, double* d_grad, double* scalars)
{
  double sc[3] = {0, 0, 0};
  int rc = guarded(sys, [&](lms::SystemBase* s) { s->eval(d_x, d_grad, sc, true); });
  if (rc == LMS_OK && scalars) std::memcpy(scalars, sc, sizeof(sc));
  return rc;
}

int lms_compute_gradient(lms_system* sys, const double* q0, const double* p0, const double* target, double lambda,
                         int timesteps, double* scalars, double* grad)
{
  return guarded(sys, [&](lms::SystemBase* s) {
    // the reference's entry point takes q0 / target / lambda / T on every call; binding uploads them and
    // captures the evaluation graph, so it is skipped when they are the ones already bound
    const size_t elems = s->cfg.n * (size_t)s->cfg.dim;
    const bool same = s->bound && s->batch == 1 && s->lambda == lambda && s->timesteps == timesteps &&
                      s->host_q0.size() == elems && s->host_target.size() == elems &&
                      std::memcmp(s->host_q0.data(), q0, elems * sizeof(double)) == 0 &&
                      std::memcmp(s->host_target.data(), target, elems * sizeof(double)) == 0;
    if (!same) s->bind(q0, target, lambda, timesteps);
    double sc[3] = {0, 0, 0};
    s->eval(p0, grad, sc, false);
    if (scalars) std::memcpy(scalars, sc, sizeof(sc));
  });
}

int lms_objective_final_q(lms_system* sys, double* out)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->final_q(out); });
}

int lms_registration_metrics(lms_system* sys, double* out)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->registration_metrics(out); });
}

double lms_last_eval_device_ms(const lms_system* sys) { return sys && sys->impl ? sys->impl->last_eval_ms : 0.0; }
int lms_last_eval_kernel_launches(const lms_system* sys)
{
  return sys && sys->impl ? sys->impl->last_eval_launches : 0;
}
int lms_set_kernel_timing(lms_system* sys, int enabled)
{
  if (!sys || !sys->impl) return LMS_ERR_STATE;
  sys->impl->kernel_timing = enabled != 0;
  return LMS_OK;
}
double lms_last_kernel_ms(const lms_system* sys, int which)
{
  if (!sys || !sys->impl || which < 0 || which > 1) return 0.0;
  return sys->impl->last_kernel_ms[which];
}

int lms_velocities(lms_system* sys, const double* q, const double* p, size_t m, const double* points, double* out)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->velocities(q, p, m, points, out); });
}

int lms_warp_points_stored(lms_system* sys, size_t m, const double* points, double* out)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->warp_stored(m, points, out); });
}

int lms_comm_unique_id(unsigned char id[128])
{
  const lms::NcclApi& nc = lms::nccl_api();
  if (!nc.ok) return LMS_ERR_COMM;
  lms::ncclUniqueId uid;
  if (nc.GetUniqueId(&uid) != 0) return LMS_ERR_COMM;
  std::memcpy(id, uid.internal, 128);
  return LMS_OK;
}

struct lms_local_group {
  lms::LocalGroup* impl;
};

int lms_local_group_create(int world, lms_local_group** out)
{
  if (!out || world < 1 || world > 64) return LMS_ERR_INVALID;
  *out = new (std::nothrow) lms_local_group{new (std::nothrow) lms::LocalGroup(world)};
  return *out && (*out)->impl ? LMS_OK : LMS_ERR_CUDA;
}

void lms_local_group_destroy(lms_local_group* group)
{
  if (!group) return;
  delete group->impl;
  delete group;
}

int lms_system_join_local_group(lms_system* sys, lms_local_group* group, int rank)
{
  if (!group) return LMS_ERR_INVALID;
  return guarded(sys, [&](lms::SystemBase* s) { s->join_local_group(group->impl, rank); });
}

int lms_row_partition(size_t n, int world, int rank, long long* slice, long long* stride, long long* row_begin,
                      long long* row_end)
{
  if (world < 1 || rank < 0 || rank >= world) return LMS_ERR_INVALID;
  const lms::RowPartition p = lms::partition_rows((long long)n, world, rank);
  if (slice) *slice = p.slice;
  if (stride) *stride = p.stride;
  if (row_begin) *row_begin = p.row_begin;
  if (row_end) *row_end = p.row_end;
  return LMS_OK;
}

int lms_system_comm_init(lms_system* sys, const unsigned char id[128], int rank, int world)
{
  return guarded(sys, [&](lms::SystemBase* s) { s->comm_init(id, rank, world); });
}

int lms_p2p_export(lms_system* sys, int rank, int world, unsigned char blob[LMS_P2P_BLOB_BYTES])
{
  if (!blob) return LMS_ERR_INVALID;
  return guarded(sys, [&](lms::SystemBase* s) { s->p2p_export(rank, world, blob); });
}

int lms_p2p_connect(lms_system* sys, const unsigned char* blobs)
{
  if (!blobs) return LMS_ERR_INVALID;
  return guarded(sys, [&](lms::SystemBase* s) { s->p2p_connect(blobs); });
}

// ---- register_impl core (registration.cpp:43-93) over the bound objective and lms_minimize ----
namespace {
struct BoundCall {
  lms_system* sys;
  std::vector<double> last_x;  // the point of the last evaluation: its trajectory is the one resident in HBM
};
}  // namespace

static double bound_objective(void* user, const double* x, double* grad, size_t n)
{
  BoundCall* call = static_cast<BoundCall*>(user);
  double loss = 0;
  int rc = lms_objective_eval(call->sys, x, grad, &loss, nullptr, nullptr);
  if (rc != LMS_OK) throw rc;  // unwinds through lms_minimize like DivergedError does through minimize
  call->last_x.assign(x, x + n);
  return loss;
}

int lms_register(lms_system* sys, const lms_lbfgs_params* params, double* momenta_out, double* warped_out,
                 lms_minimize_result* result, double* hist_loss)
{
  if (!sys || !sys->impl) return LMS_ERR_STATE;
  lms::SystemBase* s = sys->impl;
  if (!s->bound) return LMS_ERR_STATE;
  const size_t nd = s->host_q0.size();
  std::vector<double> x0(nd), g(nd);
  for (size_t e = 0; e < nd; ++e) x0[e] = (s->host_target[e] - s->host_q0[e]) / s->timesteps;  // registration.cpp:47-52
  int rc;
  BoundCall call{sys, {}};
  try {
    rc = lms_minimize(bound_objective, &call, nd, x0.data(), params, momenta_out, g.data(), result, hist_loss,
                      nullptr, nullptr, nullptr);
  } catch (int code) {
    return code;
  }
  if (rc != LMS_OK) return rc;
  // final re-integration under p0* (registration.cpp:85-93).  When the last evaluated point is p0* bit for bit (the
  // usual case: the last trial step was the accepted one) its trajectory is still resident and q(1) is read as it
  // stands; otherwise one more evaluation puts it there.
  if (call.last_x.size() != nd || std::memcmp(call.last_x.data(), momenta_out, nd * sizeof(double)) != 0) {
    double loss = 0;
    rc = lms_objective_eval(sys, momenta_out, g.data(), &loss, nullptr, nullptr);
    if (rc != LMS_OK) return rc;
  }
  return lms_objective_final_q(sys, warped_out);
}

// ---- population batches: one minimize per problem, objective calls coalesced per round ----
namespace {

// Every optimiser thread submits its trial point and sleeps; the last submitter of a round launches one batched
// evaluation for all waiting problems of its group and wakes them.  The drivers stay unchanged blocking callbacks.
// The population is cut into groups with a rendezvous each: while the GPU evaluates one group's round, the host
// threads of the other groups run their L-BFGS vector arithmetic (strictly sequential sums, the reference's order:
// ~0.3 ms per iteration and problem at N = 2000), so the device does not idle between rounds.  Evaluations of one
// handle are serialised by `eval_mutex`.
struct PinnedDoubles {  // staging the device copies read / write directly (pageable vectors cost ~1 ms per 6 MB copy)
  double* p = nullptr;
  size_t n = 0;
  bool pinned = false;
  PinnedDoubles() = default;
  PinnedDoubles(const PinnedDoubles&) = delete;
  PinnedDoubles& operator=(const PinnedDoubles&) = delete;
  void assign(size_t count)
  {
    n = count;
    if (cudaHostAlloc(&p, std::max<size_t>(count, 1) * sizeof(double), cudaHostAllocDefault) == cudaSuccess) {
      pinned = true;
    } else {
      cudaGetLastError();
      p = new double[std::max<size_t>(count, 1)];
    }
    std::memset(p, 0, std::max<size_t>(count, 1) * sizeof(double));
  }
  ~PinnedDoubles()
  {
    if (pinned) cudaFreeHost(p);
    else delete[] p;
  }
  double* data() { return p; }
};

struct Rendezvous {
  lms_system* sys;
  std::mutex* eval_mutex;  // one batched evaluation of the handle at a time
  size_t per;  // n * dim
  int batch = 0;  // problems of the handle (all groups)
  std::mutex m;
  std::condition_variable cv;
  int active = 0, submitted = 0, rounds = 0;
  unsigned long long round = 0;
  std::vector<int> waiting;  // problem ids submitted this round
  PinnedDoubles *x, *grad;   // full-batch staging shared by the groups (disjoint problem ranges)
  std::vector<double>* scalars;
  std::vector<int>* diverged;
  int failure = LMS_OK;  // a CUDA-level failure aborts everybody

  void run_round()  // caller holds the lock; everyone else of this group is asleep
  {
    // ascending ids: the device copies coalesce runs of neighbours; the whole population goes without an id list
    std::sort(waiting.begin(), waiting.end());
    const bool all = (int)waiting.size() == batch;
    int rc;
    {
      std::lock_guard<std::mutex> device(*eval_mutex);
      rc = lms_batch_eval(sys, all ? (size_t)batch : waiting.size(), all ? nullptr : waiting.data(), x->data(),
                          grad->data(), scalars->data(), diverged->data());
    }
    if (rc != LMS_OK) failure = rc;
    waiting.clear();
    submitted = 0;
    ++round;
    ++rounds;
    cv.notify_all();
  }
};

struct ProblemCtx {
  Rendezvous* rv;
  int id;
  int diverged_step = -1;
};

double batched_objective(void* user, const double* x, double* grad, size_t n)
{
  ProblemCtx* ctx = static_cast<ProblemCtx*>(user);
  Rendezvous& rv = *ctx->rv;
  std::unique_lock<std::mutex> lock(rv.m);
  std::memcpy(rv.x->data() + ctx->id * rv.per, x, n * sizeof(double));
  rv.waiting.push_back(ctx->id);
  ++rv.submitted;
  const unsigned long long my_round = rv.round;
  if (rv.submitted == rv.active)
    rv.run_round();
  else
    rv.cv.wait(lock, [&] { return rv.round != my_round || rv.failure != LMS_OK; });
  if (rv.failure != LMS_OK) throw rv.failure;
  if ((*rv.diverged)[ctx->id] >= 0) {
    ctx->diverged_step = (*rv.diverged)[ctx->id];
    throw (int)LMS_ERR_DIVERGED;  // aborts this problem's minimize, as DivergedError does in the reference
  }
  std::memcpy(grad, rv.grad->data() + ctx->id * rv.per, n * sizeof(double));
  return (*rv.scalars)[3 * ctx->id];
}

}  // namespace

int lms_batch_register(lms_system* sys, const lms_lbfgs_params* params, double* momenta_out, double* warped_out,
                       lms_minimize_result* results, int* status, int* rounds_out)
{
  if (!sys || !sys->impl || !params || !momenta_out || !results || !status) return LMS_ERR_INVALID;
  lms::SystemBase* s = sys->impl;
  if (!s->bound) return LMS_ERR_STATE;
  const int B = s->batch;
  // one blocking minimize per problem on its own host thread: bounded, so that a huge population cannot
  // exhaust the process (split it into several lms_batch_register calls, or use lms_batch_eval directly)
  if (B > LMS_BATCH_REGISTER_MAX) {
    s->last_message = "lms_batch_register: more problems than LMS_BATCH_REGISTER_MAX host threads";
    return LMS_ERR_INVALID;
  }
  const size_t per = s->host_q0.size() / (size_t)B;
  // groups of problems with a rendezvous each (see Rendezvous); LMS_BATCH_GROUPS overrides
  int groups = B >= 32 ? 2 : 1;
  if (const char* e = std::getenv("LMS_BATCH_GROUPS")) groups = std::max(1, std::min(std::atoi(e), B));
  std::mutex eval_mutex;
  PinnedDoubles x_all, grad_all;
  x_all.assign(per * B);
  grad_all.assign(per * B);
  std::vector<double> scalars_all(3 * (size_t)B, 0.0);
  std::vector<int> diverged_all(B, -1);
  std::vector<Rendezvous> rvs(groups);
  auto group_of = [&](int b) { return (int)((long long)b * groups / B); };  // contiguous, equal (+-1) ranges
  for (int g = 0; g < groups; ++g) {
    rvs[g].sys = sys;
    rvs[g].eval_mutex = &eval_mutex;
    rvs[g].per = per;
    rvs[g].batch = B;
    rvs[g].x = &x_all;
    rvs[g].grad = &grad_all;
    rvs[g].scalars = &scalars_all;
    rvs[g].diverged = &diverged_all;
  }
  for (int b = 0; b < B; ++b) ++rvs[group_of(b)].active;
  std::vector<ProblemCtx> ctx(B);
  std::vector<std::thread> threads;
  threads.reserve(B);
  for (int b = 0; b < B; ++b) {
    Rendezvous& rv = rvs[group_of(b)];
    ctx[b].rv = &rv;
    ctx[b].id = b;
    auto body = [&, b] {
      Rendezvous& mine = *ctx[b].rv;
      std::vector<double> x0(per), g(per);
      for (size_t e = 0; e < per; ++e)  // x0 = (target - q0)/T, registration.cpp:47-52
        x0[e] = (s->host_target[b * per + e] - s->host_q0[b * per + e]) / s->timesteps;
      int rc;
      try {
        rc = lms_minimize(batched_objective, &ctx[b], per, x0.data(), params, momenta_out + b * per, g.data(),
                          &results[b], nullptr, nullptr, nullptr, nullptr);
      } catch (int code) {
        rc = code;
      }
      status[b] = rc;
      std::unique_lock<std::mutex> lock(mine.m);
      --mine.active;  // this problem no longer takes part in rounds
      if (mine.failure == LMS_OK && mine.active > 0 && mine.submitted == mine.active) mine.run_round();
    };
    try {
      threads.emplace_back(body);
    } catch (...) {  // std::system_error: no more threads.  Wake and fail the ones already running.
      for (auto& r : rvs) {
        std::unique_lock<std::mutex> lock(r.m);
        r.failure = LMS_ERR_STATE;
        r.cv.notify_all();
      }
      break;
    }
  }
  for (auto& t : threads) t.join();
  int rounds_total = 0;
  for (auto& r : rvs) rounds_total += r.rounds;
  if (rounds_out) *rounds_out = rounds_total;
  for (auto& r : rvs)
    if (r.failure != LMS_OK) return r.failure;
  if (warped_out) {
    // final re-integration under every p0* (registration.cpp:85-93): one more batched evaluation
    std::vector<int> ok;
    for (int b = 0; b < B; ++b)
      if (status[b] == LMS_OK) ok.push_back(b);
    if (!ok.empty()) {
      const bool all = (int)ok.size() == B;
      int rc = lms_batch_eval(sys, ok.size(), all ? nullptr : ok.data(), momenta_out, grad_all.data(),
                              scalars_all.data(), diverged_all.data());
      if (rc != LMS_OK) return rc;
    }
    return lms_batch_final_q(sys, warped_out);
  }
  return LMS_OK;
}

#ifdef LMS_SMALL_TRACE
// measurement builds only (scripts/small_trace.py): the phase timestamps the persistent kernel left in the scratch
int lms_debug_read_trace(lms_system* sys, unsigned long long* out, size_t count)
{
  return guarded(sys, [&](lms::SystemBase* s) {
    if (cudaMemcpy(out, s->staging_scratch(), count * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
      throw lms::StatusError{LMS_ERR_CUDA, "trace read failed"};
  });
}
#endif

// ---- synthetic inputs ----
namespace {
// rng.hpp:14-48: mt19937_64 with the explicit uniform / Box-Muller transforms (pairs, spare kept).
struct Rng {
  explicit Rng(uint64_t seed) : engine(seed) {}
  double uniform() { return static_cast<double>(engine() >> 11) * 0x1.0p-53; }
  double normal()
  {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    double u1 = 0.0;
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
    spare = r * std::sin(theta);
    have_spare = true;
    return r * std::cos(theta);
  }
  std::mt19937_64 engine;
  bool have_spare = false;
  double spare = 0.0;
};
}  // namespace

void lms_rng_normals(uint64_t seed, size_t count, double* out)
{
  Rng rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng.normal();
}

void lms_rng_uniforms(uint64_t seed, size_t count, double* out)
{
  Rng rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng.uniform();
}

void lms_synth_sphere(size_t n, double extent, double* out)
{
  // Fibonacci sphere of diameter `extent`: z_i = 1 - 2(i+1/2)/n, theta_i = pi(3 - sqrt 5) i
  const double radius = 0.5 * extent;
  const double golden = 3.141592653589793238462643383279502884 * (3.0 - std::sqrt(5.0));
  for (size_t i = 0; i < n; ++i) {
    const double z = 1.0 - 2.0 * (double(i) + 0.5) / double(n);
    const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
    const double th = golden * double(i);
    out[3 * i + 0] = radius * r * std::cos(th);
    out[3 * i + 1] = radius * r * std::sin(th);
    out[3 * i + 2] = radius * z;
  }
}

}  // extern "C"
