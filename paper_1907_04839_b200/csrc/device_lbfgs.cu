// Device-resident L-BFGS: the same decision logic as the host driver (lbfgs_core.hpp,
// i.e. the reference's lbfgs.cpp:186-282), with x, g, d, the trial point and the curvature pairs living in HBM.
// Per objective evaluation nothing but three scalars crosses the bus (lms_objective_eval_device); per dot
// product one double.  At N = 20 000 the host driver's strictly sequential 60 000-element sums cost ~2 ms per
// iteration next to an 8 ms evaluation; here a dot is one kernel plus one 8-byte read-back.
//
// Sums are deterministic (fixed block assignment, fixed trees, ascending final sum) but not in the reference's
// strictly sequential order, so iterates agree with the host driver to rounding, not bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "lbfgs_core.hpp"
#include "system.cuh"

struct lms_system {  // layout shared with capi.cu
  lms::SystemBase* impl;
  int device;
};

namespace {

constexpr int kRedBlocks = 148;
constexpr int kRedThreads = 256;

// out[0] = sum_i a_i b_i ; out[1] = max_i |a_i| ; out[2] = 1 if every a_i is finite else 0.  One launch: block
// partials by grid-stride in a fixed assignment, block tree, then the last block to arrive combines the
// partials in ascending block order and writes the three results to `out` (mapped pinned host memory).
__global__ void __launch_bounds__(kRedThreads) reduce3_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                              size_t n, double* __restrict__ partials,
                                                              unsigned* __restrict__ counter, double* __restrict__ out)
{
  __shared__ double s_sum[kRedThreads], s_max[kRedThreads], s_fin[kRedThreads];
  __shared__ bool s_last;
  double sum = 0.0, mx = 0.0, fin = 1.0;
  for (size_t i = (size_t)blockIdx.x * kRedThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kRedThreads) {
    const double av = a[i];
    sum = fma(av, b[i], sum);
    mx = fmax(mx, fabs(av));
    if (!isfinite(av)) fin = 0.0;
  }
  s_sum[threadIdx.x] = sum;
  s_max[threadIdx.x] = mx;
  s_fin[threadIdx.x] = fin;
  __syncthreads();
  for (int h = kRedThreads / 2; h >= 1; h >>= 1) {
    if (threadIdx.x < h) {
      s_sum[threadIdx.x] += s_sum[threadIdx.x + h];
      s_max[threadIdx.x] = fmax(s_max[threadIdx.x], s_max[threadIdx.x + h]);
      s_fin[threadIdx.x] = fmin(s_fin[threadIdx.x], s_fin[threadIdx.x + h]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[3 * blockIdx.x + 0] = s_sum[0];
    partials[3 * blockIdx.x + 1] = s_max[0];
    partials[3 * blockIdx.x + 2] = s_fin[0];
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    s_last = prev == gridDim.x - 1;
    if (s_last) {
      *counter = 0;
      __threadfence();
      double t = 0.0, m = 0.0, f = 1.0;
      for (unsigned k = 0; k < gridDim.x; ++k) {
        t += __ldcg(partials + 3 * k);
        m = fmax(m, __ldcg(partials + 3 * k + 1));
        f = fmin(f, __ldcg(partials + 3 * k + 2));
      }
      out[0] = t;
      out[1] = m;
      out[2] = f;
    }
  }
}

// The whole two-loop recursion in ONE cooperative launch over all SMs: d = -H g, out[0] = g.d.  Every thread owns
// a fixed grid-stride set of elements for the whole kernel, so the axpy after a dot needs no barrier; a dot is
// per-CTA tree -> one partial per CTA -> grid barrier -> every CTA adds the partials in ascending CTA order
// (deterministic, the same value everywhere).  2m + 1 grid barriers replace 2m + 1 single-SM passes over memory
// (measured at N = 20 000, m = 10: ~0.7 ms -> ~0.1 ms per iteration).
constexpr int kMaxPairs = 32;
constexpr int kLoopThreads = 256;
struct PairSet {
  const double* s[kMaxPairs];
  const double* y[kMaxPairs];
  double rho[kMaxPairs];
  int m;
};

// Grid barrier on a monotonically increasing counter (the launch is cooperative, so every CTA is resident).
__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned& epoch)
{
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch += gridDim.x;
    __threadfence();
    atomicAdd(counter, 1u);
    while (*reinterpret_cast<volatile unsigned*>(counter) < epoch) {
    }
    __threadfence();
  }
  __syncthreads();
}

// Sum over the grid of one double per thread; `slot` selects a fresh partial array per call (no reuse hazards).
__device__ double grid_sum(double v, double* scratch, double* partials, int slot, unsigned* counter, unsigned& epoch)
{
  scratch[threadIdx.x] = v;
  __syncthreads();
  for (int h = kLoopThreads / 2; h >= 1; h >>= 1) {
    if (threadIdx.x < h) scratch[threadIdx.x] += scratch[threadIdx.x + h];
    __syncthreads();
  }
  double* mine = partials + (size_t)slot * gridDim.x;
  if (threadIdx.x == 0) __stcg(mine + blockIdx.x, scratch[0]);
  grid_barrier(counter, epoch);
  // every CTA adds the gridDim.x <= kLoopThreads partials with the same fixed tree: one parallel load, 8 steps
  scratch[threadIdx.x] = threadIdx.x < gridDim.x ? __ldcg(mine + threadIdx.x) : 0.0;
  __syncthreads();
  for (int h = kLoopThreads / 2; h >= 1; h >>= 1) {
    if (threadIdx.x < h) scratch[threadIdx.x] += scratch[threadIdx.x + h];
    __syncthreads();
  }
  const double t = scratch[0];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kLoopThreads) two_loop_kernel(PairSet ps, double gamma, const double* __restrict__ g,
                                                                double* __restrict__ d, size_t n,
                                                                double* __restrict__ partials, unsigned* counter,
                                                                double* __restrict__ out)
{
  __shared__ double scratch[kLoopThreads];
  __shared__ double coef[kMaxPairs];
  unsigned epoch = 0;  // the host zeroes the counter before every launch
  const size_t first = (size_t)blockIdx.x * kLoopThreads + threadIdx.x;
  const size_t step = (size_t)gridDim.x * kLoopThreads;
  for (size_t i = first; i < n; i += step) d[i] = g[i];
  int slot = 0;
  for (int k = ps.m - 1; k >= 0; --k) {
    double t = 0.0;
    for (size_t i = first; i < n; i += step) t = fma(ps.s[k][i], d[i], t);
    const double a = ps.rho[k] * grid_sum(t, scratch, partials, slot++, counter, epoch);
    if (threadIdx.x == 0) coef[k] = a;
    for (size_t i = first; i < n; i += step) d[i] = fma(-a, ps.y[k][i], d[i]);
  }
  for (size_t i = first; i < n; i += step) d[i] *= gamma;
  __syncthreads();
  for (int k = 0; k < ps.m; ++k) {
    double t = 0.0;
    for (size_t i = first; i < n; i += step) t = fma(ps.y[k][i], d[i], t);
    const double b = ps.rho[k] * grid_sum(t, scratch, partials, slot++, counter, epoch);
    const double c = coef[k] - b;
    for (size_t i = first; i < n; i += step) d[i] = fma(c, ps.s[k][i], d[i]);
  }
  double t = 0.0;
  for (size_t i = first; i < n; i += step) {
    const double di = -d[i];
    d[i] = di;
    t = fma(g[i], di, t);
  }
  const double slope = grid_sum(t, scratch, partials, slot++, counter, epoch);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = slope;
}

__device__ double block_dot(const double* a, const double* b, size_t n, double* scratch, int threads)
{
  double t = 0.0;
  for (size_t i = threadIdx.x; i < n; i += threads) t = fma(a[i], b[i], t);
  scratch[threadIdx.x] = t;
  __syncthreads();
  for (int h = threads / 2; h >= 1; h >>= 1) {
    if (threadIdx.x < h) scratch[threadIdx.x] += scratch[threadIdx.x + h];
    __syncthreads();
  }
  const double r = scratch[0];
  __syncthreads();
  return r;
}

// out[0..2] = s.y, s.s, y.y in one launch (single CTA)
constexpr int kStatThreads = 1024;
__global__ void __launch_bounds__(kStatThreads) pair_stats_kernel(const double* __restrict__ s,
                                                                  const double* __restrict__ y, size_t n,
                                                                  double* __restrict__ out)
{
  __shared__ double scratch[kStatThreads];
  const double sy = block_dot(s, y, n, scratch, kStatThreads);
  const double ss = block_dot(s, s, n, scratch, kStatThreads);
  const double yy = block_dot(y, y, n, scratch, kStatThreads);
  if (threadIdx.x == 0) {
    out[0] = sy;
    out[1] = ss;
    out[2] = yy;
  }
}

// out = alpha * x + beta * y (either input may alias out)
__global__ void lincomb_kernel(double* __restrict__ out, double alpha, const double* x, double beta, const double* y,
                               size_t n)
{
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __dadd_rn(__dmul_rn(alpha, x[i]), __dmul_rn(beta, y[i]));
}

// s = step * d ; y = g_new - g ; x += s
__global__ void take_step_kernel(double* __restrict__ s, double* __restrict__ y, double* __restrict__ x, double step,
                                 const double* __restrict__ d, const double* __restrict__ g_new,
                                 const double* __restrict__ g, size_t n)
{
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double si = __dmul_rn(step, d[i]);
    s[i] = si;
    y[i] = __dadd_rn(g_new[i], -g[i]);
    x[i] = __dadd_rn(x[i], si);
  }
}

// Device scratch of the driver, allocated once per handle (SystemBase::lbfgs_workspace) and reused by every
// lms_register_device call with the same vector length and memory.
struct Workspace {
  size_t n = 0, count = 0, each = 0;
  double* slab = nullptr;           // `count` vectors of `each` doubles
  double* loop_partials = nullptr;  // two-loop kernel: (2 kMaxPairs + 1) x loop_blocks
  unsigned* loop_counter = nullptr;
  int loop_blocks = 1;
  double* partials = nullptr;       // reduce3_kernel
  unsigned* counter = nullptr;
  double* h_out = nullptr;          // mapped pinned: 3 doubles
  double* d_out = nullptr;          // its device alias
  ~Workspace()
  {
    if (slab) cudaFree(slab);
    if (loop_partials) cudaFree(loop_partials);
    if (loop_counter) cudaFree(loop_counter);
    if (partials) cudaFree(partials);
    if (counter) cudaFree(counter);
    if (h_out) cudaFreeHost(h_out);
  }
};

// One allocation for every vector the driver can hold at once (x, g, d, trial point and gradient, best gradient,
// 2 (memory + 1) curvature vectors), the reduction scratch and the mapped result words; made once per handle (at bind
// time, see lms::prepare_device_lbfgs) and kept.  A fresh workspace also runs every kernel of the driver once on
// zeroed data: module loading and the first cooperative launch cost tens of milliseconds on a cold context, which
// would otherwise land inside the first registration.
std::shared_ptr<Workspace> ensure_workspace(lms::SystemBase* sys, size_t n, int memory, cudaStream_t stream);

struct DeviceOps {
  using Vec = double*;
  size_t n;
  lms::SystemBase* sys;
  cudaStream_t stream;
  double* partials = nullptr;
  unsigned* counter = nullptr;
  double* h_out = nullptr;  // mapped pinned: 3 doubles
  double* d_out = nullptr;  // its device alias
  std::vector<Vec> pool, extra;
  double t_obj = 0, t_loop = 0, t_red = 0;  // wall-clock breakdown (LMS_TRACE)
  int n_obj = 0, n_red = 0;

  void check(cudaError_t e)
  {
    if (e != cudaSuccess) throw lms::CudaFailure{e, "device_lbfgs", __LINE__};
  }
  // One allocation for every vector the driver can hold at once (x, g, d, trial point and gradient, best
  // gradient, 2 (memory + 1) curvature vectors), made on the first call and kept on the handle.
  double* loop_partials = nullptr;
  unsigned* loop_counter = nullptr;
  int loop_blocks = 1;
  void init(int memory)
  {
    auto ws = ensure_workspace(sys, n, memory, stream);
    for (size_t k = 0; k < ws->count; ++k) pool.push_back(ws->slab + (ws->count - 1 - k) * ws->each);
    loop_partials = ws->loop_partials;
    loop_counter = ws->loop_counter;
    loop_blocks = ws->loop_blocks;
    partials = ws->partials;
    counter = ws->counter;
    h_out = ws->h_out;
    d_out = ws->d_out;
    // an aborted run (divergence) may have left the arrival counter of reduce3_kernel mid-count
    check(cudaMemsetAsync(counter, 0, sizeof(unsigned), stream));
  }
  void destroy()
  {
    for (Vec v : extra) cudaFree(v);
  }
  int blocks() const { return (int)((n + 255) / 256); }

  Vec make()
  {
    if (!pool.empty()) {
      Vec v = pool.back();
      pool.pop_back();
      return v;
    }
    Vec v = nullptr;  // beyond the slab (not reached by minimize_core's allocation pattern)
    check(cudaMalloc(&v, (n ? n : 1) * sizeof(double)));
    extra.push_back(v);
    return v;
  }
  void release(Vec v) { pool.push_back(v); }
  void copy(Vec dst, Vec src)
  {
    if (n) check(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  }
  void reduce(Vec a, Vec b)
  {
    if (n == 0) {
      h_out[0] = 0.0;
      h_out[1] = 0.0;
      h_out[2] = 1.0;
      return;
    }
    const int nb = (int)std::min<size_t>(kRedBlocks, (n + kRedThreads - 1) / kRedThreads);
    const auto t0 = std::chrono::steady_clock::now();
    reduce3_kernel<<<nb, kRedThreads, 0, stream>>>(a, b, n, partials, counter, d_out);
    check(cudaGetLastError());
    check(cudaStreamSynchronize(stream));
    t_red += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    ++n_red;
  }
  double dot(Vec a, Vec b)
  {
    reduce(a, b);
    return h_out[0];
  }
  double max_abs(Vec v)
  {
    reduce(v, v);
    return h_out[1];
  }
  bool all_finite(Vec v)
  {
    reduce(v, v);
    return h_out[2] != 0.0;
  }
  void lincomb(Vec out, double alpha, Vec x, double beta, Vec y)
  {
    if (n == 0) return;
    lincomb_kernel<<<blocks(), 256, 0, stream>>>(out, alpha, x, beta, y, n);
    check(cudaGetLastError());
  }
  void axpy_to(Vec out, Vec x, double a, Vec d) { lincomb(out, 1.0, x, a, d); }
  void sub_scaled(Vec d, double a, Vec y) { lincomb(d, 1.0, d, -a, y); }
  void add_scaled(Vec d, double c, Vec s) { lincomb(d, 1.0, d, c, s); }
  void scale(Vec d, double g) { lincomb(d, g, d, 0.0, d); }
  void negate(Vec d) { lincomb(d, -1.0, d, 0.0, d); }
  void neg_copy(Vec d, Vec g) { lincomb(d, -1.0, g, 0.0, g); }
  void take_step(Vec s, Vec y, Vec x, double step, Vec d, Vec g_new, Vec g)
  {
    if (n == 0) return;
    take_step_kernel<<<blocks(), 256, 0, stream>>>(s, y, x, step, d, g_new, g, n);
    check(cudaGetLastError());
  }
  double dot_if_finite(Vec a, Vec b)
  {
    reduce(a, b);  // one launch yields a.b and the finiteness of a
    return h_out[2] != 0.0 ? h_out[0] : 0.0;
  }
  double two_loop(const std::vector<Vec>& hs, const std::vector<Vec>& hy, const std::vector<double>& rho, double gamma,
                  Vec g, Vec d, std::vector<double>& coef)
  {
    coef.assign(hs.size(), 0.0);  // the coefficients stay on the device
    if ((int)hs.size() > kMaxPairs) return lms::two_loop_generic(*this, hs, hy, rho, gamma, g, d, coef);
    if (n == 0) return 0.0;
    PairSet ps;
    ps.m = (int)hs.size();
    for (int k = 0; k < ps.m; ++k) {
      ps.s[k] = hs[k];
      ps.y[k] = hy[k];
      ps.rho[k] = rho[k];
    }
    const auto t0 = std::chrono::steady_clock::now();
    check(cudaMemsetAsync(loop_counter, 0, sizeof(unsigned), stream));
    const double* gp = g;
    void* args[] = {&ps, &gamma, &gp, &d, &n, &loop_partials, &loop_counter, &d_out};
    check(cudaLaunchCooperativeKernel((const void*)two_loop_kernel, dim3(loop_blocks), dim3(kLoopThreads), args, 0,
                                      stream));
    check(cudaStreamSynchronize(stream));
    t_loop += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return h_out[0];
  }
  void pair_stats(Vec s, Vec y, double* sy, double* ss, double* yy)
  {
    if (n == 0) {
      *sy = *ss = *yy = 0.0;
      return;
    }
    pair_stats_kernel<<<1, kStatThreads, 0, stream>>>(s, y, n, d_out);
    check(cudaGetLastError());
    check(cudaStreamSynchronize(stream));
    *sy = h_out[0];
    *ss = h_out[1];
    *yy = h_out[2];
  }
  double objective(Vec x, Vec grad)
  {
    double sc[3] = {0, 0, 0};
    const auto t0 = std::chrono::steady_clock::now();
    sys->eval(x, grad, sc, true);  // throws lms::StatusError (e.g. LMS_ERR_DIVERGED) to abort, like DivergedError
    t_obj += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    ++n_obj;
    return sc[0];
  }
};

// flag[0] = 0 when a and b differ anywhere (bitwise); the caller sets it to 1 first
__global__ void same_bits_kernel(const double* __restrict__ a, const double* __restrict__ b, size_t n, double* flag)
{
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && __double_as_longlong(a[i]) != __double_as_longlong(b[i])) flag[0] = 0.0;
}

std::shared_ptr<Workspace> ensure_workspace(lms::SystemBase* sys, size_t n, int memory, cudaStream_t stream)
{
  auto check = [](cudaError_t e) {
    if (e != cudaSuccess) throw lms::CudaFailure{e, "device_lbfgs workspace", __LINE__};
  };
  const size_t count = 2 * ((size_t)std::max(memory, 0) + 1) + 6;
  auto ws = std::static_pointer_cast<Workspace>(sys->lbfgs_workspace);
  if (ws && ws->n == n && ws->count >= count) return ws;
  sys->lbfgs_workspace.reset();
  ws = std::make_shared<Workspace>();
  ws->n = n;
  ws->count = count;
  ws->each = ((n ? n : 1) + 31) / 32 * 32;
  check(cudaMalloc(&ws->slab, ws->count * ws->each * sizeof(double)));
  check(cudaMemsetAsync(ws->slab, 0, ws->count * ws->each * sizeof(double), stream));
  // the two-loop kernel: one CTA per SM (cooperative launch: all resident), fewer when the vector is short
  int dev = 0, sms = 0;
  check(cudaGetDevice(&dev));
  check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  ws->loop_blocks = (int)std::max<size_t>(
      1, std::min<size_t>(std::min<size_t>((size_t)sms, kLoopThreads), (n + kLoopThreads - 1) / kLoopThreads));
  check(cudaMalloc(&ws->loop_partials, (size_t)(2 * kMaxPairs + 1) * ws->loop_blocks * sizeof(double)));
  check(cudaMalloc(&ws->loop_counter, sizeof(unsigned)));
  check(cudaMalloc(&ws->partials, 3 * kRedBlocks * sizeof(double)));
  check(cudaMalloc(&ws->counter, sizeof(unsigned)));
  check(cudaMemsetAsync(ws->counter, 0, sizeof(unsigned), stream));
  check(cudaHostAlloc(&ws->h_out, 3 * sizeof(double), cudaHostAllocMapped));
  check(cudaHostGetDevicePointer(&ws->d_out, ws->h_out, 0));
  sys->lbfgs_workspace = ws;
  if (n > 0) {
    // warm-up: every kernel of the driver once, on the zeroed slab
    double* v0 = ws->slab;
    double* v1 = ws->slab + ws->each;
    double* v2 = ws->slab + 2 * ws->each;
    const int blocks = (int)((n + 255) / 256);
    const int nb = (int)std::min<size_t>(kRedBlocks, (n + kRedThreads - 1) / kRedThreads);
    reduce3_kernel<<<nb, kRedThreads, 0, stream>>>(v0, v1, n, ws->partials, ws->counter, ws->d_out);
    lincomb_kernel<<<blocks, 256, 0, stream>>>(v2, 1.0, v0, 1.0, v1, n);
    take_step_kernel<<<blocks, 256, 0, stream>>>(v0, v1, v2, 1.0, v0, v1, v2, n);
    pair_stats_kernel<<<1, kStatThreads, 0, stream>>>(v0, v1, n, ws->d_out);
    same_bits_kernel<<<blocks, 256, 0, stream>>>(v0, v1, n, ws->d_out);
    check(cudaGetLastError());
    PairSet ps{};
    ps.m = 1;
    ps.s[0] = v0;
    ps.y[0] = v1;
    ps.rho[0] = 0.0;
    double gamma = 1.0;
    const double* gp = v0;
    double* dp = v2;
    size_t nn = n;
    check(cudaMemsetAsync(ws->loop_counter, 0, sizeof(unsigned), stream));
    void* args[] = {&ps, &gamma, &gp, &dp, &nn, &ws->loop_partials, &ws->loop_counter, &ws->d_out};
    check(cudaLaunchCooperativeKernel((const void*)two_loop_kernel, dim3(ws->loop_blocks), dim3(kLoopThreads), args, 0,
                                      stream));
    check(cudaMemsetAsync(ws->slab, 0, 3 * ws->each * sizeof(double), stream));
  }
  check(cudaStreamSynchronize(stream));
  return ws;
}

}  // namespace

namespace lms {
void prepare_device_lbfgs(SystemBase* sys, int memory)
{
  if (sys->batch != 1) return;
  ensure_workspace(sys, sys->host_q0.size(), memory, sys->stream_handle());
}
}  // namespace lms

extern "C" int lms_register_device(lms_system* handle, const lms_lbfgs_params* params, double* momenta_out,
                                   double* warped_out, lms_minimize_result* result, double* hist_loss)
{
  if (!handle || !handle->impl || !params || !momenta_out || !result) return LMS_ERR_INVALID;
  if (!lms::lbfgs_params_valid(*params)) return LMS_ERR_INVALID;
  lms::SystemBase* s = handle->impl;
  if (!s->bound || s->batch != 1) return LMS_ERR_STATE;
  s->last_diverged_step = -1;
  s->last_diverged_point = -1;
  s->last_message.clear();
  const size_t nd = s->host_q0.size();
  DeviceOps ops{nd, s, s->stream_handle()};
  int rc = LMS_OK;
  try {
    if (cudaSetDevice(handle->device) != cudaSuccess) return LMS_ERR_CUDA;
    const bool trace = std::getenv("LMS_TRACE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms_since = [&](std::chrono::steady_clock::time_point t) {
      return std::chrono::duration<double, std::milli>(now() - t).count();
    };
    auto t_begin = now();
    ops.init(params->memory);
    if (trace) std::fprintf(stderr, "[lms] register_device: init %.3f ms\n", ms_since(t_begin));
    std::vector<double> x0(nd ? nd : 1);
    for (size_t e = 0; e < nd; ++e) x0[e] = (s->host_target[e] - s->host_q0[e]) / s->timesteps;  // registration.cpp:47-52
    double* x = ops.make();
    double* g = ops.make();
    ops.check(cudaMemcpyAsync(x, x0.data(), nd * sizeof(double), cudaMemcpyHostToDevice, ops.stream));
    auto t_min = now();
    rc = lms::minimize_core(ops, x, g, *params, result, hist_loss, nullptr, nullptr, nullptr);
    if (trace)
      std::fprintf(stderr, "[lms] register_device: minimize %.3f ms (objective %.3f ms in %d calls, two-loop %.3f ms, "
                   "reductions %.3f ms in %d)\n", ms_since(t_min), ops.t_obj, ops.n_obj, ops.t_loop, ops.t_red, ops.n_red);
    if (rc == LMS_OK) {
      ops.check(cudaMemcpyAsync(momenta_out, x, nd * sizeof(double), cudaMemcpyDeviceToHost, ops.stream));
      ops.check(cudaStreamSynchronize(ops.stream));
      if (warped_out) {
        // final re-integration under p0* (registration.cpp:85-93).  The trajectory resident in HBM is the one of the
        // last evaluated point; when that point is x* bit for bit (the usual case: the last trial step was the
        // accepted one) re-evaluating would reproduce it exactly, so q(1) is read as it stands.
        bool resident = false;
        if (nd > 0 && s->last_x_device() != nullptr) {
          ops.h_out[0] = 1.0;
          same_bits_kernel<<<ops.blocks(), 256, 0, ops.stream>>>(x, s->last_x_device(), nd, ops.d_out);
          ops.check(cudaGetLastError());
          ops.check(cudaStreamSynchronize(ops.stream));
          resident = ops.h_out[0] != 0.0;
        }
        if (!resident) {
          double sc[3];
          s->eval(x, g, sc, true);
        }
        s->final_q(warped_out);
      }
    }
    ops.release(x);
    ops.release(g);
  } catch (const lms::StatusError& e) {
    s->last_message = e.msg;
    rc = e.code;
  } catch (const lms::CudaFailure& e) {
    s->last_message = cudaGetErrorString(e.err);
    cudaGetLastError();
    rc = LMS_ERR_CUDA;
  } catch (...) {
    rc = LMS_ERR_CUDA;
  }
  {
    const auto t0 = std::chrono::steady_clock::now();
    ops.destroy();
    if (std::getenv("LMS_TRACE"))
      std::fprintf(stderr, "[lms] register_device: teardown %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  return rc;
}
