// Device-resident L-BFGS: the same decision logic as the host driver (lbfgs_core.hpp,
// i.e. the reference's lbfgs.cpp:186-282), with x, g, d, the trial point and the curvature pairs living in HBM.
// Per objective evaluation nothing but three scalars crosses the bus (lms_objective_eval_device); per dot
// product one double.  At N = 20 000 the host driver's strictly sequential 60 000-element sums cost ~2 ms per
// iteration next to an 8 ms evaluation; here a dot is one kernel plus one 8-byte read-back.
//
// Sums are deterministic (fixed block assignment, fixed trees, ascending final sum) but not in the reference's
// strictly sequential order, so iterates agree with the host driver to rounding, not bit for bit.
#include <cuda_runtime.h>

#include <cstring>
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

// The whole two-loop recursion in ONE launch (single CTA, so the 2m dependent dot products need no host round
// trip): d = -H g, out[0] = g.d.  Dots: per-thread strided partial + fixed shared-memory tree (deterministic).
constexpr int kMaxPairs = 32;
constexpr int kLoopThreads = 1024;
struct PairSet {
  const double* s[kMaxPairs];
  const double* y[kMaxPairs];
  double rho[kMaxPairs];
  int m;
};

__device__ double block_dot(const double* a, const double* b, size_t n, double* scratch)
{
  double t = 0.0;
  for (size_t i = threadIdx.x; i < n; i += kLoopThreads) t = fma(a[i], b[i], t);
  scratch[threadIdx.x] = t;
  __syncthreads();
  for (int h = kLoopThreads / 2; h >= 1; h >>= 1) {
    if (threadIdx.x < h) scratch[threadIdx.x] += scratch[threadIdx.x + h];
    __syncthreads();
  }
  const double r = scratch[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kLoopThreads) two_loop_kernel(PairSet ps, double gamma, const double* __restrict__ g,
                                                                double* __restrict__ d, size_t n,
                                                                double* __restrict__ out)
{
  __shared__ double scratch[kLoopThreads];
  __shared__ double coef[kMaxPairs];
  for (size_t i = threadIdx.x; i < n; i += kLoopThreads) d[i] = g[i];
  __syncthreads();
  for (int k = ps.m - 1; k >= 0; --k) {
    const double a = ps.rho[k] * block_dot(ps.s[k], d, n, scratch);
    if (threadIdx.x == 0) coef[k] = a;
    for (size_t i = threadIdx.x; i < n; i += kLoopThreads) d[i] = fma(-a, ps.y[k][i], d[i]);
    __syncthreads();
  }
  for (size_t i = threadIdx.x; i < n; i += kLoopThreads) d[i] *= gamma;
  __syncthreads();
  for (int k = 0; k < ps.m; ++k) {
    const double b = ps.rho[k] * block_dot(ps.y[k], d, n, scratch);
    const double c = coef[k] - b;
    for (size_t i = threadIdx.x; i < n; i += kLoopThreads) d[i] = fma(c, ps.s[k][i], d[i]);
    __syncthreads();
  }
  for (size_t i = threadIdx.x; i < n; i += kLoopThreads) d[i] = -d[i];
  __syncthreads();
  const double slope = block_dot(g, d, n, scratch);
  if (threadIdx.x == 0) out[0] = slope;
}

// out[0..2] = s.y, s.s, y.y in one launch (single CTA)
__global__ void __launch_bounds__(kLoopThreads) pair_stats_kernel(const double* __restrict__ s,
                                                                  const double* __restrict__ y, size_t n,
                                                                  double* __restrict__ out)
{
  __shared__ double scratch[kLoopThreads];
  const double sy = block_dot(s, y, n, scratch);
  const double ss = block_dot(s, s, n, scratch);
  const double yy = block_dot(y, y, n, scratch);
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

struct DeviceOps {
  using Vec = double*;
  size_t n;
  lms::SystemBase* sys;
  cudaStream_t stream;
  double* partials = nullptr;
  unsigned* counter = nullptr;
  double* h_out = nullptr;  // mapped pinned: 3 doubles
  double* d_out = nullptr;  // its device alias
  std::vector<Vec> pool;

  void check(cudaError_t e)
  {
    if (e != cudaSuccess) throw lms::CudaFailure{e, "device_lbfgs", __LINE__};
  }
  void init()
  {
    check(cudaMalloc(&partials, 3 * kRedBlocks * sizeof(double)));
    check(cudaMalloc(&counter, sizeof(unsigned)));
    check(cudaMemset(counter, 0, sizeof(unsigned)));
    check(cudaHostAlloc(&h_out, 3 * sizeof(double), cudaHostAllocMapped));
    check(cudaHostGetDevicePointer(&d_out, h_out, 0));
  }
  void destroy()
  {
    for (Vec v : pool) cudaFree(v);
    if (partials) cudaFree(partials);
    if (counter) cudaFree(counter);
    if (h_out) cudaFreeHost(h_out);
  }
  int blocks() const { return (int)((n + 255) / 256); }

  Vec make()
  {
    if (!pool.empty()) {
      Vec v = pool.back();
      pool.pop_back();
      return v;
    }
    Vec v = nullptr;
    check(cudaMalloc(&v, (n ? n : 1) * sizeof(double)));
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
    reduce3_kernel<<<nb, kRedThreads, 0, stream>>>(a, b, n, partials, counter, d_out);
    check(cudaGetLastError());
    check(cudaStreamSynchronize(stream));
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
    two_loop_kernel<<<1, kLoopThreads, 0, stream>>>(ps, gamma, g, d, n, d_out);
    check(cudaGetLastError());
    check(cudaStreamSynchronize(stream));
    return h_out[0];
  }
  void pair_stats(Vec s, Vec y, double* sy, double* ss, double* yy)
  {
    if (n == 0) {
      *sy = *ss = *yy = 0.0;
      return;
    }
    pair_stats_kernel<<<1, kLoopThreads, 0, stream>>>(s, y, n, d_out);
    check(cudaGetLastError());
    check(cudaStreamSynchronize(stream));
    *sy = h_out[0];
    *ss = h_out[1];
    *yy = h_out[2];
  }
  double objective(Vec x, Vec grad)
  {
    double sc[3] = {0, 0, 0};
    sys->eval(x, grad, sc, true);  // throws lms::StatusError (e.g. LMS_ERR_DIVERGED) to abort, like DivergedError
    return sc[0];
  }
};

}  // namespace

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
    ops.init();
    std::vector<double> x0(nd ? nd : 1);
    for (size_t e = 0; e < nd; ++e) x0[e] = (s->host_target[e] - s->host_q0[e]) / s->timesteps;  // registration.cpp:47-52
    double* x = ops.make();
    double* g = ops.make();
    ops.check(cudaMemcpyAsync(x, x0.data(), nd * sizeof(double), cudaMemcpyHostToDevice, ops.stream));
    rc = lms::minimize_core(ops, x, g, *params, result, hist_loss, nullptr, nullptr, nullptr);
    if (rc == LMS_OK) {
      ops.check(cudaMemcpyAsync(momenta_out, x, nd * sizeof(double), cudaMemcpyDeviceToHost, ops.stream));
      ops.check(cudaStreamSynchronize(ops.stream));
      if (warped_out) {
        double sc[3];
        s->eval(x, g, sc, true);  // final re-integration under p0* (registration.cpp:85-93)
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
  ops.destroy();
  return rc;
}
