// Host-side L-BFGS driver: the library's own implementation of the optimiser contract in the reference's
// lbfgs.hpp:11-82 (behaviour: lbfgs.cpp:186-282), host vectors.  The hot path is a drop-in behind
// lmshoot::Objective, so a deployment keeps the reference's minimize(); this driver exists so that the library
// can run and time whole registrations by itself and is checked iterate-for-iterate against the reference's
// minimize in tests/test_lbfgs.py.  To make that comparison exact the vector operations below keep the
// reference's association order (strictly sequential dot products, x + a*d, ...).  The algorithm itself lives in
// lbfgs_core.hpp and is shared with the device-resident driver.
#include <cstddef>
#include <cstring>
#include <vector>

#include "lbfgs_core.hpp"

namespace {

struct HostOps {
  using Vec = double*;
  size_t n;
  lms_objective_fn fn;
  void* user;

  Vec make() { return new double[n ? n : 1]; }
  void release(Vec v) { delete[] v; }
  void copy(Vec dst, Vec src) { std::memcpy(dst, src, n * sizeof(double)); }
  double dot(Vec a, Vec b)
  {
    double s = 0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
  }
  double max_abs(Vec v)
  {
    double m = 0;
    for (size_t i = 0; i < n; ++i) m = std::max(m, std::abs(v[i]));
    return m;
  }
  bool all_finite(Vec v)
  {
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(v[i])) return false;
    return true;
  }
  void axpy_to(Vec out, Vec x, double a, Vec d)
  {
    for (size_t i = 0; i < n; ++i) out[i] = x[i] + a * d[i];
  }
  void sub_scaled(Vec d, double a, Vec y)
  {
    for (size_t i = 0; i < n; ++i) d[i] -= a * y[i];
  }
  void add_scaled(Vec d, double c, Vec s)
  {
    for (size_t i = 0; i < n; ++i) d[i] += c * s[i];
  }
  void scale(Vec d, double g)
  {
    for (size_t i = 0; i < n; ++i) d[i] *= g;
  }
  void negate(Vec d)
  {
    for (size_t i = 0; i < n; ++i) d[i] = -d[i];
  }
  void neg_copy(Vec d, Vec g)
  {
    for (size_t i = 0; i < n; ++i) d[i] = -g[i];
  }
  void take_step(Vec s, Vec y, Vec x, double step, Vec d, Vec g_new, Vec g)
  {
    for (size_t i = 0; i < n; ++i) {
      s[i] = step * d[i];
      y[i] = g_new[i] - g[i];
      x[i] += s[i];
    }
  }
  double dot_if_finite(Vec a, Vec b) { return all_finite(a) ? dot(a, b) : 0.0; }
  double two_loop(const std::vector<Vec>& hs, const std::vector<Vec>& hy, const std::vector<double>& rho, double gamma,
                  Vec g, Vec d, std::vector<double>& coef)
  {
    return lms::two_loop_generic(*this, hs, hy, rho, gamma, g, d, coef);
  }
  void pair_stats(Vec s, Vec y, double* sy, double* ss, double* yy)
  {
    *sy = dot(s, y);
    *ss = dot(s, s);
    *yy = dot(y, y);
  }
  double objective(Vec x, Vec grad) { return fn(user, x, grad, n); }
};

}  // namespace

extern "C" {

void lms_lbfgs_default_params(lms_lbfgs_params* p)
{
  if (!p) return;
  p->memory = 10;  // lbfgs.hpp:12-17
  p->max_iter = 100;
  p->grad_tol = 1e-6;
  p->c1 = 1e-4;
  p->c2 = 0.9;
  p->max_line_search = 20;
}

int lms_minimize(lms_objective_fn fn, void* user, size_t n, const double* x0, const lms_lbfgs_params* params,
                 double* x_out, double* grad_out, lms_minimize_result* result, double* hist_loss,
                 double* hist_grad_inf_norm, double* hist_step, int* hist_evals)
{
  if (!fn || !params || !result || (n && (!x0 || !x_out || !grad_out))) return LMS_ERR_INVALID;
  if (!lms::lbfgs_params_valid(*params)) return LMS_ERR_INVALID;
  HostOps ops{n, fn, user};
  std::vector<double> x(x0, x0 + n), g(n ? n : 1);
  if (x.empty()) x.resize(1);
  const int rc = lms::minimize_core(ops, x.data(), g.data(), *params, result, hist_loss, hist_grad_inf_norm,
                                    hist_step, hist_evals);
  if (rc == LMS_OK && n) {
    std::memcpy(x_out, x.data(), n * sizeof(double));
    std::memcpy(grad_out, g.data(), n * sizeof(double));
  }
  return rc;
}

}  // extern "C"
