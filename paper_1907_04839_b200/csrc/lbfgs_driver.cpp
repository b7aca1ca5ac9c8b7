// Host-side L-BFGS driver with a strong-Wolfe line search: the library's own implementation of the
// optimiser contract in the reference's lbfgs.hpp:11-82 (behaviour: lbfgs.cpp:186-282).  The hot path
// is a drop-in behind lmshoot::Objective, so a deployment keeps the reference's minimize(); this
// driver exists so that the library can run and time whole registrations by itself (bench.py's
// "ms per L-BFGS iteration") and is checked iterate-for-iterate against the reference's minimize in
// tests/test_lbfgs.py.  To make that comparison exact the floating-point expressions below keep the
// reference's association order (sequential dot products, (c1*a)*df0, ...).
//
// Algorithm (Nocedal & Wright, Numerical Optimization, Alg. 7.4/7.5 and 3.5/3.6):
//   direction   two-loop recursion over the last m curvature pairs, H0 = gamma*I with
//               gamma = s.y / y.y of the newest pair; non-descent directions reset to -g
//   first step  min(1, 1/|g|_2) when no pair is stored, else 1
//   search      bracket by doubling, then zoom with a safeguarded quadratic step (middle 80 % of the
//               bracket, bisection otherwise); non-finite values count as overshoot
//   update      pairs with s.y <= 1e-10 |s||y| are dropped
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <vector>

#include "../../include/lmshoot_b200.h"

namespace {

using Vec = std::vector<double>;

double dot_seq(const double* a, const double* b, size_t n)
{
  double s = 0;
  for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

double max_abs(const double* v, size_t n)
{
  double m = 0;
  for (size_t i = 0; i < n; ++i) m = std::max(m, std::abs(v[i]));
  return m;
}

bool every_finite(const double* v, size_t n)
{
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

struct SearchOutcome {
  double step = 0;  // 0: not even a sufficient-decrease point was seen
  double loss = 0;
  Vec grad;
  bool wolfe = false;  // both strong-Wolfe conditions hold at `step`
  int evals = 0;
};

// Strong-Wolfe search along d from x, given f(x) = f0 and slope g.d = slope0 < 0.
class WolfeSearch {
 public:
  WolfeSearch(lms_objective_fn fn, void* user, const Vec& x, const Vec& d, double f0, double slope0, double c1,
              double c2, int budget)
      : fn_(fn), user_(user), x_(x), d_(d), f0_(f0), slope0_(slope0), c1_(c1), c2_(c2), budget_(budget),
        trial_x_(x.size()), trial_g_(x.size())
  {
  }

  SearchOutcome run(double first_step)
  {
    double prev_a = 0, prev_f = f0_, prev_slope = slope0_;
    double a = first_step;
    for (bool first = true; evals_ < budget_; first = false) {
      const double f = value_at(a);
      const double slope = every_finite(trial_g_.data(), trial_g_.size())
                               ? dot_seq(trial_g_.data(), d_.data(), d_.size())
                               : 0.0;
      if (!std::isfinite(f) || f > f0_ + c1_ * a * slope0_ || (!first && f >= prev_f))
        return zoom(prev_a, prev_f, prev_slope, a, f);
      if (std::abs(slope) <= -c2_ * slope0_) return accepted(a, f);
      if (slope >= 0) return zoom(a, f, slope, prev_a, prev_f);
      prev_a = a;
      prev_f = f;
      prev_slope = slope;
      a *= 2;
    }
    return gave_up();
  }

 private:
  // f(x + a d); leaves the gradient in trial_g_ and remembers the best sufficient-decrease point.
  double value_at(double a)
  {
    for (size_t i = 0; i < x_.size(); ++i) trial_x_[i] = x_[i] + a * d_[i];
    ++evals_;
    const double f = fn_(user_, trial_x_.data(), trial_g_.data(), trial_x_.size());
    if (std::isfinite(f) && f <= f0_ + c1_ * a * slope0_ && (best_a_ == 0 || f < best_f_)) {
      best_a_ = a;
      best_f_ = f;
      best_g_ = trial_g_;
    }
    return f;
  }

  // [lo, hi] by role: lo carries the lowest sufficient-decrease value seen so far.
  SearchOutcome zoom(double lo, double f_lo, double slope_lo, double hi, double f_hi)
  {
    while (evals_ < budget_) {
      const double width = hi - lo;
      const double curvature = f_hi - f_lo - slope_lo * width;
      double a = lo + 0.5 * width;  // bisection unless the quadratic minimiser is well inside
      if (curvature != 0 && std::isfinite(curvature) && std::isfinite(f_hi)) {
        const double quad = lo - 0.5 * slope_lo * width * width / curvature;
        const double frac = (quad - lo) / width;
        if (frac > 0.1 && frac < 0.9) a = quad;
      }
      const double f = value_at(a);
      const double slope = dot_seq(trial_g_.data(), d_.data(), d_.size());
      if (!std::isfinite(f) || f > f0_ + c1_ * a * slope0_ || f >= f_lo) {
        hi = a;
        f_hi = f;
      } else {
        if (std::abs(slope) <= -c2_ * slope0_) return accepted(a, f);
        if (slope * (hi - lo) >= 0) {
          hi = lo;
          f_hi = f_lo;
        }
        lo = a;
        f_lo = f;
        slope_lo = slope;
      }
      if (std::abs(hi - lo) < 1e-16 * std::max(1.0, std::abs(lo))) break;
    }
    return gave_up();
  }

  SearchOutcome accepted(double a, double f)
  {
    SearchOutcome r;
    r.step = a;
    r.loss = f;
    r.grad = trial_g_;
    r.wolfe = true;
    r.evals = evals_;
    return r;
  }

  SearchOutcome gave_up()
  {
    SearchOutcome r;
    r.step = best_a_;
    r.loss = best_f_;
    r.grad = std::move(best_g_);
    r.wolfe = false;
    r.evals = evals_;
    return r;
  }

  lms_objective_fn fn_;
  void* user_;
  const Vec& x_;
  const Vec& d_;
  double f0_, slope0_, c1_, c2_;
  int budget_;
  int evals_ = 0;
  Vec trial_x_, trial_g_;
  double best_a_ = 0, best_f_ = 0;
  Vec best_g_;
};

// Fixed-capacity history of curvature pairs, oldest first.
class PairHistory {
 public:
  explicit PairHistory(int capacity) : cap_(capacity) {}
  size_t size() const { return s_.size(); }
  void clear()
  {
    s_.clear();
    y_.clear();
    rho_.clear();
  }
  void push(Vec s, Vec y, double rho)
  {
    s_.push_back(std::move(s));
    y_.push_back(std::move(y));
    rho_.push_back(rho);
    if ((int)s_.size() > cap_) {
      s_.erase(s_.begin());
      y_.erase(y_.begin());
      rho_.erase(rho_.begin());
    }
  }
  const Vec& s(size_t k) const { return s_[k]; }
  const Vec& y(size_t k) const { return y_[k]; }
  double rho(size_t k) const { return rho_[k]; }

 private:
  int cap_;
  std::vector<Vec> s_, y_;
  Vec rho_;
};

// d = -H g by the two-loop recursion (newest pair first, then oldest first).
void two_loop(const PairHistory& hist, double gamma, const Vec& g, Vec& d, Vec& coef)
{
  const size_t n = g.size();
  d = g;
  coef.assign(hist.size(), 0.0);
  for (size_t k = hist.size(); k-- > 0;) {
    const double a = hist.rho(k) * dot_seq(hist.s(k).data(), d.data(), n);
    coef[k] = a;
    const Vec& y = hist.y(k);
    for (size_t i = 0; i < n; ++i) d[i] -= a * y[i];
  }
  for (size_t i = 0; i < n; ++i) d[i] *= gamma;
  for (size_t k = 0; k < hist.size(); ++k) {
    const double b = hist.rho(k) * dot_seq(hist.y(k).data(), d.data(), n);
    const Vec& s = hist.s(k);
    for (size_t i = 0; i < n; ++i) d[i] += (coef[k] - b) * s[i];
  }
  for (size_t i = 0; i < n; ++i) d[i] = -d[i];
}

bool params_valid(const lms_lbfgs_params& p)
{
  // LbfgsParams::validate, lbfgs.hpp:19-26
  return p.memory >= 1 && p.max_iter >= 1 && 0 < p.c1 && p.c1 < p.c2 && p.c2 < 1 && p.max_line_search >= 1;
}

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
  if (!params_valid(*params)) return LMS_ERR_INVALID;

  Vec x(x0, x0 + n), g(n);
  double loss = fn(user, x.data(), g.data(), n);
  result->evaluations = 1;
  result->iterations = 0;
  result->reason = 1;
  if (!std::isfinite(loss) || !every_finite(g.data(), n)) return LMS_ERR_NUMERICAL;  // lbfgs.cpp:197-198
  result->initial_loss = loss;
  result->initial_grad_inf_norm = max_abs(g.data(), n);

  auto finish = [&](int reason) {
    result->reason = reason;
    result->loss = loss;
    if (n) {
      std::memcpy(x_out, x.data(), n * sizeof(double));
      std::memcpy(grad_out, g.data(), n * sizeof(double));
    }
    return LMS_OK;
  };
  if (result->initial_grad_inf_norm < params->grad_tol) return finish(0);

  PairHistory hist(params->memory);
  double gamma = 1.0;
  Vec d(n), coef;
  for (int iter = 0; iter < params->max_iter; ++iter) {
    two_loop(hist, gamma, g, d, coef);
    double slope = dot_seq(g.data(), d.data(), n);
    if (!(slope < 0)) {  // stale curvature information: restart from steepest descent
      hist.clear();
      gamma = 1.0;
      for (size_t i = 0; i < n; ++i) d[i] = -g[i];
      slope = -dot_seq(g.data(), g.data(), n);
    }
    const double first_step =
        hist.size() == 0 ? std::min(1.0, 1.0 / std::sqrt(dot_seq(g.data(), g.data(), n))) : 1.0;
    WolfeSearch search(fn, user, x, d, loss, slope, params->c1, params->c2, params->max_line_search);
    SearchOutcome ls = search.run(first_step);
    result->evaluations += ls.evals;

    if (ls.step > 0) {
      Vec s(n), y(n);
      for (size_t i = 0; i < n; ++i) {
        s[i] = ls.step * d[i];
        y[i] = ls.grad[i] - g[i];
        x[i] += s[i];
      }
      loss = ls.loss;
      g = std::move(ls.grad);
      const int k = result->iterations++;
      if (hist_loss) hist_loss[k] = loss;
      if (hist_grad_inf_norm) hist_grad_inf_norm[k] = max_abs(g.data(), n);
      if (hist_step) hist_step[k] = ls.step;
      if (hist_evals) hist_evals[k] = ls.evals;

      const double sy = dot_seq(s.data(), y.data(), n);
      const double s_norm = std::sqrt(dot_seq(s.data(), s.data(), n));
      const double y_norm = std::sqrt(dot_seq(y.data(), y.data(), n));
      if (sy > 1e-10 * s_norm * y_norm) {
        gamma = sy / dot_seq(y.data(), y.data(), n);
        hist.push(std::move(s), std::move(y), 1.0 / sy);
      }
    }
    if (!ls.wolfe) return finish(2);
    if (max_abs(g.data(), n) < params->grad_tol) return finish(0);
  }
  return finish(1);
}

}  // extern "C"
