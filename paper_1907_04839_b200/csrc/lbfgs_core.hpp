// L-BFGS with a strong-Wolfe line search, written once against a small vector-operations policy so that the
// same decision logic runs with host vectors (lbfgs_driver.cpp: sequential sums, iterate-for-iterate equal to
// the reference's minimize, lbfgs.cpp:186-282) and with device-resident vectors (device_lbfgs.cu: only scalars
// cross the bus).
//
// Algorithm (Nocedal & Wright, Numerical Optimization, Alg. 7.4/7.5 and 3.5/3.6), with the reference's choices:
//   direction   two-loop recursion over the last m curvature pairs, H0 = gamma*I with gamma = s.y / y.y of the
//               newest pair; a non-descent direction resets the history to steepest descent
//   first step  min(1, 1/|g|_2) when no pair is stored, else 1
//   search      bracket by doubling, then zoom with a safeguarded quadratic step (middle 80 % of the bracket,
//               bisection otherwise); non-finite values count as overshoot; at most max_line_search evaluations
//   update      pairs with s.y <= 1e-10 |s||y| are dropped
//
// Ops concept:
//   using Vec = ...;                       handle of a length-n vector
//   Vec make(); void release(Vec);
//   void copy(Vec dst, Vec src);
//   double dot(Vec a, Vec b); double max_abs(Vec v); bool all_finite(Vec v);
//   void axpy_to(Vec out, Vec x, double a, Vec d);        out = x + a*d
//   void sub_scaled(Vec d, double a, Vec y);              d -= a*y
//   void add_scaled(Vec d, double c, Vec s);              d += c*s
//   void scale(Vec d, double g); void negate(Vec d); void neg_copy(Vec d, Vec g);   d *= g; d = -d; d = -g
//   void take_step(Vec s, Vec y, Vec x, double step, Vec d, Vec g_new, Vec g);      s = step*d; y = g_new-g; x += s
//   double dot_if_finite(Vec a, Vec b);    a.b, or 0 when a has a non-finite entry
//   double two_loop(pairs s, y, rho, gamma, g, d, coef);   d = -H g, returns g.d
//   void pair_stats(Vec s, Vec y, double* sy, double* ss, double* yy);
//   double objective(Vec x, Vec grad);     may throw to abort the run
// (two_loop_generic below is the reference sequence of dots and updates; the host policy uses it as is.)
#pragma once

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/lmshoot_b200.h"

namespace lms {

template <class Ops>
struct SearchOutcome {
  double step = 0;  // 0: not even a sufficient-decrease point was seen
  double loss = 0;
  bool wolfe = false;  // both strong-Wolfe conditions hold at `step`
  bool have_grad = false;
  int evals = 0;
};

// Strong-Wolfe search along d from x, given f(x) = f0 and slope g.d = slope0 < 0.  The gradient at the returned
// step is left in `out_g`.
template <class Ops>
class WolfeSearch {
 public:
  using Vec = typename Ops::Vec;
  WolfeSearch(Ops& ops, Vec x, Vec d, double f0, double slope0, double c1, double c2, int budget, Vec trial_x,
              Vec trial_g, Vec best_g)
      : ops_(ops), x_(x), d_(d), f0_(f0), slope0_(slope0), c1_(c1), c2_(c2), budget_(budget), trial_x_(trial_x),
        trial_g_(trial_g), best_g_(best_g)
  {
  }

  // On return the gradient to use is trial_g (wolfe == true) or best_g (wolfe == false, step > 0).
  SearchOutcome<Ops> run(double first_step)
  {
    double prev_a = 0, prev_f = f0_, prev_slope = slope0_;
    double a = first_step;
    for (bool first = true; evals_ < budget_; first = false) {
      const double f = value_at(a);
      const double slope = ops_.dot_if_finite(trial_g_, d_);  // g.d, or 0 when the gradient is not finite
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
    ops_.axpy_to(trial_x_, x_, a, d_);
    ++evals_;
    const double f = ops_.objective(trial_x_, trial_g_);
    if (std::isfinite(f) && f <= f0_ + c1_ * a * slope0_ && (best_a_ == 0 || f < best_f_)) {
      best_a_ = a;
      best_f_ = f;
      ops_.copy(best_g_, trial_g_);
    }
    return f;
  }

  // [lo, hi] by role: lo carries the lowest sufficient-decrease value seen so far.
  SearchOutcome<Ops> zoom(double lo, double f_lo, double slope_lo, double hi, double f_hi)
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
      const double slope = ops_.dot(trial_g_, d_);
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

  SearchOutcome<Ops> accepted(double a, double f)
  {
    SearchOutcome<Ops> r;
    r.step = a;
    r.loss = f;
    r.wolfe = true;
    r.have_grad = true;
    r.evals = evals_;
    return r;
  }

  SearchOutcome<Ops> gave_up()
  {
    SearchOutcome<Ops> r;
    r.step = best_a_;
    r.loss = best_f_;
    r.wolfe = false;
    r.have_grad = best_a_ != 0;
    r.evals = evals_;
    return r;
  }

  Ops& ops_;
  Vec x_, d_;
  double f0_, slope0_, c1_, c2_;
  int budget_;
  int evals_ = 0;
  Vec trial_x_, trial_g_, best_g_;
  double best_a_ = 0, best_f_ = 0;
};

// d = -H g with H built from the stored pairs (newest pair first, then oldest first); returns g.d.
template <class Ops>
double two_loop_generic(Ops& ops, const std::vector<typename Ops::Vec>& hist_s,
                        const std::vector<typename Ops::Vec>& hist_y, const std::vector<double>& hist_rho, double gamma,
                        typename Ops::Vec g, typename Ops::Vec d, std::vector<double>& coef)
{
  ops.copy(d, g);
  coef.assign(hist_s.size(), 0.0);
  for (size_t k = hist_s.size(); k-- > 0;) {
    const double a = hist_rho[k] * ops.dot(hist_s[k], d);
    coef[k] = a;
    ops.sub_scaled(d, a, hist_y[k]);
  }
  ops.scale(d, gamma);
  for (size_t k = 0; k < hist_s.size(); ++k) {
    const double b = hist_rho[k] * ops.dot(hist_y[k], d);
    ops.add_scaled(d, coef[k] - b, hist_s[k]);
  }
  ops.negate(d);
  return ops.dot(g, d);
}

inline bool lbfgs_params_valid(const lms_lbfgs_params& p)
{
  // LbfgsParams::validate, lbfgs.hpp:19-26
  return p.memory >= 1 && p.max_iter >= 1 && 0 < p.c1 && p.c1 < p.c2 && p.c2 < 1 && p.max_line_search >= 1;
}

// minimize (lbfgs.hpp:81-82).  x holds x0 on entry and the minimiser on return; g receives the final gradient.
// Returns an LMS_* status; the objective may throw to abort (the caller catches).
template <class Ops>
int minimize_core(Ops& ops, typename Ops::Vec x, typename Ops::Vec g, const lms_lbfgs_params& params,
                  lms_minimize_result* result, double* hist_loss, double* hist_grad_inf_norm, double* hist_step,
                  int* hist_evals)
{
  using Vec = typename Ops::Vec;
  double loss = ops.objective(x, g);
  result->evaluations = 1;
  result->iterations = 0;
  result->reason = 1;
  if (!std::isfinite(loss) || !ops.all_finite(g)) return LMS_ERR_NUMERICAL;  // lbfgs.cpp:197-198
  result->initial_loss = loss;
  result->initial_grad_inf_norm = ops.max_abs(g);
  result->loss = loss;
  if (result->initial_grad_inf_norm < params.grad_tol) {
    result->reason = 0;
    return LMS_OK;
  }

  // curvature pairs, oldest first
  std::vector<Vec> hist_s, hist_y;
  std::vector<double> hist_rho, coef;
  double gamma = 1.0;
  Vec d = ops.make(), trial_x = ops.make(), trial_g = ops.make(), best_g = ops.make();
  auto cleanup = [&] {
    for (Vec v : hist_s) ops.release(v);
    for (Vec v : hist_y) ops.release(v);
    ops.release(d);
    ops.release(trial_x);
    ops.release(trial_g);
    ops.release(best_g);
  };
  int status = LMS_OK;
  try {
    for (int iter = 0; iter < params.max_iter; ++iter) {
      // d = -H g by the two-loop recursion (newest pair first, then oldest first); slope = g.d
      double slope = ops.two_loop(hist_s, hist_y, hist_rho, gamma, g, d, coef);
      if (!(slope < 0)) {  // stale curvature information: restart from steepest descent
        for (Vec v : hist_s) ops.release(v);
        for (Vec v : hist_y) ops.release(v);
        hist_s.clear();
        hist_y.clear();
        hist_rho.clear();
        gamma = 1.0;
        ops.neg_copy(d, g);
        slope = -ops.dot(g, g);
      }
      const double first_step = hist_s.empty() ? std::min(1.0, 1.0 / std::sqrt(ops.dot(g, g))) : 1.0;
      WolfeSearch<Ops> search(ops, x, d, loss, slope, params.c1, params.c2, params.max_line_search, trial_x, trial_g,
                              best_g);
      SearchOutcome<Ops> ls = search.run(first_step);
      result->evaluations += ls.evals;

      if (ls.step > 0) {
        Vec g_new = ls.wolfe ? trial_g : best_g;
        // s and y belong to nobody until they enter the history: a throwing vector operation in between
        // (device policy: a failed launch) must hand them back
        Vec s = ops.make(), y = ops.make();
        bool kept = false;
        try {
          ops.take_step(s, y, x, ls.step, d, g_new, g);
          loss = ls.loss;
          ops.copy(g, g_new);
          const int k = result->iterations++;
          if (k < params.max_iter) {  // capacity of the hist_* arrays (one record per accepted iterate)
            if (hist_loss) hist_loss[k] = loss;
            if (hist_grad_inf_norm) hist_grad_inf_norm[k] = ops.max_abs(g);
            if (hist_step) hist_step[k] = ls.step;
            if (hist_evals) hist_evals[k] = ls.evals;
          }

          double sy, ss, yy;
          ops.pair_stats(s, y, &sy, &ss, &yy);  // s.y, s.s, y.y
          const double s_norm = std::sqrt(ss);
          const double y_norm = std::sqrt(yy);
          if (sy > 1e-10 * s_norm * y_norm) {
            gamma = sy / yy;
            hist_s.push_back(s);
            kept = true;  // from here on cleanup() releases them through the history
            hist_y.push_back(y);
            hist_rho.push_back(1.0 / sy);
            if ((int)hist_s.size() > params.memory) {
              ops.release(hist_s.front());
              ops.release(hist_y.front());
              hist_s.erase(hist_s.begin());
              hist_y.erase(hist_y.begin());
              hist_rho.erase(hist_rho.begin());
            }
          }
        } catch (...) {
          if (!kept) {
            ops.release(s);
            ops.release(y);
          } else if (hist_y.size() < hist_s.size()) {
            ops.release(y);  // s made it into the history, y did not
          }
          throw;
        }
        if (!kept) {
          ops.release(s);
          ops.release(y);
        }
      }
      result->loss = loss;
      if (!ls.wolfe) {
        result->reason = 2;
        break;
      }
      if (ops.max_abs(g) < params.grad_tol) {
        result->reason = 0;
        break;
      }
    }
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  return status;
}

}  // namespace lms
