// Header-only C++ adapter: wraps an lms_system handle (include/lmshoot_b200.h) into the reference's
// own objective type, `lmshoot::Objective` (lbfgs.hpp:48-50), so the unchanged host-side
// `lmshoot::minimize` (lbfgs.cpp:186-282) drives the CUDA hot path.  It replaces exactly the closure
// at registration.cpp:58-74 and rethrows the reference's exception types (errors.hpp) from the C-ABI
// status codes.  Compile with the reference's include directory on the include path.
//
//   lmshoot_b200::DeviceObjective dev(cfg.sigma, n, D, cfg.precision == Precision::f32, cfg.timesteps);
//   dev.bind(q0_flat, target_flat, cfg.lambda, cfg.timesteps);      // registration.cpp:43-45 captures
//   MinimizeResult opt = minimize(dev.objective(), std::move(x0), lp);   // registration.cpp:79, unchanged
//   dev.final_q(warped_flat);                                       // replaces registration.cpp:85-93
#pragma once

#include <cstddef>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "lmshoot/errors.hpp"
#include "lmshoot/lbfgs.hpp"
#include "lmshoot_b200.h"

namespace lmshoot_b200 {

// C-ABI status -> the reference's exception taxonomy (errors.hpp:10-77).
inline void throw_status(int status, const lms_system* sys)
{
  if (status == LMS_OK) return;
  const std::string detail = sys ? lms_last_error_message(sys) : "";
  const std::string text = std::string(lms_status_string(status)) + (detail.empty() ? "" : ": " + detail);
  switch (status) {
    case LMS_ERR_SHAPE: throw lmshoot::ShapeError(text);
    case LMS_ERR_DIVERGED:
      throw lmshoot::DivergedError(lms_last_diverged_step(sys), static_cast<std::ptrdiff_t>(lms_last_diverged_point(sys)));
    case LMS_ERR_INVALID: throw std::invalid_argument(text);
    case LMS_ERR_NUMERICAL: throw lmshoot::NumericalError(text);
    default: throw std::runtime_error(text);
  }
}

class DeviceObjective {
 public:
  DeviceObjective(double sigma, std::size_t n, int dim, bool f32, int max_timesteps, int device = 0)
      : n_(n), dim_(dim)
  {
    lms_config cfg{};
    cfg.precision = f32 ? LMS_PRECISION_F32 : LMS_PRECISION_F64;
    cfg.dim = dim;
    cfg.n = n;
    cfg.sigma = sigma;
    cfg.max_timesteps = max_timesteps;
    cfg.device = device;
    throw_status(lms_system_create(&cfg, &sys_), nullptr);
  }
  ~DeviceObjective() { lms_system_destroy(sys_); }
  DeviceObjective(const DeviceObjective&) = delete;
  DeviceObjective& operator=(const DeviceObjective&) = delete;

  // What the closure captures (registration.cpp:43-45): uploaded once, device-resident afterwards.
  void bind(std::span<const double> q0, std::span<const double> target, double lambda, int timesteps)
  {
    if (q0.size() != n_ * dim_ || target.size() != n_ * dim_)
      throw lmshoot::ShapeError("template and target must have equal count and dimension");
    throw_status(lms_bind_registration(sys_, q0.data(), target.data(), lambda, timesteps), sys_);
  }

  // The drop-in for the lambda at registration.cpp:58-74.  kinetic / mismatch of the last call stay
  // available for the verbose line (:70-72).
  lmshoot::Objective objective()
  {
    return [this](std::span<const double> x, std::span<double> grad) -> double {
      if (x.size() != n_ * dim_ || grad.size() != n_ * dim_) throw lmshoot::ShapeError("objective: bad vector length");
      double loss = 0;
      throw_status(lms_objective_eval(sys_, x.data(), grad.data(), &loss, &kinetic_, &mismatch_), sys_);
      ++evaluations_;
      return loss;
    };
  }

  void final_q(std::span<double> out) const { throw_status(lms_objective_final_q(sys_, out.data()), sys_); }
  // {avg_before, max_before, avg_after, max_after}: average_dist / max_dist of (template, target) and of
  // (q(1) of the last evaluation, target) -- registration.cpp:39-40,95-96 -- computed on the device
  struct Metrics { double avg_before, max_before, avg_after, max_after; };
  Metrics metrics() const
  {
    double m[4];
    throw_status(lms_registration_metrics(sys_, m), sys_);
    return {m[0], m[1], m[2], m[3]};
  }
  double last_kinetic() const { return kinetic_; }
  double last_mismatch() const { return mismatch_; }
  long evaluations() const { return evaluations_; }
  lms_system* handle() const { return sys_; }

 private:
  lms_system* sys_ = nullptr;
  std::size_t n_;
  int dim_;
  double kinetic_ = 0, mismatch_ = 0;
  long evaluations_ = 0;
};

}  // namespace lmshoot_b200
