// TEST INFRASTRUCTURE ONLY (oracle/): the reference's UNMODIFIED minimize (lbfgs.cpp, compiled where it
// lies) driving the CUDA objective through include/lmshoot_b200/objective.hpp -- the integration a
// maintainer would make at registration.cpp:58-79.  Built by oracle/Makefile into
// oracle/_ref/libref_cuda_driver.so and linked against the product's C-ABI library.
#include "ref_shim.hpp"

#include <cstring>
#include <vector>

#include "lmshoot_b200/objective.hpp"

extern "C" {

struct RefCudaOut {
  double loss, initial_loss;
  int evaluations, iterations, reason, status, diverged_step;
};

// Restates registration.cpp:43-93 around the adapter: x0 = (target - q0)/T, minimize, warped = q(1).
int ref_cuda_register(int f32, int dim, std::size_t n, double sigma, double lambda, int timesteps, int max_iter,
                      double grad_tol, const double* q0, const double* target, double* momenta, double* warped,
                      RefCudaOut* out, double* hist_loss)
{
  out->status = 0;
  out->diverged_step = -1;
  try {
    lmshoot_b200::DeviceObjective dev(sigma, n, dim, f32 != 0, timesteps);
    dev.bind({q0, n * dim}, {target, n * dim}, lambda, timesteps);
    std::vector<double> x0(n * dim);
    for (std::size_t e = 0; e < n * dim; ++e) x0[e] = (target[e] - q0[e]) / timesteps;
    lmshoot::LbfgsParams lp;
    lp.max_iter = max_iter;
    lp.grad_tol = grad_tol;
    lmshoot::MinimizeResult opt = lmshoot::minimize(dev.objective(), std::move(x0), lp);
    std::memcpy(momenta, opt.x.data(), n * dim * sizeof(double));
    std::vector<double> g(n * dim);
    dev.objective()(opt.x, g);  // final re-integration under p0* (registration.cpp:85-93)
    dev.final_q({warped, n * dim});
    out->loss = opt.loss;
    out->initial_loss = opt.history.initial_loss;
    out->evaluations = opt.history.evaluations;
    out->iterations = static_cast<int>(opt.history.iterations.size());
    out->reason = static_cast<int>(opt.history.reason);
    if (hist_loss)
      for (std::size_t k = 0; k < opt.history.iterations.size(); ++k) hist_loss[k] = opt.history.iterations[k].loss;
  } catch (const lmshoot::DivergedError& e) {
    out->status = 2;
    out->diverged_step = e.timestep();
  } catch (const lmshoot::ShapeError&) {
    out->status = 1;
  } catch (const lmshoot::NumericalError&) {
    out->status = 4;
  } catch (const std::invalid_argument&) {
    out->status = 3;
  } catch (...) {
    out->status = 5;
  }
  return out->status;
}

}  // extern "C"
