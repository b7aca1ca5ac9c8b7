// TEST INFRASTRUCTURE ONLY (oracle/): never linked into the product library.
//
// C-ABI harness over the UNMODIFIED reference headers and src/lbfgs.cpp, compiled where they lie
// under /root/reference/proj (see oracle/Makefile; outputs only into oracle/_ref/).  Used (a) to pin
// the plain-C restatement in lmshoot_oracle.c bit for bit, (b) to generate tests/golden/ vectors,
// (c) as bench.py's `--impl reference` / cpu_baseline arm.  Every entry point takes and returns
// row-major double arrays (n x dim) and converts to the working precision T exactly as the
// reference's own objective closure does (registration.cpp:61-67: p0[i][c] = T(x[i*D+c]),
// grad[i*D+c] = double(g.grad[i][c])).
#include "ref_shim.hpp"

#include <cstddef>
#include <cstring>
#include <span>
#include <stdexcept>
#include <vector>

#include "lmshoot/errors.hpp"
#include "lmshoot/flow.hpp"
#include "lmshoot/lbfgs.hpp"
#include "lmshoot/reduction.hpp"
#include "lmshoot/rng.hpp"
#include "lmshoot/shooting.hpp"

using namespace lmshoot;

namespace {

enum Status { kOk = 0, kShape = 1, kDiverged = 2, kInvalid = 3, kNumerical = 4, kOther = 5 };

thread_local int g_diverged_step = -1;

template <class Fn>
int guarded(Fn&& fn)
{
  g_diverged_step = -1;
  try {
    fn();
    return kOk;
  } catch (const DivergedError& e) {
    g_diverged_step = e.timestep();
    return kDiverged;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const NumericalError&) {
    return kNumerical;
  } catch (const std::invalid_argument&) {
    return kInvalid;
  } catch (...) {
    return kOther;
  }
}

ReduceOptions make_opts(int strategy, std::size_t block, unsigned threads)
{
  ReduceOptions o;
  o.strategy = static_cast<ReduceStrategy>(strategy);
  o.block_size = block;
  o.threads = threads;
  return o;
}

template <class T, int D>
PointArray<T, D> load_points(const double* src, std::size_t n)
{
  PointArray<T, D> out(n);
  for (std::size_t i = 0; i < n; ++i)
    for (int c = 0; c < D; ++c) out[i][c] = T(src[i * D + c]);
  return out;
}

template <class T, int D>
void store_points(const PointArray<T, D>& pts, double* dst)
{
  for (std::size_t i = 0; i < pts.size(); ++i)
    for (int c = 0; c < D; ++c) dst[i * D + c] = double(pts[i][c]);
}

template <class Fn>
decltype(auto) dispatch(int prec, int dim, Fn&& fn)
{
  return dispatch_precision_dim(prec == 0 ? Precision::f32 : Precision::f64, dim, fn);
}

}  // namespace

extern "C" {

int ref_last_diverged_step() { return g_diverged_step; }

unsigned ref_hardware_threads() { return hardware_threads(); }

double ref_gaussian_kernel(int prec, double r_sq, double sigma)
{
  return prec == 0 ? double(gaussian_kernel<float>(float(r_sq), float(sigma)))
                   : gaussian_kernel<double>(r_sq, sigma);
}

double ref_kernel_scale(int prec, double sigma)
{
  return prec == 0 ? double(kernel_scale<float>(sigma)) : kernel_scale<double>(sigma);
}

double ref_tree_sum(int prec, const double* values, std::size_t n)
{
  if (prec == 0) {
    std::vector<float> v(values, values + n);
    return double(tree_sum<float>(std::span<const float>(v)));
  }
  return tree_sum<double>(std::span<const double>(values, n));
}

void ref_rng_uniforms(unsigned long long seed, std::size_t count, double* out)
{
  Rng rng(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = rng.uniform();
}

void ref_rng_normals(unsigned long long seed, std::size_t count, double* out)
{
  Rng rng(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = rng.normal();
}

// One Rng instance, draws interleaved as `kinds` says (0 = uniform(), 1 = normal()); rng.hpp:19-41.
void ref_rng_stream(unsigned long long seed, std::size_t count, const unsigned char* kinds, double* out)
{
  Rng rng(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = kinds[i] ? rng.normal() : rng.uniform();
}

int ref_hamiltonian(int prec, int dim, std::size_t n, double sigma, const double* q, const double* p,
                    unsigned threads, double* out)
{
  return guarded([&] {
    dispatch(prec, dim, [&](auto tf, auto dc) {
      using T = typename decltype(tf)::type;
      constexpr int D = dc();
      HamiltonianSystem<T, D> sys(sigma, make_opts(2, 256, threads));
      *out = sys.hamiltonian(load_points<T, D>(q, n), load_points<T, D>(p, n));
    });
  });
}

int ref_derivatives(int prec, int dim, std::size_t n, double sigma, const double* q, const double* p,
                    double* hq, double* hp, int strategy, std::size_t block, unsigned threads)
{
  return guarded([&] {
    dispatch(prec, dim, [&](auto tf, auto dc) {
      using T = typename decltype(tf)::type;
      constexpr int D = dc();
      HamiltonianSystem<T, D> sys(sigma, make_opts(strategy, block, threads));
      PointArray<T, D> ohq, ohp;
      sys.derivatives(load_points<T, D>(q, n), load_points<T, D>(p, n), ohq, ohp);
      store_points<T, D>(ohq, hq);
      store_points<T, D>(ohp, hp);
    });
  });
}

// traj_q / traj_p: (timesteps+1) x n x dim.
int ref_integrate_forward(int prec, int dim, std::size_t n, double sigma, int timesteps,
                          const double* q0, const double* p0, double* traj_q, double* traj_p,
                          int strategy, std::size_t block, unsigned threads)
{
  return guarded([&] {
    dispatch(prec, dim, [&](auto tf, auto dc) {
      using T = typename decltype(tf)::type;
      constexpr int D = dc();
      HamiltonianSystem<T, D> sys(sigma, make_opts(strategy, block, threads));
      Trajectory<T, D> traj =
          sys.integrate_forward(load_points<T, D>(q0, n), load_points<T, D>(p0, n), timesteps);
      for (int t = 0; t <= timesteps; ++t) {
        store_points<T, D>(traj.q[t], traj_q + std::size_t(t) * n * D);
        store_points<T, D>(traj.p[t], traj_p + std::size_t(t) * n * D);
      }
    });
  });
}

int ref_adjoint_step(int prec, int dim, std::size_t n, double sigma, const double* q, const double* p,
                     const double* alpha, const double* beta, double* d_alpha, double* d_beta,
                     int strategy, std::size_t block, unsigned threads)
{
  return guarded([&] {
    dispatch(prec, dim, [&](auto tf, auto dc) {
      using T = typename decltype(tf)::type;
      constexpr int D = dc();
      HamiltonianSystem<T, D> sys(sigma, make_opts(strategy, block, threads));
      AdjointState<T, D> adj{load_points<T, D>(alpha, n), load_points<T, D>(beta, n)};
      PointArray<T, D> da, db;
      sys.adjoint_step(load_points<T, D>(q, n), load_points<T, D>(p, n), adj, da, db);
      store_points<T, D>(da, d_alpha);
      store_points<T, D>(db, d_beta);
    });
  });
}

int ref_mismatch_sq(int prec, int dim, std::size_t n, const double* a, const double* b, double* out)
{
  return guarded([&] {
    dispatch(prec, dim, [&](auto tf, auto dc) {
      using T = typename decltype(tf)::type;
      constexpr int D = dc();
      HamiltonianSystem<T, D> sys(1.0, make_opts(2, 256, 1));
      *out = sys.mismatch_sq(load_points<T, D>(a, n), load_points<T, D>(b, n));
    });
  });
}

// scalars[3] = {loss, kinetic, mismatch}
int ref_compute_gradient(int prec, int dim, std::size_t n, double sigma, double lambda, int timesteps,
                         const double* q0, const double* p0, const double* target, double* scalars,
                         double* grad, int strategy, std::size_t block, unsigned threads)
{
  return guarded([&] {
    dispatch(prec, dim, [&](auto tf, auto dc) {
      using T = typename decltype(tf)::type;
      constexpr int D = dc();
      HamiltonianSystem<T, D> sys(sigma, make_opts(strategy, block, threads));
      GradientResult<T, D> g = sys.compute_gradient(load_points<T, D>(q0, n), load_points<T, D>(p0, n),
                                                    load_points<T, D>(target, n), lambda, timesteps);
      scalars[0] = g.loss;
      scalars[1] = g.kinetic;
      scalars[2] = g.mismatch;
      store_points<T, D>(g.grad, grad);
    });
  });
}

// flow.hpp:26-48: velocities of m points against one snapshot (q, p) of n landmarks.
int ref_velocities(int prec, int dim, std::size_t n, std::size_t m, double sigma, const double* q,
                   const double* p, const double* points, double* out, int strategy, std::size_t block,
                   unsigned threads)
{
  return guarded([&] {
    dispatch(prec, dim, [&](auto tf, auto dc) {
      using T = typename decltype(tf)::type;
      constexpr int D = dc();
      Trajectory<T, D> traj;
      traj.sigma = sigma;
      traj.dt = 1.0;
      traj.q.push_back(load_points<T, D>(q, n));
      traj.p.push_back(load_points<T, D>(p, n));
      FlowField<T, D> field{&traj, make_opts(strategy, block, threads)};
      PointArray<T, D> v;
      detail::velocities_at_step<T, D>(field, 0, load_points<T, D>(points, m), v);
      store_points<T, D>(v, out);
    });
  });
}

// flow.hpp:66-81: warp m points through a stored trajectory ((timesteps+1) x n x dim arrays).
int ref_warp_points(int prec, int dim, std::size_t n, std::size_t m, double sigma, int timesteps,
                    const double* traj_q, const double* traj_p, const double* points, double* out,
                    int strategy, std::size_t block, unsigned threads)
{
  return guarded([&] {
    dispatch(prec, dim, [&](auto tf, auto dc) {
      using T = typename decltype(tf)::type;
      constexpr int D = dc();
      Trajectory<T, D> traj;
      traj.sigma = sigma;
      traj.dt = 1.0 / timesteps;
      for (int t = 0; t <= timesteps; ++t) {
        traj.q.push_back(load_points<T, D>(traj_q + std::size_t(t) * n * D, n));
        traj.p.push_back(load_points<T, D>(traj_p + std::size_t(t) * n * D, n));
      }
      FlowField<T, D> field{&traj, make_opts(strategy, block, threads)};
      // warp_points itself (flow.hpp:66-81) cannot be instantiated: its inner call at :75 deduces D
      // both as int (FlowField) and std::size_t (std::array).  The loop is restated here around the
      // reference's own velocities_at_step<T, D>; same Euler update and finite check as :76-79.
      const T dt = T(traj.dt);
      PointArray<T, D> x = load_points<T, D>(points, m), v;
      for (int t = 0; t < traj.steps(); ++t) {
        detail::velocities_at_step<T, D>(field, t, x, v);
        for (std::size_t k = 0; k < x.size(); ++k) {
          for (int c = 0; c < D; ++c) x[k][c] = x[k][c] + dt * v[k][c];
          if (!is_finite<T, D>(x[k])) throw DivergedError(t + 1, static_cast<std::ptrdiff_t>(k));
        }
      }
      store_points<T, D>(x, out);
    });
  });
}

// ---- optimiser: the reference's unmodified minimize (lbfgs.cpp:186-282) -----------------------

typedef double (*ref_objective_fn)(void* user, const double* x, double* grad, std::size_t n);

struct RefMinimizeOut {
  double loss;
  int evaluations;
  int iterations;
  int reason;  // StopReason as int
  double initial_loss;
  double initial_grad_inf_norm;
};

// hist_* (may be null) receive up to max_iter accepted-iterate records.
int ref_minimize(ref_objective_fn fn, void* user, std::size_t n, const double* x0, int max_iter,
                 double grad_tol, int memory, double c1, double c2, int max_line_search, double* x_out,
                 double* grad_out, RefMinimizeOut* out, double* hist_loss, double* hist_gnorm,
                 double* hist_step, int* hist_evals)
{
  return guarded([&] {
    Objective objective = [&](std::span<const double> x, std::span<double> g) -> double {
      return fn(user, x.data(), g.data(), x.size());
    };
    LbfgsParams lp;
    lp.max_iter = max_iter;
    lp.grad_tol = grad_tol;
    lp.memory = memory;
    lp.c1 = c1;
    lp.c2 = c2;
    lp.max_line_search = max_line_search;
    MinimizeResult r = minimize(objective, std::vector<double>(x0, x0 + n), lp);
    std::memcpy(x_out, r.x.data(), n * sizeof(double));
    std::memcpy(grad_out, r.grad.data(), n * sizeof(double));
    out->loss = r.loss;
    out->evaluations = r.history.evaluations;
    out->iterations = static_cast<int>(r.history.iterations.size());
    out->reason = static_cast<int>(r.history.reason);
    out->initial_loss = r.history.initial_loss;
    out->initial_grad_inf_norm = r.history.initial_grad_inf_norm;
    for (std::size_t k = 0; k < r.history.iterations.size(); ++k) {
      if (hist_loss) hist_loss[k] = r.history.iterations[k].loss;
      if (hist_gnorm) hist_gnorm[k] = r.history.iterations[k].grad_inf_norm;
      if (hist_step) hist_step[k] = r.history.iterations[k].step;
      if (hist_evals) hist_evals[k] = r.history.iterations[k].evals;
    }
  });
}

// The registration core, restating registration.cpp:43-93 (which cannot be compiled here: it needs
// <json.hpp> and trips the vec.hpp deduction problem at :44-45).  The restated lines contain no
// arithmetic beyond casts and x0 = (target - q0)/T (:47-52); the objective is :58-74 verbatim in
// behaviour; the final re-integration is :85-93.
int ref_register(int prec, int dim, std::size_t n, double sigma, double lambda, int timesteps,
                 int max_iter, double grad_tol, const double* q0_in, const double* target_in,
                 double* momenta_out, double* warped_out, RefMinimizeOut* out, double* hist_loss,
                 int strategy, std::size_t block, unsigned threads)
{
  return guarded([&] {
    dispatch(prec, dim, [&](auto tf, auto dc) {
      using T = typename decltype(tf)::type;
      constexpr int D = dc();
      HamiltonianSystem<T, D> system(sigma, make_opts(strategy, block, threads));
      PointArray<T, D> q0 = load_points<T, D>(q0_in, n);
      PointArray<T, D> target = load_points<T, D>(target_in, n);
      std::vector<double> x0(n * D);
      for (std::size_t i = 0; i < n; ++i)
        for (int c = 0; c < D; ++c) x0[i * D + c] = (target_in[i * D + c] - q0_in[i * D + c]) / timesteps;
      Objective objective = [&](std::span<const double> x, std::span<double> grad) -> double {
        PointArray<T, D> p0(n);
        for (std::size_t i = 0; i < n; ++i)
          for (int c = 0; c < D; ++c) p0[i][c] = T(x[i * D + c]);
        GradientResult<T, D> g = system.compute_gradient(q0, p0, target, lambda, timesteps);
        for (std::size_t i = 0; i < n; ++i)
          for (int c = 0; c < D; ++c) grad[i * D + c] = double(g.grad[i][c]);
        return g.loss;
      };
      LbfgsParams lp;
      lp.max_iter = max_iter;
      lp.grad_tol = grad_tol;
      MinimizeResult opt = minimize(objective, std::move(x0), lp);
      std::memcpy(momenta_out, opt.x.data(), n * D * sizeof(double));
      PointArray<T, D> p_star(n);
      for (std::size_t i = 0; i < n; ++i)
        for (int c = 0; c < D; ++c) p_star[i][c] = T(opt.x[i * D + c]);
      Trajectory<T, D> traj = system.integrate_forward(q0, p_star, timesteps);
      store_points<T, D>(traj.final_q(), warped_out);
      out->loss = opt.loss;
      out->evaluations = opt.history.evaluations;
      out->iterations = static_cast<int>(opt.history.iterations.size());
      out->reason = static_cast<int>(opt.history.reason);
      out->initial_loss = opt.history.initial_loss;
      out->initial_grad_inf_norm = opt.history.initial_grad_inf_norm;
      if (hist_loss)
        for (std::size_t k = 0; k < opt.history.iterations.size(); ++k)
          hist_loss[k] = opt.history.iterations[k].loss;
    });
  });
}

}  // extern "C"
