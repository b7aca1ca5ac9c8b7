"""Generates tests/golden/*.npz from the UNMODIFIED reference compiled in place
(oracle/_ref/liblmshoot_ref.so, built by oracle/Makefile from /root/reference/proj).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures carry their own inputs, so the GPU box needs neither /root/reference nor numpy's RNG.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import load_reference  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SIGMA = 1.5


def hotpath():
    ref = load_reference()
    rng = np.random.default_rng(20190704839 % (2**32))
    out = {}
    for prec in ("f32", "f64"):
        for dim in (2, 3):
            for n in (1, 2, 7, 33, 200):
                key = f"{prec}_d{dim}_n{n}_"
                q = rng.uniform(-4.0, 4.0, (n, dim))
                p = 0.75 * rng.normal(size=(n, dim))
                target = q + 0.5 * rng.normal(size=(n, dim))
                alpha = rng.normal(size=(n, dim))
                beta = rng.normal(size=(n, dim))
                pts = rng.uniform(-4.0, 4.0, (5, dim))
                T, lam = 4, 10.0
                out[key + "q"], out[key + "p"], out[key + "target"] = q, p, target
                out[key + "alpha"], out[key + "beta"], out[key + "pts"] = alpha, beta, pts
                hq, hp = ref.derivatives(prec, q, p, SIGMA)
                out[key + "hq"], out[key + "hp"] = hq, hp
                out[key + "H"] = np.array(ref.hamiltonian(prec, q, p, SIGMA))
                da, db = ref.adjoint_step(prec, q, p, alpha, beta, SIGMA)
                out[key + "dalpha"], out[key + "dbeta"] = da, db
                out[key + "mismatch"] = np.array(ref.mismatch_sq(prec, q, target))
                tq, tp = ref.integrate_forward(prec, q, p, SIGMA, T)
                out[key + "traj_q"], out[key + "traj_p"] = tq, tp
                loss, kin, mm, grad = ref.compute_gradient(prec, q, p, target, SIGMA, lam, T)
                out[key + "scalars"] = np.array([loss, kin, mm])
                out[key + "grad"] = grad
                out[key + "vel"] = ref.velocities(prec, q, p, pts, SIGMA)
                out[key + "warped"] = ref.warp_points(prec, tq, tp, pts, SIGMA)
    out["meta_sigma_T_lambda"] = np.array([SIGMA, 4, 10.0])
    np.savez_compressed(os.path.join(HERE, "hotpath_golden.npz"), **out)
    print("hotpath_golden.npz:", len(out), "arrays")


def rng_streams():
    ref = load_reference()
    out = {}
    for seed in (0, 42, 2**40 + 7):
        out[f"normals_{seed}"] = ref.rng_normals(seed, 33)
        out[f"uniforms_{seed}"] = ref.rng_uniforms(seed, 33)
    np.savez_compressed(os.path.join(HERE, "rng_golden.npz"), **out)


def optimiser():
    """The reference's minimize (lbfgs.cpp:186-282) on analytic objectives and on a small registration."""
    ref = load_reference()
    out = {}

    def rosenbrock(x):
        f = 100.0 * (x[1] - x[0] ** 2) ** 2 + (1 - x[0]) ** 2
        g = np.array([-400.0 * x[0] * (x[1] - x[0] ** 2) - 2 * (1 - x[0]), 200.0 * (x[1] - x[0] ** 2)])
        return f, g

    r = ref.minimize(rosenbrock, np.array([-1.2, 1.0]), max_iter=200, grad_tol=1e-8)
    out["rosen_x"], out["rosen_hist_loss"] = r["x"], r["hist_loss"]
    out["rosen_counts"] = np.array([r["evaluations"], r["iterations"], r["reason"]])
    out["rosen_hist_step"], out["rosen_hist_evals"] = r["hist_step"], r["hist_evals"]

    diag = np.array([1.0, 10.0, 100.0, 0.5, 3.0])

    def quadratic(x):
        return 0.5 * float(np.sum(diag * x * x)), diag * x

    r = ref.minimize(quadratic, np.ones(5), max_iter=50, grad_tol=1e-10)
    out["quad_x"], out["quad_hist_loss"] = r["x"], r["hist_loss"]
    out["quad_counts"] = np.array([r["evaluations"], r["iterations"], r["reason"]])

    # small registration through the restated closure (registration.cpp:43-93), f64 and f32
    rng = np.random.default_rng(7)
    n = 96
    q0 = rng.uniform(-5, 5, (n, 3))
    target = q0 + 0.4 * rng.normal(size=(n, 3))
    out["reg_q0"], out["reg_target"] = q0, target
    for prec in ("f64", "f32"):
        r = ref.register(prec, q0, target, SIGMA, 50.0, 5, 12)
        out[f"reg_{prec}_momenta"], out[f"reg_{prec}_warped"] = r["momenta"], r["warped"]
        out[f"reg_{prec}_hist_loss"] = r["hist_loss"]
        out[f"reg_{prec}_summary"] = np.array([r["loss"], r["initial_loss"], r["evaluations"], r["iterations"],
                                               r["reason"]])
    out["reg_meta_sigma_lambda_T_iters"] = np.array([SIGMA, 50.0, 5, 12])
    np.savez_compressed(os.path.join(HERE, "optimiser_golden.npz"), **out)
    print("optimiser_golden.npz:", len(out), "arrays")


if __name__ == "__main__":
    hotpath()
    rng_streams()
    optimiser()
