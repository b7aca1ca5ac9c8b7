"""The library's own L-BFGS driver (csrc/lbfgs_driver.cpp) against the reference's minimize
(lbfgs.cpp:186-282): committed golden runs, the reference build itself, and SPEC.md:355-357 sanity."""
import numpy as np
import pytest

from paper_1907_04839_b200 import LbfgsParams, NumericalError, minimize


def rosenbrock(x):
    f = 100.0 * (x[1] - x[0] ** 2) ** 2 + (1 - x[0]) ** 2
    g = np.array([-400.0 * x[0] * (x[1] - x[0] ** 2) - 2 * (1 - x[0]), 200.0 * (x[1] - x[0] ** 2)])
    return f, g


DIAG = np.array([1.0, 10.0, 100.0, 0.5, 3.0])


def quadratic(x):
    return 0.5 * float(np.sum(DIAG * x * x)), DIAG * x


def test_rosenbrock_matches_golden_iterate_for_iterate(golden_optimiser):
    g = golden_optimiser
    r = minimize(rosenbrock, [-1.2, 1.0], LbfgsParams(max_iter=200, grad_tol=1e-8))
    evals, iters, reason = (int(v) for v in g["rosen_counts"])
    assert (r.evaluations, len(r.iterations)) == (evals, iters)
    assert r.reason == ("gradient-tolerance", "max-iterations", "line-search-failure")[reason]
    assert np.array_equal(r.x, g["rosen_x"])
    assert np.array_equal([it[0] for it in r.iterations], g["rosen_hist_loss"])
    assert np.array_equal([it[2] for it in r.iterations], g["rosen_hist_step"])
    assert np.array_equal([it[3] for it in r.iterations], g["rosen_hist_evals"])
    assert np.allclose(r.x, [1.0, 1.0], atol=1e-6)


def test_quadratic_matches_golden(golden_optimiser):
    g = golden_optimiser
    r = minimize(quadratic, np.ones(5), LbfgsParams(max_iter=50, grad_tol=1e-10))
    assert np.array_equal(r.x, g["quad_x"])
    assert np.array_equal([it[0] for it in r.iterations], g["quad_hist_loss"])
    assert (r.evaluations, len(r.iterations)) == tuple(int(v) for v in g["quad_counts"][:2])


def test_well_conditioned_quadratic_in_three_iterations():
    r = minimize(lambda x: (0.5 * float(x @ x), x.copy()), np.array([3.0, -4.0, 5.0]), LbfgsParams(grad_tol=1e-9))
    assert len(r.iterations) <= 3 and r.reason == "gradient-tolerance"


def test_accepted_losses_are_monotone():
    r = minimize(rosenbrock, [-1.2, 1.0], LbfgsParams(max_iter=60))
    losses = [r.initial_loss] + [it[0] for it in r.iterations]
    assert all(b <= a for a, b in zip(losses, losses[1:]))


def test_against_reference_minimize_on_oracle_objective(oracle, reference):
    """Same objective (the CPU oracle's compute_gradient), two drivers: identical iterates."""
    rng = np.random.default_rng(3)
    n = 40
    q0 = rng.uniform(-3, 3, (n, 3))
    target = q0 + 0.3 * rng.normal(size=(n, 3))

    def objective(x):
        loss, _, _, grad = oracle.compute_gradient("f64", q0, x.reshape(n, 3), target, 1.5, 20.0, 4)
        return loss, grad.ravel()

    x0 = ((target - q0) / 4).ravel()
    mine = minimize(objective, x0, LbfgsParams(max_iter=15))
    theirs = reference.minimize(objective, x0, max_iter=15)
    assert mine.evaluations == theirs["evaluations"] and len(mine.iterations) == theirs["iterations"]
    assert np.array_equal(mine.x, theirs["x"]) and mine.loss == theirs["loss"]
    assert np.array_equal([it[0] for it in mine.iterations], theirs["hist_loss"])


def test_error_behaviour():
    with pytest.raises(NumericalError):
        minimize(lambda x: (float("nan"), x), [1.0, 2.0])  # lbfgs.cpp:197-198
    with pytest.raises(ValueError):
        minimize(quadratic, np.ones(5), LbfgsParams(c1=0.95))
    with pytest.raises(ValueError):
        minimize(quadratic, np.ones(5), LbfgsParams(memory=0))
    # already optimal: returns at once with gradient-tolerance and one evaluation
    r = minimize(quadratic, np.zeros(5))
    assert r.reason == "gradient-tolerance" and r.evaluations == 1 and not r.iterations
    # a line search that can only overshoot must fail cleanly, not hang
    calls = []

    def cliff(x):
        calls.append(1)
        return (float(x[0] ** 2) if abs(x[0]) <= 1.0 else float("inf")), np.array([2 * x[0]])

    r = minimize(cliff, [1.0], LbfgsParams(max_iter=5))
    assert np.isfinite(r.loss) and len(calls) < 200
