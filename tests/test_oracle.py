"""CPU tests that pin the oracle (oracle/lmshoot_oracle.c): against the committed golden vectors
generated from the reference build, against the reference build itself when present, against the
analytic known-answer values of SPEC.md:148-216 and the finite-difference criteria of SPEC.md:173,207,217."""
import numpy as np
import pytest

from conftest import rel_inf, synth_case

SIGMA = 1.5
CASES = [(prec, dim, n) for prec in ("f32", "f64") for dim in (2, 3) for n in (1, 2, 7, 33, 200)]


@pytest.mark.parametrize("prec,dim,n", CASES)
def test_oracle_matches_golden_bitwise(oracle, golden_hotpath, prec, dim, n):
    g = golden_hotpath
    k = f"{prec}_d{dim}_n{n}_"
    q, p, target, alpha, beta, pts = (g[k + s] for s in ("q", "p", "target", "alpha", "beta", "pts"))
    hq, hp = oracle.derivatives(prec, q, p, SIGMA)
    assert np.array_equal(hq, g[k + "hq"]) and np.array_equal(hp, g[k + "hp"])
    assert oracle.hamiltonian(prec, q, p, SIGMA) == float(g[k + "H"])
    da, db = oracle.adjoint_step(prec, q, p, alpha, beta, SIGMA)
    assert np.array_equal(da, g[k + "dalpha"]) and np.array_equal(db, g[k + "dbeta"])
    assert oracle.mismatch_sq(prec, q, target) == float(g[k + "mismatch"])
    tq, tp = oracle.integrate_forward(prec, q, p, SIGMA, 4)
    assert np.array_equal(tq, g[k + "traj_q"]) and np.array_equal(tp, g[k + "traj_p"])
    loss, kin, mm, grad = oracle.compute_gradient(prec, q, p, target, SIGMA, 10.0, 4)
    assert np.array_equal(np.array([loss, kin, mm]), g[k + "scalars"])
    assert np.array_equal(grad, g[k + "grad"])
    assert np.array_equal(oracle.velocities(prec, q, p, pts, SIGMA), g[k + "vel"])
    assert np.array_equal(oracle.warp_points(prec, tq, tp, pts, SIGMA), g[k + "warped"])


def test_rng_matches_golden(oracle, golden_rng):
    for key, want in golden_rng.items():
        kind, seed = key.split("_")
        got = (oracle.rng_normals if kind == "normals" else oracle.rng_uniforms)(int(seed), want.size)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("strategy", ["sequential", "precompute_matrix", "blocked_tree"])
def test_oracle_matches_reference_build(oracle, reference, prec, strategy):
    for dim, n, seed in ((3, 257, 1), (2, 255, 2), (3, 600, 3)):
        q, p, target, alpha, beta = synth_case(n, dim, seed)
        for threads in (1, 3):
            a = oracle.derivatives(prec, q, p, SIGMA, strategy, 256, threads)
            b = reference.derivatives(prec, q, p, SIGMA, strategy, 256, threads)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        a = oracle.adjoint_step(prec, q, p, alpha, beta, SIGMA, strategy, 64)
        b = reference.adjoint_step(prec, q, p, alpha, beta, SIGMA, strategy, 64)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        a = oracle.compute_gradient(prec, q, p, target, SIGMA, 5e5, 3, strategy)
        b = reference.compute_gradient(prec, q, p, target, SIGMA, 5e5, 3, strategy)
        assert a[:3] == b[:3] and np.array_equal(a[3], b[3])


def test_survey_probe_values(oracle):
    """SURVEY.md §8c recorded values for the reference build: Rng(0), interleaved draws, N=1000."""
    n = 1000
    kinds = np.tile(np.array([0, 1, 1], dtype=np.uint8), n * 3)
    draws = oracle.rng_stream(0, kinds).reshape(n, 3, 3)
    q = -20.0 + 40.0 * draws[:, :, 0]
    p = 0.75 * draws[:, :, 1]
    target = q + 0.5 * draws[:, :, 2]
    loss, kin, mm, grad = oracle.compute_gradient("f64", q, p, target, 1.5, 10.0, 10)
    assert loss == pytest.approx(27731.548462408453, rel=1e-13)
    assert kin == pytest.approx(809.27571844628255, rel=1e-13)
    assert mm == pytest.approx(2692.2272743962171, rel=1e-13)
    assert float((grad * grad).sum()) == pytest.approx(2505931.5814837986, rel=1e-12)


# ---- analytic known answers -----------------------------------------------------
def test_kat_gaussian_kernel(oracle):
    assert oracle.gaussian_kernel("f64", 0.0, 1.5) == 1.0
    assert oracle.gaussian_kernel("f64", 2 * 1.5**2 * np.log(2.0), 1.5) == pytest.approx(0.5, rel=1e-15)
    assert oracle.gaussian_kernel("f64", 1.5**2, 1.5) == pytest.approx(0.606531, abs=5e-7)
    assert oracle.kernel_scale("f64", 1.5) == -0.5 / 2.25
    assert oracle.kernel_scale("f32", 1.5) == float(np.float32(-0.5) * (np.float32(1) / np.float32(2.25)))


def test_kat_hamiltonian(oracle):
    assert oracle.hamiltonian("f64", [[0, 0, 0]], [[1, 0, 0]], 1.5) == 0.5
    h = oracle.hamiltonian("f64", [[0, 0, 0], [1.5, 0, 0]], [[1, 0, 0], [1, 0, 0]], 1.5)
    assert h == pytest.approx(1 + np.exp(-0.5), rel=1e-15)
    q, p, *_ = synth_case(9, 3, 5)
    assert oracle.hamiltonian("f64", q, np.zeros_like(p), 1.5) == 0.0


def test_kat_single_landmark(oracle):
    q, p = np.array([[0.3, -1.0, 2.0]]), np.array([[1.0, 0.5, -0.25]])
    hq, hp = oracle.derivatives("f64", q, p, 1.5)
    assert np.array_equal(hp, p) and np.array_equal(hq, np.zeros_like(q))
    tq, _ = oracle.integrate_forward("f64", [[0, 0, 0]], [[1, 0, 0]], 1.5, 8)
    assert np.array_equal(tq[-1], [[1.0, 0, 0]])
    alpha, beta = np.array([[0.2, 0.1, -0.4]]), np.array([[1.0, 2.0, 3.0]])
    da, db = oracle.adjoint_step("f64", q, p, alpha, beta, 1.5)
    assert np.array_equal(da, np.zeros_like(q)) and np.array_equal(db, alpha)
    # N = 1, T = 1: grad = p0 + 2 lambda (q0 + p0 - target)
    target, lam = np.array([[1.0, 1.0, 1.0]]), 3.0
    loss, kin, mm, grad = oracle.compute_gradient("f64", q, p, target, 1.5, lam, 1)
    assert np.allclose(grad, p + 2 * lam * (q + p - target), rtol=1e-15)
    assert loss == pytest.approx(0.5 * float((p * p).sum()) + lam * float(((q + p - target) ** 2).sum()), rel=1e-15)


def test_kat_loss_examples(oracle):
    q, _, target, *_ = synth_case(6, 3, 11)
    zero = np.zeros_like(q)
    loss, *_ = oracle.compute_gradient("f64", q, zero, q, 1.5, 7.0, 3)
    assert loss == 0.0
    loss, kin, mm, _ = oracle.compute_gradient("f64", q, zero, target, 1.5, 7.0, 3)
    assert kin == 0.0 and loss == pytest.approx(7.0 * float(((q - target) ** 2).sum()), rel=1e-14)


# ---- finite-difference oracles -------------------------------------------------
def test_derivatives_vs_fd_of_hamiltonian(oracle):
    q, p, *_ = synth_case(30, 3, 21, spread=2.0)
    hq, hp = oracle.derivatives("f64", q, p, SIGMA)
    eps = 1e-5
    for arr, want in ((q, hq), (p, hp)):
        fd = np.zeros_like(arr)
        for idx in np.ndindex(*arr.shape):
            orig = arr[idx]
            arr[idx] = orig + eps
            hi = oracle.hamiltonian("f64", q, p, SIGMA)
            arr[idx] = orig - eps
            lo = oracle.hamiltonian("f64", q, p, SIGMA)
            arr[idx] = orig
            fd[idx] = (hi - lo) / (2 * eps)
        assert rel_inf(fd, want) <= 1e-6


def test_adjoint_vs_fd_jacobian(oracle):
    n, d = 20, 3
    q, p, _, alpha, beta = synth_case(n, d, 22, spread=2.0)

    def field(z):
        qq, pp = z[: n * d].reshape(n, d), z[n * d:].reshape(n, d)
        hq, hp = oracle.derivatives("f64", qq, pp, SIGMA)
        return np.concatenate([hp.ravel(), -hq.ravel()])

    z0 = np.concatenate([q.ravel(), p.ravel()])
    eps = 1e-5
    J = np.zeros((2 * n * d, 2 * n * d))
    for k in range(2 * n * d):
        zp, zm = z0.copy(), z0.copy()
        zp[k] += eps
        zm[k] -= eps
        J[:, k] = (field(zp) - field(zm)) / (2 * eps)
    want = J.T @ np.concatenate([alpha.ravel(), beta.ravel()])
    da, db = oracle.adjoint_step("f64", q, p, alpha, beta, SIGMA)
    assert rel_inf(np.concatenate([da.ravel(), db.ravel()]), want) <= 1e-6


@pytest.mark.parametrize("n,T", [(1, 1), (2, 5), (20, 10), (20, 1), (2, 40)])
def test_gradient_vs_fd_of_discrete_loss(oracle, n, T):
    q, p, target, *_ = synth_case(n, 3, 30 + n + T, spread=2.0)
    lam = 10.0
    _, _, _, grad = oracle.compute_gradient("f64", q, p, target, SIGMA, lam, T)
    eps = 1e-5
    fd = np.zeros_like(p)
    for idx in np.ndindex(*p.shape):
        orig = p[idx]
        p[idx] = orig + eps
        hi = oracle.compute_gradient("f64", q, p, target, SIGMA, lam, T)[0]
        p[idx] = orig - eps
        lo = oracle.compute_gradient("f64", q, p, target, SIGMA, lam, T)[0]
        p[idx] = orig
        fd[idx] = (hi - lo) / (2 * eps)
    assert rel_inf(fd, grad) <= 1e-6


# ---- invariants -------------------------------------------------------------
def test_invariants(oracle):
    q, p, target, *_ = synth_case(40, 3, 40)
    h = oracle.hamiltonian("f64", q, p, SIGMA)
    assert oracle.hamiltonian("f64", q + np.array([3.0, -2.0, 5.0]), p, SIGMA) == pytest.approx(h, rel=1e-12)
    _, tp = oracle.integrate_forward("f64", q, p, SIGMA, 100)
    drift = np.abs(tp.sum(axis=1) - p.sum(axis=0)).max()
    assert drift <= 1e-10 * np.linalg.norm(p, axis=1).sum()
    perm = np.random.default_rng(0).permutation(40)
    a = oracle.compute_gradient("f64", q, p, target, SIGMA, 10.0, 5, "sequential")
    b = oracle.compute_gradient("f64", q[perm], p[perm], target[perm], SIGMA, 10.0, 5, "sequential")
    assert b[0] == pytest.approx(a[0], rel=1e-12) and rel_inf(b[3], a[3][perm]) <= 1e-11


def test_backends_agree_and_tree_is_more_accurate(oracle):
    for n in (7, 200, 2000):
        q, p, *_ = synth_case(n, 3, 50 + n, spread=6.0)
        seq = oracle.derivatives("f64", q, p, SIGMA, "sequential")
        tree = oracle.derivatives("f64", q, p, SIGMA, "blocked_tree")
        pre = oracle.derivatives("f64", q, p, SIGMA, "precompute_matrix")
        assert np.array_equal(seq[0], pre[0]) and np.array_equal(seq[1], pre[1])
        assert rel_inf(tree[0], seq[0]) <= 1e-12 and rel_inf(tree[1], seq[1]) <= 1e-12
    q, p, *_ = synth_case(2000, 3, 77, spread=3.0)
    exact = oracle.derivatives("f64", q, p, SIGMA, "blocked_tree")[1]
    e_seq = np.abs(oracle.derivatives("f32", q, p, SIGMA, "sequential")[1] - exact).max()
    e_tree = np.abs(oracle.derivatives("f32", q, p, SIGMA, "blocked_tree")[1] - exact).max()
    assert e_tree <= e_seq
    vals = np.random.default_rng(1).normal(size=1000)
    assert oracle.tree_sum("f64", vals) == pytest.approx(float(np.sum(vals)), rel=1e-12)
    assert oracle.tree_sum("f64", []) == 0.0 and oracle.tree_sum("f32", [2.5]) == 2.5


def test_error_behaviour(oracle):
    from oracle.binding import OracleError

    q, p, target, *_ = synth_case(5, 3, 60)
    bad = p.copy()
    bad[2, 1] = np.nan
    with pytest.raises(OracleError) as e:
        oracle.integrate_forward("f64", q, bad, SIGMA, 3)
    assert e.value.code == 2 and e.value.timestep == 0  # DivergedError(0), shooting.hpp:185-186
    huge = p.copy()
    huge[0, 0] = 1e30
    with pytest.raises(OracleError) as e:
        oracle.integrate_forward("f32", q * 1e18, huge, SIGMA, 6)
    assert e.value.code == 2 and e.value.timestep >= 1  # first non-finite step, shooting.hpp:210-211
    with pytest.raises(OracleError) as e:
        oracle.derivatives("f64", q, p, -1.0)
    assert e.value.code == 3
    with pytest.raises(OracleError) as e:
        oracle.integrate_forward("f64", q, p, SIGMA, 0)
    assert e.value.code == 3
    # empty problem: zero loss, empty gradient
    z = np.zeros((0, 3))
    loss, kin, mm, grad = oracle.compute_gradient("f64", z, z, z, SIGMA, 1.0, 2)
    assert (loss, kin, mm) == (0.0, 0.0, 0.0) and grad.shape == (0, 3)


def test_pair_rows_equal_full_calls(oracle):
    """The row-subset helper used for full-size GPU checks is the same arithmetic as the full calls."""
    for prec in ("f32", "f64"):
        for dim in (2, 3):
            q, p, _, alpha, beta = synth_case(300, dim, 90 + dim)
            rows = [0, 5, 299, 128, 17]
            hq, hp = oracle.derivatives(prec, q, p, SIGMA)
            got = oracle.pair_rows(prec, q, p, rows, SIGMA)
            assert np.array_equal(got[0], hq[rows]) and np.array_equal(got[1], hp[rows])
            da, db = oracle.adjoint_step(prec, q, p, alpha, beta, SIGMA)
            got = oracle.pair_rows(prec, q, p, rows, SIGMA, alpha, beta)
            assert np.array_equal(got[0], da[rows]) and np.array_equal(got[1], db[rows])


def test_landmark_distances_restatement(oracle):
    """average_dist / max_dist (landmarks.cpp:148-179): hand-checked values (3-4-5 and 5-12-13 triangles, a
    coincident pair), the sequential-sum order, and two dimensions."""
    a = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [2.0, 0.0, -1.0]])
    b = np.array([[3.0, 4.0, 0.0], [1.0, 1.0, 1.0], [2.0, 5.0, 11.0]])
    avg, mx = oracle.landmark_distances(a, b)
    assert avg == (5.0 + 0.0 + 13.0) / 3.0 and mx == 13.0
    rng = np.random.default_rng(5)
    a2, b2 = rng.normal(size=(1000, 2)), rng.normal(size=(1000, 2))
    avg2, mx2 = oracle.landmark_distances(a2, b2)
    dist = [float(np.sqrt((x[0] - y[0]) * (x[0] - y[0]) + (x[1] - y[1]) * (x[1] - y[1]))) for x, y in zip(a2, b2)]
    total = 0.0
    for d in dist:
        total += d  # the reference's sequential order
    assert avg2 == total / 1000.0 and mx2 == max(dist)
