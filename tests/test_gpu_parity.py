"""GPU parity tests proper: the CUDA path, called through the C ABI (ctypes -> liblmshoot_b200.so),
against the CPU oracle on the same seeded inputs, against the committed golden fixtures, and -- at
BASELINE.json's full sizes -- through row subsets and size-independent properties.

Tolerances (BASELINE.json north_star / BASELINE.md §4): loss, H and ||dg||_inf/||g||_inf per evaluation
within 1e-10 in fp64 and 1e-5 in fp32 (at well-conditioned evaluation points); integer/index results and
the strictly sequential double sums are bit-exact."""
import ctypes

import numpy as np
import pytest

from conftest import rel_inf, synth_case

pytestmark = pytest.mark.gpu

SIGMA = 1.5
TOL = {"f64": 1e-10, "f32": 1e-5}
EDGE_N = [1, 2, 7, 255, 256, 257, 513, 1000]


@pytest.fixture(scope="module")
def hs():
    from paper_1907_04839_b200 import HamiltonianSystem

    cache = {}

    def make(n, dim, prec, max_t=40, variant=0, tiled_only=False):
        key = (n, dim, prec, max_t, variant, tiled_only)
        if key not in cache:
            cache[key] = HamiltonianSystem(SIGMA, n, dim, prec, device=0, max_timesteps=max_t, variant=variant,
                                           tiled_only=tiled_only)
        return cache[key]

    yield make
    for s in cache.values():
        s.close()


def test_extension_is_loaded_and_runs_on_device(hs):
    import ctypes

    from paper_1907_04839_b200 import _lib

    assert isinstance(_lib.load(), ctypes.CDLL)
    q, p, target, *_ = synth_case(64, 3, 1)
    s = hs(64, 3, "f32")  # small problems: the whole evaluation is one persistent kernel
    s.compute_gradient(q, p, target, 10.0, 4)
    assert s.last_eval_kernel_launches() == 1
    assert s.last_eval_device_ms() > 0.0
    s = hs(64, 3, "f32", tiled_only=True)  # the tiled path: conversion + T forward + scalars + T adjoint launches
    s.compute_gradient(q, p, target, 10.0, 4)
    assert s.last_eval_kernel_launches() == 2 * 4 + 2
    assert s.last_eval_device_ms() > 0.0


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("n", [1, 2, 7, 33, 200])
def test_against_golden_fixtures(hs, golden_hotpath, prec, dim, n):
    g, k, tol = golden_hotpath, f"{prec}_d{dim}_n{n}_", TOL[prec]
    q, p, target, alpha, beta, pts = (g[k + s] for s in ("q", "p", "target", "alpha", "beta", "pts"))
    s = hs(n, dim, prec)
    hq, hp = s.derivatives(q, p)
    assert rel_inf(hq, g[k + "hq"]) <= tol and rel_inf(hp, g[k + "hp"]) <= tol
    assert s.hamiltonian(q, p) == pytest.approx(float(g[k + "H"]), rel=tol)
    da, db = s.adjoint_step(q, p, alpha, beta)
    assert rel_inf(da, g[k + "dalpha"]) <= tol and rel_inf(db, g[k + "dbeta"]) <= tol
    assert s.mismatch_sq(q, target) == float(g[k + "mismatch"])  # sequential double sum: bit-exact
    tq, tp = s.integrate_forward(q, p, 4)
    assert rel_inf(tq, g[k + "traj_q"]) <= tol and rel_inf(tp, g[k + "traj_p"]) <= tol
    assert np.array_equal(tq[0], g[k + "traj_q"][0])  # snapshot 0 is the input cast to T, exactly
    assert rel_inf(s.warp_points(pts), g[k + "warped"]) <= tol
    assert rel_inf(s.velocities_at_step(q, p, pts), g[k + "vel"]) <= tol
    r = s.compute_gradient(q, p, target, 10.0, 4)
    want = g[k + "scalars"]
    assert r.loss == pytest.approx(want[0], rel=tol) and r.kinetic == pytest.approx(want[1], rel=tol)
    assert r.mismatch == pytest.approx(want[2], rel=tol)
    assert rel_inf(r.grad, g[k + "grad"]) <= tol


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("n", EDGE_N)
def test_per_function_parity_vs_oracle(hs, oracle, prec, n):
    """Tile-boundary sizes (255/256/257 straddle the 128-column tile and the 256/512-row tiles)."""
    tol = TOL[prec]
    q, p, target, alpha, beta = synth_case(n, 3, 100 + n, spread=6.0)
    s = hs(n, 3, prec)
    hq, hp = s.derivatives(q, p)
    ohq, ohp = oracle.derivatives(prec, q, p, SIGMA)
    assert rel_inf(hq, ohq) <= tol and rel_inf(hp, ohp) <= tol
    da, db = s.adjoint_step(q, p, alpha, beta)
    oda, odb = oracle.adjoint_step(prec, q, p, alpha, beta, SIGMA)
    assert rel_inf(da, oda) <= tol and rel_inf(db, odb) <= tol
    assert s.hamiltonian(q, p) == pytest.approx(oracle.hamiltonian(prec, q, p, SIGMA), rel=tol)
    assert s.mismatch_sq(q, target) == oracle.mismatch_sq(prec, q, target)
    tq, tp = s.integrate_forward(q, p, 10)
    otq, otp = oracle.integrate_forward(prec, q, p, SIGMA, 10)
    assert rel_inf(tq, otq) <= tol and rel_inf(tp, otp) <= tol


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("n,T,lam", [(1, 1, 3.0), (2, 5, 10.0), (7, 10, 10.0), (257, 10, 10.0), (1000, 10, 10.0),
                                     (1000, 10, 5e5), (600, 40, 5e5)])
@pytest.mark.parametrize("tiled_only", [False, True], ids=["persistent", "tiled"])
def test_compute_gradient_parity(hs, oracle, prec, n, T, lam, tiled_only):
    """The complete objective evaluation against the oracle, through both device paths: the persistent
    one-launch kernel small problems select by default, and the tiled stream-K kernels (pinned)."""
    tol = TOL[prec]
    q, p, target, *_ = synth_case(n, 3, 200 + n + T, spread=8.0)
    s = hs(n, 3, prec, tiled_only=tiled_only)
    r = s.compute_gradient(q, p, target, lam, T)
    loss, kin, mm, grad = oracle.compute_gradient(prec, q, p, target, SIGMA, lam, T)
    assert r.loss == pytest.approx(loss, rel=tol)
    assert r.kinetic == pytest.approx(kin, rel=tol)
    assert r.mismatch == pytest.approx(mm, rel=tol)
    assert rel_inf(r.grad, grad) <= tol
    assert rel_inf(s.final_q(), oracle.integrate_forward(prec, q, p, SIGMA, T)[0][-1]) <= tol


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 31, 32, 33, 255, 256, 257, 295, 296, 297, 511, 512, 513, 1000, 1184, 1185, 2047, 2048,
                               2049, 2369, 2900, 3400, 3401, 4095, 4096, 4097, 4737, 8191, 8192, 8193])
def test_persistent_kernel_edge_sizes(hs, oracle, prec, dim, n):
    """The persistent path at the sizes where its decomposition changes: fewer rows than one slot, fewer work items
    than warps, one chunk of staged columns +- 1 (2048 fp32 / 1024 fp64), one slot per CTA +- 1 (148 SMs x 2 rows),
    several slots per CTA (a warp's run then spans two or three slots: 4737 is the first size with more than 16),
    one adjoint window +- 1 (4096 fp32 / 2048 fp64: above it the adjoint sweep stages two windows per step), the
    largest size it is chosen for +- 1 (8192 fp32, the capacity; 3400 fp64, the crossover with the tiled path), an
    odd last row of a packed pair; odd T and even T end in different adjoint buffers.  Checked against the
    oracle, against the tiled path (same epilogue arithmetic, different summation order) and for run-to-run bits."""
    tol = TOL[prec]
    # constant landmark density (a denser cloud than ~500 per 14^dim box makes the flow itself ill-conditioned in fp32)
    q, p, target, *_ = synth_case(n, dim, 4000 + n + dim, spread=7.0 * max(1.0, (n / 500.0) ** (1.0 / dim)))
    s = hs(n, dim, prec, max_t=8)
    tiled = hs(n, dim, prec, max_t=8, tiled_only=True)
    for T in (3, 4):
        r = s.compute_gradient(q, p, target, 25.0, T)
        # the persistent kernel stages the state in shared memory: chosen up to 8192 landmarks in fp32, 3400 in fp64
        assert s.last_eval_kernel_launches() == (1 if n <= (8192 if prec == "f32" else 3400) else 2 * T + 2)
        loss, kin, mm, grad = oracle.compute_gradient(prec, q, p, target, SIGMA, 25.0, T)
        assert r.loss == pytest.approx(loss, rel=tol) and r.kinetic == pytest.approx(kin, rel=tol, abs=1e-300)
        assert r.mismatch == pytest.approx(mm, rel=tol)
        assert rel_inf(r.grad, grad) <= tol
        assert rel_inf(s.final_q(), oracle.integrate_forward(prec, q, p, SIGMA, T)[0][-1]) <= tol
        again = s.compute_gradient(q, p, target, 25.0, T)
        assert again.loss == r.loss and np.array_equal(again.grad, r.grad)
        rt = tiled.compute_gradient(q, p, target, 25.0, T)
        assert rt.loss == pytest.approx(r.loss, rel=tol) and rel_inf(rt.grad, r.grad) <= tol
    # the stored trajectory of the persistent evaluation feeds the warp exactly like the tiled one's
    assert rel_inf(s.warp_points(q), s.final_q()) <= 3 * tol  # two different fp32 summation orders


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("n", [4500, 6100, 8200, 11000])
def test_mid_size_parity(hs, oracle, prec, n):
    """Mid-size single problems, where the machinery differs from both ends of the range: the persistent kernel with
    two adjoint windows per step (fp32 up to 8192), and on the tiled path programmatic dependent launch between the pair
    kernels (below 8000 landmarks), the combine's shared-memory landing zone (at most two CTAs per SM, up to 20
    partial segments per row tile), four-row shapes from 8000 on unless they pad more than they gain (11 000).
    Against the oracle, and bitwise run to run."""
    tol = TOL[prec]
    T, lam = 3, 50.0
    q, p, target, *_ = synth_case(n, 3, 5000 + n, spread=7.0 * (n / 500.0) ** (1.0 / 3))
    s = hs(n, 3, prec, max_t=4)
    r = s.compute_gradient(q, p, target, lam, T)
    persistent = n <= (8192 if prec == "f32" else 3400)  # the persistent kernel's range (two adjoint windows above 4096 / 2048)
    assert s.last_eval_kernel_launches() == (1 if persistent else 2 * T + 2)
    loss, kin, mm, grad = oracle.compute_gradient(prec, q, p, target, SIGMA, lam, T)
    assert r.loss == pytest.approx(loss, rel=tol) and r.kinetic == pytest.approx(kin, rel=tol)
    assert r.mismatch == pytest.approx(mm, rel=tol)
    assert rel_inf(r.grad, grad) <= tol
    again = s.compute_gradient(q, p, target, lam, T)
    assert again.loss == r.loss and np.array_equal(again.grad, r.grad)


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_two_dimensional_landmarks(hs, oracle, prec):
    tol = TOL[prec]
    q, p, target, alpha, beta = synth_case(300, 2, 7, spread=5.0)
    s = hs(300, 2, prec)
    r = s.compute_gradient(q, p, target, 10.0, 6)
    loss, kin, mm, grad = oracle.compute_gradient(prec, q, p, target, SIGMA, 10.0, 6)
    assert r.loss == pytest.approx(loss, rel=tol) and rel_inf(r.grad, grad) <= tol
    da, db = s.adjoint_step(q, p, alpha, beta)
    oda, odb = oracle.adjoint_step(prec, q, p, alpha, beta, SIGMA)
    assert rel_inf(da, oda) <= tol and rel_inf(db, odb) <= tol


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("variant", [1, 5])
def test_kernel_variants_agree_with_oracle(hs, oracle, prec, variant):
    tol = TOL[prec]
    n = 700
    q, p, target, *_ = synth_case(n, 3, 300 + variant, spread=7.0)
    s = hs(n, 3, prec, variant=variant)
    r = s.compute_gradient(q, p, target, 10.0, 5)
    loss, kin, mm, grad = oracle.compute_gradient(prec, q, p, target, SIGMA, 10.0, 5)
    assert r.loss == pytest.approx(loss, rel=tol) and rel_inf(r.grad, grad) <= tol


@pytest.mark.parametrize("variant", [0, 11, 25])
@pytest.mark.parametrize("n", [300, 1100, 2300])
def test_fp32_shape_variants_agree_with_oracle(hs, oracle, variant, n):
    """The default shapes (0), the pinned two-row shapes (11) and four rows per thread with column-major adjoint
    tiles (25 = the default from N = 16 000): sizes below, at and above one row tile of every shape (256 / 512 rows),
    with plane lengths that are not multiples of the larger tile."""
    q, p, target, *_ = synth_case(n, 3, 700 + variant + n, spread=7.0)
    s = hs(n, 3, "f32", variant=variant)
    r = s.compute_gradient(q, p, target, 10.0, 4)
    loss, kin, mm, grad = oracle.compute_gradient("f32", q, p, target, SIGMA, 10.0, 4)
    assert r.loss == pytest.approx(loss, rel=1e-5) and rel_inf(r.grad, grad) <= 1e-5
    again = s.compute_gradient(q, p, target, 10.0, 4)
    assert np.array_equal(again.grad, r.grad)
    hq, hp = s.derivatives(q, p)
    ohq, ohp = oracle.derivatives("f32", q, p, SIGMA)
    assert rel_inf(hq, ohq) <= 1e-5 and rel_inf(hp, ohp) <= 1e-5
    alpha, beta = p[::-1].copy(), q[::-1].copy() * 0.1
    da, db = s.adjoint_step(q, p, alpha, beta)
    oda, odb = oracle.adjoint_step("f32", q, p, alpha, beta, SIGMA)
    assert rel_inf(da, oda) <= 1e-5 and rel_inf(db, odb) <= 1e-5


@pytest.mark.parametrize("variant,n", [(25, n) for n in (30, 64, 65, 128, 129, 544, 576, 577, 640, 641, 768, 769, 1056, 1080, 2180)]
                         + [(0, n) for n in (20, 64, 65, 300, 320, 321, 384, 385, 1100)])
def test_thin_last_row_tile_agrees_with_oracle(hs, oracle, variant, n):
    """The tiled path's thin last row tile: a last 512-row tile (four-row shapes, variant 25 = the default of large
    problems) or 256-row tile (two-row shapes, variant 0 at these sizes) holding at most a quarter (half) of its rows
    is swept with those rows replicated over 4 (2) groups of warps, each sweeping a quarter (half) of every staged
    column tile, with phantom cells in the stream-K cell space; at most an eighth of a four-row tile (64 rows) is swept
    8 ways -- the two packed row pairs of a thread hold the same rows and take the two halves of the group's window.  Sizes at and around both thresholds, a single thin
    tile, and thin tiles behind one to four full ones; every entry point that launches the pair kernels, and
    run-to-run bitwise reproducibility."""
    q, p, target, *_ = synth_case(n, 3, 900 + n, spread=7.0)
    s = hs(n, 3, "f32", variant=variant, tiled_only=True)
    r = s.compute_gradient(q, p, target, 10.0, 4)
    loss, kin, mm, grad = oracle.compute_gradient("f32", q, p, target, SIGMA, 10.0, 4)
    assert r.loss == pytest.approx(loss, rel=1e-5) and rel_inf(r.grad, grad) <= 1e-5
    again = s.compute_gradient(q, p, target, 10.0, 4)
    assert np.array_equal(again.grad, r.grad) and again.loss == r.loss
    hq, hp = s.derivatives(q, p)
    ohq, ohp = oracle.derivatives("f32", q, p, SIGMA)
    assert rel_inf(hq, ohq) <= 1e-5 and rel_inf(hp, ohp) <= 1e-5
    assert s.hamiltonian(q, p) == pytest.approx(oracle.hamiltonian("f32", q, p, SIGMA), rel=1e-5)
    alpha, beta = p[::-1].copy(), q[::-1].copy() * 0.1
    da, db = s.adjoint_step(q, p, alpha, beta)
    oda, odb = oracle.adjoint_step("f32", q, p, alpha, beta, SIGMA)
    assert rel_inf(da, oda) <= 1e-5 and rel_inf(db, odb) <= 1e-5


@pytest.mark.parametrize("n", [544, 1200])
def test_thin_last_row_tile_two_dimensional(hs, oracle, n):
    q, p, target, *_ = synth_case(n, 2, 60 + n, spread=9.0)
    s = hs(n, 2, "f32", variant=25, tiled_only=True)
    r = s.compute_gradient(q, p, target, 10.0, 4)
    loss, kin, mm, grad = oracle.compute_gradient("f32", q, p, target, SIGMA, 10.0, 4)
    assert r.loss == pytest.approx(loss, rel=1e-5) and rel_inf(r.grad, grad) <= 1e-5


@pytest.mark.parametrize("n", [700, 1500])
def test_two_dimensional_four_row_shapes(hs, oracle, n):
    """D = 2 with the shapes large problems select (variant 25)."""
    q, p, target, *_ = synth_case(n, 2, 40 + n, spread=9.0)
    s = hs(n, 2, "f32", variant=25)
    r = s.compute_gradient(q, p, target, 10.0, 4)
    loss, kin, mm, grad = oracle.compute_gradient("f32", q, p, target, SIGMA, 10.0, 4)
    assert r.loss == pytest.approx(loss, rel=1e-5) and rel_inf(r.grad, grad) <= 1e-5


def test_default_shapes_switch_with_problem_size(hs):
    """Variant 0 chooses the kernel shapes by problem size (System::pick_kernels)."""
    r2 = b"fwd_f32x2_r2_j4_b6_u2_tma / adj_f32x2_r2_j2_b5_u2"
    r4 = b"fwd_f32x2_r4_j4_b3_u2_tma / adj_f32x2_r4_aos_b3_u4"
    # four rows per thread from N = 10 500 on, unless their 512-row tiles pad more than they gain -- a last tile that is
    # at most half live rows counts as the thin tile it is swept as (N = 11 000: 0.36 % vs 0.07 %; N = 12 200: last tile
    # 424 live rows of 512, 0.7 % more padding than 256-row tiles, still within the 1.5 % the shapes gain)
    for n, want in ((2000, r2), (7000, r2), (10000, r2), (11000, r4), (12200, r4), (16000, r4), (20000, r4)):
        s = hs(n, 3, "f32")
        assert s.lib.lms_system_kernel_names(s.handle) == want, n


def test_known_answers_through_the_abi(hs):
    """SPEC.md:158-216 closed forms, fp64."""
    s1 = hs(1, 3, "f64")
    q, p = np.array([[0.3, -1.0, 2.0]]), np.array([[1.0, 0.5, -0.25]])
    assert s1.hamiltonian([[0, 0, 0]], [[1, 0, 0]]) == 0.5
    hq, hp = s1.derivatives(q, p)
    assert np.array_equal(hp, p) and np.array_equal(hq, np.zeros_like(q))
    tq, _ = s1.integrate_forward([[0, 0, 0]], [[1, 0, 0]], 8)
    assert np.allclose(tq[-1], [[1.0, 0, 0]], rtol=0, atol=1e-15)
    alpha, beta = np.array([[0.2, 0.1, -0.4]]), np.array([[1.0, 2.0, 3.0]])
    da, db = s1.adjoint_step(q, p, alpha, beta)
    assert np.array_equal(da, np.zeros_like(q)) and np.array_equal(db, alpha)
    target, lam = np.array([[1.0, 1.0, 1.0]]), 3.0
    r = s1.compute_gradient(q, p, target, lam, 1)
    assert np.allclose(r.grad, p + 2 * lam * (q + p - target), rtol=1e-15)
    s2 = hs(2, 3, "f64")
    h = s2.hamiltonian([[0, 0, 0], [1.5, 0, 0]], [[1, 0, 0], [1, 0, 0]])
    assert h == pytest.approx(1 + np.exp(-0.5), rel=1e-14)
    q6, _, t6, *_ = synth_case(6, 3, 11)
    s6 = hs(6, 3, "f64")
    r = s6.compute_gradient(q6, np.zeros_like(q6), q6, 7.0, 3)
    assert r.loss == 0.0 and not r.grad.any()
    r = s6.compute_gradient(q6, np.zeros_like(q6), t6, 7.0, 3)
    assert r.kinetic == 0.0 and r.loss == pytest.approx(7.0 * float(((q6 - t6) ** 2).sum()), rel=1e-14)


def test_gradient_vs_finite_differences_on_device(hs):
    """the device gradient is the exact gradient of the device's own discrete loss."""
    n, T, lam = 20, 10, 10.0
    q, p, target, *_ = synth_case(n, 3, 61, spread=2.0)
    s = hs(n, 3, "f64")
    grad = s.compute_gradient(q, p, target, lam, T).grad
    s.bind_registration(q, target, lam, T)
    eps = 1e-5
    fd = np.zeros_like(p)
    for idx in np.ndindex(*p.shape):
        orig = p[idx]
        p[idx] = orig + eps
        hi, _ = s.objective(p)
        p[idx] = orig - eps
        lo, _ = s.objective(p)
        p[idx] = orig
        fd[idx] = (hi - lo) / (2 * eps)
    assert rel_inf(fd, grad) <= 1e-6


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("tiled_only", [False, True], ids=["persistent", "tiled"])
def test_bitwise_run_to_run_determinism(hs, prec, tiled_only):
    n = 3000
    q, p, target, *_ = synth_case(n, 3, 5, spread=10.0)
    s = hs(n, 3, prec, tiled_only=tiled_only)
    s.bind_registration(q, target, 5e5, 10)
    first = s.objective(p)
    for _ in range(3):
        again = s.objective(p)
        assert again[0] == first[0] and np.array_equal(again[1], first[1])
    # a fresh handle (new buffers, new graph) gives the same bits too
    from paper_1907_04839_b200 import HamiltonianSystem

    other = HamiltonianSystem(SIGMA, n, 3, prec, max_timesteps=10, tiled_only=tiled_only)
    other.bind_registration(q, target, 5e5, 10)
    fresh = other.objective(p)
    other.close()
    assert fresh[0] == first[0] and np.array_equal(fresh[1], first[1])


def test_divergence_semantics(hs, oracle):
    from oracle.binding import OracleError
    from paper_1907_04839_b200 import DivergedError

    n = 40
    q, p, target, *_ = synth_case(n, 3, 8)
    s = hs(n, 3, "f32")
    bad = p.copy()
    bad[3, 1] = np.nan
    with pytest.raises(DivergedError) as e:
        s.integrate_forward(q, bad, 5)
    assert e.value.timestep == 0  # shooting.hpp:185-186
    with pytest.raises(DivergedError) as e:
        s.compute_gradient(q, bad, target, 1.0, 5)
    assert e.value.timestep == 0
    bad_q = q.copy()
    bad_q[0, 0] = np.inf
    with pytest.raises(DivergedError) as e:
        s.compute_gradient(bad_q, p, target, 1.0, 5)
    assert e.value.timestep == 0
    # overflow part-way: the reported step equals the reference's first non-finite step (:210-211)
    huge = p.copy()
    huge[0, 0] = 1e30
    with pytest.raises(OracleError) as want:
        oracle.integrate_forward("f32", q * 1e18, huge, SIGMA, 6)
    with pytest.raises(DivergedError) as got:
        s.integrate_forward(q * 1e18, huge, 6)
    assert got.value.timestep == want.value.timestep >= 1
    # the handle stays usable after an error
    r = s.compute_gradient(q, p, target, 1.0, 5)
    assert np.isfinite(r.loss)


def test_shape_and_state_errors(hs):
    from paper_1907_04839_b200 import HamiltonianSystem, ShapeError, StateError

    s = hs(10, 3, "f64")
    q, p, *_ = synth_case(10, 3, 1)
    with pytest.raises(ShapeError):
        s.derivatives(q, p[:9])  # require_same, shooting.hpp:332-338
    with pytest.raises(ShapeError):
        s.derivatives(q[:, :2], p[:, :2])
    with pytest.raises(ValueError):
        s.integrate_forward(q, p, 0)  # shooting.hpp:184
    with pytest.raises(ValueError):
        s.integrate_forward(q, p, 41)  # beyond the handle's trajectory capacity
    fresh = HamiltonianSystem(SIGMA, 10, 3, "f64", max_timesteps=4)
    with pytest.raises(StateError):
        fresh.objective(p)
    with pytest.raises(StateError):
        fresh.warp_points(q)
    fresh.close()


def test_empty_problem(hs):
    s = hs(0, 3, "f64")
    z = np.zeros((0, 3))
    r = s.compute_gradient(z, z, z, 1.0, 2)
    assert (r.loss, r.kinetic, r.mismatch) == (0.0, 0.0, 0.0) and r.grad.shape == (0, 3)
    assert s.hamiltonian(z, z) == 0.0


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_flow_velocities_and_warp(hs, oracle, prec):
    tol = TOL[prec]
    n, m, T = 500, 1300, 10
    q, p, *_ = synth_case(n, 3, 17, spread=6.0)
    pts = np.random.default_rng(3).uniform(-7, 7, (m, 3))
    s = hs(n, 3, prec)
    assert rel_inf(s.velocities_at_step(q, p, pts), oracle.velocities(prec, q, p, pts, SIGMA)) <= tol
    tq, tp = s.integrate_forward(q, p, T)
    otq, otp = oracle.integrate_forward(prec, q, p, SIGMA, T)
    assert rel_inf(s.warp_points(pts), oracle.warp_points(prec, otq, otp, pts, SIGMA)) <= tol
    # warping the template itself reproduces q(T)
    assert rel_inf(s.warp_points(q), tq[-1]) <= tol


def test_dense_warp_between_evaluations_keeps_the_graph_valid(hs):
    """bind -> evaluate -> warp a point set 100x larger than the landmark set -> evaluate again: the captured
    evaluation graph holds the stream-K partial / counter buffers, so nothing a larger launch needs may be
    reallocated under it.  The second evaluation must be bitwise the first."""
    n, T = 1000, 6
    q, p, target, *_ = synth_case(n, 3, 99, spread=8.0)
    for prec in ("f32", "f64"):
        s = hs(n, 3, prec, max_t=T)
        s.bind_registration(q, target, 50.0, T)
        loss1, grad1 = s.objective(p)
        grad1 = grad1.copy()
        pts = np.random.default_rng(12).uniform(-9, 9, (100 * n, 3))
        moved = s.warp_points(pts)
        assert np.isfinite(moved).all()
        vel = s.velocities_at_step(q, p, pts)
        assert np.isfinite(vel).all()
        loss2, grad2 = s.objective(p)
        assert loss2 == loss1 and np.array_equal(grad2, grad1)
        # and the dense warp agrees with warping in small pieces (different stream-K splits, same per-row order
        # within a CTA range: equal to rounding)
        piece = s.warp_points(pts[:1500])
        assert rel_inf(moved[:1500], piece) <= TOL[prec]


# ---- full-size checks (BASELINE.json configs[1]: N = 20 000, T = 10) ---------------------------------------
@pytest.fixture(scope="module")
def full_case():
    from paper_1907_04839_b200 import make_synthetic_pair

    n, T = 20000, 10
    # constant landmark density (radius ~ sqrt(N)): the fixed-diameter N = 20 000 flow is chaotic
    q0, target, p_true = make_synthetic_pair(n, SIGMA, T, density_scaled=True)
    x0 = (target - q0) / T  # paper initialisation, registration.cpp:47-52
    return n, T, q0, target, p_true, x0


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_full_size_row_subset_parity(hs, oracle, full_case, prec):
    """N = 20 000: 96 rows of derivatives and adjoint_step against the oracle's identical per-row sums."""
    n, T, q0, target, p_true, x0 = full_case
    tol = TOL[prec]
    rows = np.unique(np.concatenate([[0, 1, 127, 128, 511, 512, n - 1], np.random.default_rng(9).integers(0, n, 89)]))
    s = hs(n, 3, prec, max_t=T)
    hq, hp = s.derivatives(q0, p_true)
    ohq, ohp = oracle.pair_rows(prec, q0, p_true, rows, SIGMA)
    scale_q, scale_p = np.abs(hq).max(), np.abs(hp).max()
    assert np.abs(hq[rows] - ohq).max() <= tol * scale_q and np.abs(hp[rows] - ohp).max() <= tol * scale_p
    rng = np.random.default_rng(10)
    alpha, beta = rng.normal(size=(n, 3)), rng.normal(size=(n, 3))
    da, db = s.adjoint_step(q0, p_true, alpha, beta)
    oda, odb = oracle.pair_rows(prec, q0, p_true, rows, SIGMA, alpha, beta)
    assert np.abs(da[rows] - oda).max() <= tol * np.abs(da).max()
    assert np.abs(db[rows] - odb).max() <= tol * np.abs(db).max()


def test_full_size_properties_fp64(hs, full_case):
    """Size-independent properties at N = 20 000."""
    n, T, q0, target, p_true, x0 = full_case
    s = hs(n, 3, "f64", max_t=T)
    # the synthetic target is reachable: shooting with the true momenta lands on it exactly
    tq, tp = s.integrate_forward(q0, p_true, T)
    assert np.array_equal(tq[-1], target)
    # total momentum is conserved by the Euler flow
    drift = np.abs(tp.sum(axis=1) - p_true.sum(axis=0)).max()
    assert drift <= 1e-10 * np.linalg.norm(p_true, axis=1).sum()
    # translation invariance of H, and H = 1/2 sum p.hp
    h = s.hamiltonian(q0, p_true)
    assert s.hamiltonian(q0 + np.array([3.0, -2.0, 5.0]), p_true) == pytest.approx(h, rel=1e-12)
    hq, hp = s.derivatives(q0, p_true)
    assert 0.5 * float((p_true * hp).sum()) == pytest.approx(h, rel=1e-12)
    assert np.abs(hq.sum(axis=0)).max() <= 1e-9 * np.abs(hq).sum()
    # gradient: at p_true the mismatch vanishes, so grad = hp(q0, p_true) and loss = H
    s.bind_registration(q0, target, 5e5, T)
    loss, grad = s.objective(p_true)
    assert loss == pytest.approx(h, rel=1e-12)
    assert rel_inf(grad.reshape(n, 3), hp) <= 1e-9
    # directional finite difference of the discrete loss at the paper's initial point
    rng = np.random.default_rng(4)
    v = rng.normal(size=x0.shape)
    v /= np.linalg.norm(v)
    loss0, g0 = s.objective(x0)
    # loss0 ~ 2e10 carries ~1e-5 of absolute rounding noise and the slope is ~2e6 along a unit vector: a step of
    # 1e-4 keeps the difference quotient's noise at ~1e-7 relative (1e-6 left it at ~1e-6, the tolerance itself)
    eps = 1e-4
    hi, _ = s.objective(x0 + eps * v)
    lo, _ = s.objective(x0 - eps * v)
    assert (hi - lo) / (2 * eps) == pytest.approx(float(g0 @ v.ravel()), rel=1e-6)
    # permutation equivariance
    perm = rng.permutation(n)
    s.bind_registration(q0[perm], target[perm], 5e5, T)
    loss_p, g_p = s.objective(x0[perm])
    assert loss_p == pytest.approx(loss0, rel=1e-12)
    assert rel_inf(g_p.reshape(n, 3), g0.reshape(n, 3)[perm]) <= 1e-10


def test_full_size_fp32_tracks_fp64(hs, full_case):
    """fp32 at N = 20 000 against the device's own fp64 result at the paper's initial point (the comparison with
    the CPU oracle at this exact configuration is test_headline_config_full_gradient_vs_cpu_oracle)."""
    n, T, q0, target, p_true, x0 = full_case
    s64, s32 = hs(n, 3, "f64", max_t=T), hs(n, 3, "f32", max_t=T)
    s64.bind_registration(q0, target, 5e5, T)
    s32.bind_registration(q0, target, 5e5, T)
    l64, g64 = s64.objective(x0)
    l32, g32 = s32.objective(x0)
    assert l32 == pytest.approx(l64, rel=1e-5)
    assert s32.last_kinetic == pytest.approx(s64.last_kinetic, rel=1e-5)
    assert rel_inf(g32, g64) <= 1e-5


# ---- the optimiser end to end (BASELINE.json configs[0]) ----------------------------------------------------
def test_small_registration_matches_reference_golden(golden_optimiser):
    """The reference's own register run (oracle/_ref, committed fixture): 96 landmarks, 12 iterations."""
    from paper_1907_04839_b200 import ShootingConfig, register_landmarks

    g = golden_optimiser
    sigma, lam, T, iters = g["reg_meta_sigma_lambda_T_iters"]
    for prec, tol_mm in (("f64", 1e-6), ("f32", 5e-3)):
        cfg = ShootingConfig(sigma=float(sigma), timesteps=int(T), lam=float(lam), max_iter=int(iters), precision=prec)
        r = register_landmarks(g["reg_q0"], g["reg_target"], cfg)
        want_loss, want_init, want_evals, want_iters, _ = g[f"reg_{prec}_summary"]
        assert r.initial_loss == pytest.approx(want_init, rel=TOL[prec])
        assert np.abs(r.warped - g[f"reg_{prec}_warped"]).max() <= tol_mm
        if prec == "f64":
            assert (r.evaluations, r.iterations) == (int(want_evals), int(want_iters))
            assert r.final_loss == pytest.approx(want_loss, rel=1e-7)
            assert np.allclose(r.hist_loss, g["reg_f64_hist_loss"], rtol=1e-7)


def test_hundred_iteration_registration_n1000(oracle, reference):
    """configs[0]: N = 1000, T = 10, 100 L-BFGS iterations; the reference CPU path runs it too.
    Final matched landmarks within 1e-6 mm in fp64."""
    from paper_1907_04839_b200 import ShootingConfig, make_synthetic_pair, register_landmarks

    n, T, lam = 1000, 10, 5e5
    q0, target, _ = make_synthetic_pair(n, SIGMA, T)
    cfg = ShootingConfig(sigma=SIGMA, timesteps=T, lam=lam, max_iter=100, precision="f64")
    got = register_landmarks(q0, target, cfg)
    want = reference.register("f64", q0, target, SIGMA, lam, T, 100)
    assert got.initial_loss == pytest.approx(want["initial_loss"], rel=1e-10)
    assert np.abs(got.warped - want["warped"]).max() <= 1e-6
    assert got.final_loss == pytest.approx(want["loss"], rel=1e-6)
    assert got.avg_after < 1e-2 * got.avg_before
    # the registration metrics come from the device (lms_registration_metrics): bit-identical to the reference's
    # average_dist / max_dist loops (landmarks.cpp:164-179) on the same double sets
    assert (got.avg_before, got.max_before) == oracle.landmark_distances(q0, target)
    assert (got.avg_after, got.max_after) == oracle.landmark_distances(got.warped, target)
    cfg32 = ShootingConfig(sigma=SIGMA, timesteps=T, lam=lam, max_iter=100, precision="f32")
    got32 = register_landmarks(q0, target, cfg32)
    assert np.abs(got32.warped - want["warped"]).max() <= 5e-3


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("n,dim", [(1, 3), (257, 2), (5000, 3)])
def test_registration_metrics_on_device(hs, oracle, prec, n, dim):
    """avg / max landmark distance before and after (registration.cpp:39-40,95-96) from the device against the
    restated landmarks.cpp:164-179 loops: bitwise, both for the bound double sets and for q(1) widened from the
    working precision; and the state errors."""
    from paper_1907_04839_b200 import HamiltonianSystem, _lib
    from paper_1907_04839_b200.errors import StateError

    q, p, target, *_ = synth_case(n, dim, 77 + n, spread=7.0 * max(1.0, (n / 500.0) ** (1.0 / dim)))
    s = HamiltonianSystem(SIGMA, n, dim, prec, max_timesteps=4)
    out = np.zeros(4)
    dp = out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    with pytest.raises(StateError):
        _lib.check(s.lib.lms_registration_metrics(s.handle, dp), s.handle)  # nothing bound
    s.bind_registration(q, target, 25.0, 4)
    s.objective(np.ascontiguousarray(p.ravel()))
    _lib.check(s.lib.lms_registration_metrics(s.handle, dp), s.handle)
    assert tuple(out[:2]) == oracle.landmark_distances(q, target)
    assert tuple(out[2:]) == oracle.landmark_distances(s.final_q(), target)
    s.close()


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("n", [700, 6000, 9000])
def test_host_and_device_buffer_calls_agree(hs, prec, n):
    """lms_objective_eval (host buffers; the persistent kernel reads / writes them in place through mapped pinned
    memory) and lms_objective_eval_device (x / grad in HBM) are the same evaluation: bitwise equal loss, H, mismatch
    and gradient, in either order, for persistent-size (one and two adjoint windows) and tiled-size problems; a non-finite x is DivergedError(0)
    through both."""
    import torch

    from paper_1907_04839_b200 import DivergedError

    q, p, target, *_ = synth_case(n, 3, 900 + n, spread=7.0 * max(1.0, (n / 500.0) ** (1.0 / 3)))
    s = hs(n, 3, prec, max_t=6)
    s.bind_registration(q, target, 40.0, 6)
    x = np.ascontiguousarray(p.ravel())
    xd = torch.from_numpy(x).cuda()
    gd = torch.empty_like(xd)
    loss_h, grad_h = s.objective(x)
    kin_h, mm_h = s.last_kinetic, s.last_mismatch
    loss_d, kin_d, mm_d = s.objective_ptrs(xd.data_ptr(), gd.data_ptr(), device=True)
    assert (loss_d, kin_d, mm_d) == (loss_h, kin_h, mm_h)
    assert np.array_equal(gd.cpu().numpy(), grad_h)
    loss_h2, grad_h2 = s.objective(x)  # and back: nothing of the device call leaks into the host call
    assert loss_h2 == loss_h and np.array_equal(grad_h2, grad_h)
    bad = x.copy()
    bad[5] = np.inf
    with pytest.raises(DivergedError) as e:
        s.objective(bad)
    assert e.value.timestep == 0
    with pytest.raises(DivergedError) as e:
        s.objective_ptrs(torch.from_numpy(bad).cuda().data_ptr(), gd.data_ptr(), device=True)
    assert e.value.timestep == 0
    loss_h3, _ = s.objective(x)  # the handle recovers
    assert loss_h3 == loss_h


def test_reference_minimize_drives_cuda_objective_through_cpp_adapter():
    """Drop-in check: the reference's UNMODIFIED minimize (lbfgs.cpp compiled in place into
    oracle/_ref/libref_cuda_driver.so) calls the CUDA objective through include/lmshoot_b200/objective.hpp.
    Same deterministic objective, two drivers (the reference's and the library's own): identical iterates."""
    import ctypes
    import os

    from paper_1907_04839_b200 import ShootingConfig, register_landmarks

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                        "libref_cuda_driver.so")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref/libref_cuda_driver.so not built (needs /root/reference at build time)")
    lib = ctypes.CDLL(path)

    class Out(ctypes.Structure):
        _fields_ = [("loss", ctypes.c_double), ("initial_loss", ctypes.c_double), ("evaluations", ctypes.c_int),
                    ("iterations", ctypes.c_int), ("reason", ctypes.c_int), ("status", ctypes.c_int),
                    ("diverged_step", ctypes.c_int)]

    dp = ctypes.POINTER(ctypes.c_double)
    lib.ref_cuda_register.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_size_t, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_double, dp, dp, dp, dp,
                                      ctypes.POINTER(Out), dp]
    n, T, lam, iters = 700, 8, 1e4, 25
    rng = np.random.default_rng(12)
    q0 = rng.uniform(-12, 12, (n, 3))
    target = q0 + 0.5 * rng.normal(size=(n, 3))
    for prec in ("f64", "f32"):
        mom, warped, hist = np.empty((n, 3)), np.empty((n, 3)), np.zeros(iters)
        out = Out()
        rc = lib.ref_cuda_register(int(prec == "f32"), 3, n, SIGMA, lam, T, iters, 1e-6, q0.ctypes.data_as(dp),
                                   target.ctypes.data_as(dp), mom.ctypes.data_as(dp), warped.ctypes.data_as(dp),
                                   ctypes.byref(out), hist.ctypes.data_as(dp))
        assert rc == 0
        mine = register_landmarks(q0, target, ShootingConfig(sigma=SIGMA, timesteps=T, lam=lam, max_iter=iters,
                                                             precision=prec))
        assert (out.evaluations, out.iterations) == (mine.evaluations, mine.iterations)
        assert out.loss == mine.final_loss and out.initial_loss == mine.initial_loss
        assert np.array_equal(mom, mine.momenta) and np.array_equal(warped, mine.warped)
        assert np.array_equal(hist[: out.iterations], mine.hist_loss)
        assert mine.final_loss < 0.5 * mine.initial_loss
    # the adapter rethrows the reference's DivergedError with its timestep
    bad = q0.copy()
    bad[0, 0] = np.inf
    out = Out()
    rc = lib.ref_cuda_register(0, 3, n, SIGMA, lam, T, 3, 1e-6, bad.ctypes.data_as(dp), target.ctypes.data_as(dp),
                               mom.ctypes.data_as(dp), warped.ctypes.data_as(dp), ctypes.byref(out),
                               hist.ctypes.data_as(dp))
    assert rc == 2 and out.diverged_step == 0


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_nccl_path_single_rank(hs, monkeypatch, prec):
    """The row-partitioned code path (NCCL communicator, per-step in-place all-gathers, no CUDA graph) with a
    world of one rank on the single GPU: must give the same bits as the plain path."""
    from paper_1907_04839_b200 import HamiltonianSystem, comm_unique_id

    n, T = 1500, 6
    q, p, target, *_ = synth_case(n, 3, 77, spread=9.0)
    plain = hs(n, 3, prec, tiled_only=True)  # the partitioned ranks run the tiled kernels: compare like with like
    plain.bind_registration(q, target, 100.0, T)
    want = plain.objective(p)
    monkeypatch.setenv("LMS_FORCE_NCCL", "1")
    s = HamiltonianSystem(SIGMA, n, 3, prec, max_timesteps=T)
    s.comm_init(comm_unique_id(), 0, 1)
    s.bind_registration(q, target, 100.0, T)
    got = s.objective(p)
    assert got[0] == want[0] and np.array_equal(got[1], want[1])
    assert np.array_equal(s.final_q(), plain.final_q())
    s.close()


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_device_gaussian_kernel_values(hs, prec):
    """gaussian_kernel known answers and the accuracy of the device exp over its whole range,
    read back through velocities_at_step with one landmark of unit momentum: v = K(|x - q|^2) * (1, 0, 0)."""
    s = hs(1, 3, prec)
    q, p = np.zeros((1, 3)), np.array([[1.0, 0.0, 0.0]])
    r = np.concatenate([[0.0, np.sqrt(2 * SIGMA**2 * np.log(2.0)), 1.5], np.linspace(0.0, 60.0, 4001)])
    pts = np.zeros((r.size, 3))
    pts[:, 1] = r
    k = s.velocities_at_step(q, p, pts)[:, 0]
    t = np.float32 if prec == "f32" else np.float64
    r2 = (pts.astype(t)[:, 1] ** 2).astype(np.float64)
    want = np.exp(r2 * (-0.5 / SIGMA**2))
    assert k[0] == 1.0
    assert k[1] == pytest.approx(0.5, rel=4e-7 if prec == "f32" else 1e-15)
    assert k[2] == pytest.approx(0.606531, abs=5e-7)
    # relative accuracy where K is normal; exact zero (flush) once exp underflows
    if prec == "f64":
        live = want > 1e-300
        assert np.abs(k[live] / want[live] - 1).max() < 5e-13  # |arg| up to 690: the rounded scale costs ~|arg| ulp
        near = want > 1e-12
        assert np.abs(k[near] / want[near] - 1).max() < 2e-14
        assert (k[want < 1e-320] == 0).all()
    else:
        live = want > 1e-30
        assert np.abs(k[live] / want[live] - 1).max() < 2e-5
        near = want > 1e-6
        assert np.abs(k[near] / want[near] - 1).max() < 2e-6
    assert (np.diff(k[3:]) <= 0).all()  # monotone in distance


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("sigma,spread,lam,T", [(0.1, 2.0, 10.0, 5), (100.0, 5.0, 10.0, 5), (1.5, 1e4, 1.0, 3),
                                               (1.5, 0.0, 10.0, 4), (3.0, 4.0, 0.0, 1), (1.5, 6.0, 5e5, 40)])
def test_parameter_extremes(oracle, prec, sigma, spread, lam, T):
    """Kernel widths from 'no pair interacts' to 'every pair has K = 1', landmarks 1e4 mm apart (exp underflows for
    almost every pair), coincident landmarks (spread 0: r = 0 for i != j), lambda = 0, T = 1 and the reference's
    default T = 40."""
    from paper_1907_04839_b200 import HamiltonianSystem

    n = 300
    rng = np.random.default_rng(int(sigma * 10) + T)
    q = rng.uniform(-spread, spread, (n, 3)) if spread > 0 else np.zeros((n, 3))
    p = 0.05 * rng.normal(size=(n, 3)) if sigma > 10 or spread == 0 else 0.75 * rng.normal(size=(n, 3))
    target = q + 0.5 * rng.normal(size=(n, 3))
    s = HamiltonianSystem(sigma, n, 3, prec, max_timesteps=T)
    r = s.compute_gradient(q, p, target, lam, T)
    loss, kin, mm, grad = oracle.compute_gradient(prec, q, p, target, sigma, lam, T)
    tol = TOL[prec] * (10 if prec == "f32" and (sigma > 10 or spread == 0) else 1)  # N coherent terms per row in fp32
    assert r.loss == pytest.approx(loss, rel=tol) and r.kinetic == pytest.approx(kin, rel=tol, abs=1e-300)
    assert r.mismatch == pytest.approx(mm, rel=tol)
    assert rel_inf(r.grad, grad) <= tol
    s.close()


def test_large_n_row_subset_fp32(oracle):
    """N = 200 000 (BASELINE configs[2] size on one GPU): 48 rows of one forward and one adjoint launch against the
    oracle's identical per-row sums; run-to-run bitwise determinism at that size."""
    from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals

    n = 200000
    q = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
    p = (0.75 * rng_normals(3, n * 3)).reshape(n, 3)
    alpha = rng_normals(4, n * 3).reshape(n, 3)
    beta = rng_normals(5, n * 3).reshape(n, 3)
    rows = np.unique(np.concatenate([[0, 511, 512, n - 1], np.random.default_rng(1).integers(0, n, 44)]))
    s = HamiltonianSystem(SIGMA, n, 3, "f32", max_timesteps=1)
    hq, hp = s.derivatives(q, p)
    ohq, ohp = oracle.pair_rows("f32", q, p, rows, SIGMA)
    assert np.abs(hq[rows] - ohq).max() <= 1e-5 * np.abs(hq).max()
    assert np.abs(hp[rows] - ohp).max() <= 1e-5 * np.abs(hp).max()
    da, db = s.adjoint_step(q, p, alpha, beta)
    oda, odb = oracle.pair_rows("f32", q, p, rows, SIGMA, alpha, beta)
    assert np.abs(da[rows] - oda).max() <= 1e-5 * np.abs(da).max()
    assert np.abs(db[rows] - odb).max() <= 1e-5 * np.abs(db).max()
    again = s.derivatives(q, p)
    assert np.array_equal(again[0], hq) and np.array_equal(again[1], hp)
    s.close()


def test_configs2_full_size_properties_fp32(oracle):
    """BASELINE configs[2] on one GPU -- N = 200 000, T = 20, fp32, the evaluation bench.py times at that size -- through
    the properties that do not need an O(N^2) CPU run: momentum conservation of the Euler flow over
    all 21 snapshots, H = 1/2 sum p.hp and sum_i hq_i = 0, "at the true momenta of a reachable target the gradient is
    hp(q0, p) and the loss is H" (the fp64 flow of the same handle family builds the target), a directional finite
    difference of the loss at the paper's initial point, and 40 rows of the final positions against the oracle's own
    per-row sums for the first Euler step."""
    from paper_1907_04839_b200 import HamiltonianSystem, make_synthetic_pair

    n, T, lam = 200000, 20, 5e5
    q0, target, p_true = make_synthetic_pair(n, SIGMA, T, density_scaled=True)
    s = HamiltonianSystem(SIGMA, n, 3, "f32", max_timesteps=T)
    tq, tp = s.integrate_forward(q0, p_true, T)
    # fp32 flow against the fp64 flow that made the target
    assert rel_inf(tq[-1], target) <= 1e-5
    drift = np.abs(tp.sum(axis=1) - p_true.sum(axis=0)).max()
    assert drift <= 1e-5 * np.linalg.norm(p_true, axis=1).sum() / np.sqrt(n)  # N random roundings of ~6e-8 |p| each
    # first Euler step of 40 rows against the oracle's per-row sums: q1 = q0 + dt hp, p1 = p0 - dt hq
    rows = np.unique(np.concatenate([[0, 511, 512, n - 1], np.random.default_rng(2).integers(0, n, 36)]))
    ohq, ohp = oracle.pair_rows("f32", q0, p_true, rows, SIGMA)
    dt = 1.0 / T
    assert np.abs(tq[1][rows] - (q0[rows] + dt * ohp)).max() <= 1e-5 * np.abs(tq[1]).max()
    assert np.abs(tp[1][rows] - (p_true[rows] - dt * ohq)).max() <= 1e-5 * np.abs(tp[1]).max()
    del tq, tp
    h = s.hamiltonian(q0, p_true)
    hq, hp = s.derivatives(q0, p_true)
    assert 0.5 * float((p_true * hp).sum()) == pytest.approx(h, rel=1e-6)
    assert np.abs(hq.sum(axis=0)).max() <= 1e-5 * np.abs(hq).sum() / np.sqrt(n)
    # the fp32 flow misses the fp64 target by rounding only: loss = H + lambda * (rounding)^2, grad = hp + 2 lambda * rounding
    s.bind_registration(q0, target, lam, T)
    loss, grad = s.objective(p_true)
    assert s.last_kinetic == pytest.approx(h, rel=1e-6)
    assert s.last_mismatch <= n * 3 * (1e-5 * np.abs(target).max()) ** 2
    assert s.last_eval_kernel_launches() == 2 * T + 2
    # finite difference of the loss along its own gradient at the paper's initial point (registration.cpp:47-52).  The
    # fp32 loss (~1e11 here) carries ~1e-7 of relative rounding noise, which swamps the slope along a random unit vector
    # (~|g| / sqrt(3N)); along g / |g| the slope is |g| itself and a central difference resolves it to about a per cent.
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    loss0, g0 = s.objective(x0)
    again, g1 = s.objective(x0)
    assert again == loss0 and np.array_equal(g0, g1)  # bitwise run to run at this size too
    gnorm = float(np.linalg.norm(g0))
    v = g0 / gnorm
    eps = 3e-2
    hi, _ = s.objective(x0 + eps * v)
    lo, _ = s.objective(x0 - eps * v)
    assert hi > loss0 > lo
    assert (hi - lo) / (2 * eps) == pytest.approx(gnorm, rel=2e-2)
    s.close()


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("world,n", [(2, 1500), (3, 2600), (4, 700), (2, 20000)])
def test_row_partition_loopback(hs, oracle, prec, world, n):
    """The row-partitioned evaluation with world > 1 on ONE GPU: every rank is a handle driven by its own host
    thread, the per-step exchange goes through the loopback transport (same schedule and slice layout as the
    NCCL path).  Every rank must end with the same full gradient, equal to the unpartitioned result."""
    import threading

    from paper_1907_04839_b200 import HamiltonianSystem, LocalGroup

    T, lam = 5, 100.0
    q, p, target, *_ = synth_case(n, 3, 500 + n + world, spread=10.0 if n < 10000 else 60.0)
    plain = hs(n, 3, prec, tiled_only=True)  # the partitioned ranks run the tiled kernels: compare like with like
    plain.bind_registration(q, target, lam, T)
    want_loss, want_grad = plain.objective(p)
    want_q = plain.final_q()
    group = LocalGroup(world)
    ranks = [HamiltonianSystem(SIGMA, n, 3, prec, max_timesteps=T) for _ in range(world)]
    results, errors = [None] * world, []

    def run(r):
        try:
            s = ranks[r]
            s.join_local_group(group, r)
            s.bind_registration(q, target, lam, T)
            first = s.objective(p)
            second = s.objective(p)  # a second evaluation reuses the buffers the first one exchanged through
            results[r] = (first, second, s.last_kinetic, s.last_mismatch, s.final_q())
        except Exception as e:  # pragma: no cover
            errors.append(e)

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    tol = 1e-12 if prec == "f64" else 2e-6
    for r in range(world):
        (loss, grad), (loss2, grad2), kin, mm, fq = results[r]
        assert loss == results[0][0][0] and np.array_equal(grad, results[0][0][1])  # identical on every rank
        assert loss2 == loss and np.array_equal(grad2, grad)                          # and run to run
        assert loss == pytest.approx(want_loss, rel=tol) and rel_inf(grad, want_grad) <= tol
        assert kin == pytest.approx(plain.last_kinetic, rel=tol) and mm == pytest.approx(plain.last_mismatch, rel=tol)
        assert rel_inf(fq, want_q) <= tol
    if n <= 3000:
        o = oracle.compute_gradient(prec, q, p, target, SIGMA, lam, T)
        assert rel_inf(results[0][0][1].reshape(n, 3), o[3]) <= TOL[prec]
    for s in ranks:
        s.close()
    group.close()


@pytest.mark.parametrize("transport", ["loopback", "p2p"])
def test_row_partition_ranks_agree_on_divergence(hs, transport):
    """A state that turns non-finite in rows owned by ONE rank: every rank must raise DivergedError with the step
    the unpartitioned evaluation reports (shooting.hpp:210-211) -- also when that is the last step, where the other
    ranks never see the non-finite values in a gathered state.  (The ranks exchange their divergence words with
    the scalar partials; without that they would disagree and the optimisers would part ways mid-collective.)"""
    import threading

    from paper_1907_04839_b200 import DivergedError, HamiltonianSystem, LocalGroup

    n, world, prec = 1500, 2, "f32"
    q, p, target, *_ = synth_case(n, 3, 77, spread=10.0)
    q = q * 1e18
    target = q.copy()
    huge = p.copy()
    huge[3, 0] = 1e30  # row 3 belongs to rank 0
    plain = hs(n, 3, prec, tiled_only=True)  # the partitioned ranks run the tiled kernels: compare like with like
    plain.bind_registration(q, target, 1.0, 6)
    with pytest.raises(DivergedError) as want:
        plain.objective(huge)
    t_star = want.value.timestep
    assert t_star >= 1
    for T in (6, t_star):  # blow-up part-way, and at the very last step
        plain.bind_registration(q, target, 1.0, T)
        with pytest.raises(DivergedError) as want:
            plain.objective(huge * (T / 6.0))  # same per-step increments
        group = LocalGroup(world) if transport == "loopback" else None
        ranks = [HamiltonianSystem(SIGMA, n, 3, prec, max_timesteps=6) for _ in range(world)]
        if transport == "p2p":
            blobs = [s.p2p_export(r, world) for r, s in enumerate(ranks)]
            for s in ranks:
                s.p2p_connect(blobs)
        steps, errors = [None] * world, []
        meet = threading.Barrier(world)

        def run(r):
            try:
                s = ranks[r]
                if transport == "loopback":
                    s.join_local_group(group, r)
                s.bind_registration(q, target, 1.0, T)
                meet.wait(timeout=120)
                try:
                    s.objective(huge * (T / 6.0))
                    steps[r] = -1
                except DivergedError as e:
                    steps[r] = e.timestep
                # the handles stay usable and in step with each other
                loss, _ = s.objective(p * 1e-3)
                assert np.isfinite(loss)
            except Exception as e:  # pragma: no cover
                errors.append(e)
                meet.abort()

        threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
        assert not errors, errors
        assert steps == [want.value.timestep] * world, (T, steps, want.value.timestep)
        for s in ranks:
            s.close()
        if group is not None:
            group.close()


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_device_resident_lbfgs_matches_host_driver(prec):
    """lms_register_device (optimiser vectors in HBM) against lms_register (host vectors,
    the reference's summation order): same decision logic, sums differ by rounding only."""
    from paper_1907_04839_b200 import DivergedError, ShootingConfig, register_landmarks

    n, T, lam, iters = 1500, 8, 1e4, 30
    rng = np.random.default_rng(31)
    q0 = rng.uniform(-15, 15, (n, 3))
    target = q0 + 0.5 * rng.normal(size=(n, 3))
    cfg = ShootingConfig(sigma=SIGMA, timesteps=T, lam=lam, max_iter=iters, precision=prec)
    host = register_landmarks(q0, target, cfg)
    dev = register_landmarks(q0, target, cfg, device_vectors=True)
    assert dev.initial_loss == host.initial_loss
    assert dev.reason == host.reason
    if prec == "f64":
        assert (dev.iterations, dev.evaluations) == (host.iterations, host.evaluations)
        assert dev.final_loss == pytest.approx(host.final_loss, rel=1e-8)
        assert np.abs(dev.warped - host.warped).max() <= 1e-6
        assert np.allclose(dev.hist_loss, host.hist_loss, rtol=1e-8)
    else:
        assert dev.final_loss == pytest.approx(host.final_loss, rel=0.05)
        assert np.abs(dev.warped - host.warped).max() <= 5e-3
    assert dev.final_loss < 0.5 * dev.initial_loss
    bad = q0.copy()
    bad[5, 0] = np.nan
    with pytest.raises(DivergedError) as e:
        register_landmarks(bad, target, cfg, device_vectors=True)
    assert e.value.timestep == 0


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_headline_config_full_gradient_vs_cpu_oracle(hs, oracle, full_case, prec):
    """BASELINE configs[1] itself -- N = 20 000, T = 10, lambda = 5e5, every row, at the paper's initial point
    x0 = (target - q0)/T (registration.cpp:47-52) -- against the CPU oracle's compute_gradient
    (shooting.hpp:277-315; (2T+2) N^2 = 8.8e9 pair evaluations, ~10 s on 16 host threads): loss, H, mismatch and
    dL/dp0 within 1e-5 (fp32) / 1e-10 (fp64), the tolerances of BASELINE.json's north_star.  Both the call the
    bench times (bind + objective, evaluation graph) and lms_compute_gradient are checked."""
    n, T, q0, target, p_true, x0 = full_case
    lam = 5e5
    loss, kin, mm, grad = oracle.compute_gradient(prec, q0, x0, target, SIGMA, lam, T)
    s = hs(n, 3, prec, max_t=T)
    s.bind_registration(q0, target, lam, T)
    got_loss, got_grad = s.objective(x0)
    tol = TOL[prec]
    assert got_loss == pytest.approx(loss, rel=tol)
    assert s.last_kinetic == pytest.approx(kin, rel=tol)
    assert s.last_mismatch == pytest.approx(mm, rel=tol)
    assert rel_inf(got_grad.reshape(n, 3), grad) <= tol
    r = s.compute_gradient(q0, x0, target, lam, T)
    assert r.loss == got_loss and np.array_equal(r.grad.ravel(), got_grad)  # same graph, same bits
    # q(1) of that evaluation against the oracle's forward flow
    otq, _ = oracle.integrate_forward(prec, q0, x0, SIGMA, T)
    assert rel_inf(s.final_q(), otq[-1]) <= tol


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_full_size_full_gradient_second_point(hs, oracle, full_case, prec):
    """N = 20 000, every row, at a second evaluation point and step count (T = 2, momenta rescaled to land near
    the target) against the CPU oracle."""
    n, _, q0, target, p_true, x0 = full_case
    T, lam = 2, 5e5
    s = hs(n, 3, prec, max_t=10)
    r = s.compute_gradient(q0, x0 * 5.0, target, lam, T)  # x0 was built for T = 10: rescale to land near the target
    loss, kin, mm, grad = oracle.compute_gradient(prec, q0, x0 * 5.0, target, SIGMA, lam, T)
    assert r.loss == pytest.approx(loss, rel=TOL[prec])
    assert r.kinetic == pytest.approx(kin, rel=TOL[prec])
    assert r.mismatch == pytest.approx(mm, rel=TOL[prec])
    assert rel_inf(r.grad, grad) <= TOL[prec]


# ---- SPEC.md acceptance runs on the device path (long trajectories) ----------------------------------------
def test_momentum_conservation_long_trajectory_on_device(oracle):
    """SPEC.md acceptance 3 (:222,559): N = 100, T = 100 in fp64 -- the total momentum sum_i p_i(t) drifts by at most
    1e-10 * sum_i |p_i(0)| over the whole trajectory; and the device trajectory equals the oracle's to 1e-10."""
    from paper_1907_04839_b200 import HamiltonianSystem

    n, T = 100, 100
    q, p, *_ = synth_case(n, 3, 2024, spread=5.0)
    s = HamiltonianSystem(SIGMA, n, 3, "f64", max_timesteps=T)
    tq, tp = s.integrate_forward(q, p, T)
    s.close()
    drift = np.abs(tp.sum(axis=1) - p.sum(axis=0)).max()
    assert drift <= 1e-10 * np.linalg.norm(p, axis=1).sum()
    otq, otp = oracle.integrate_forward("f64", q, p, SIGMA, T)
    assert rel_inf(tq, otq) <= 1e-10 and rel_inf(tp, otp) <= 1e-10


def test_hamiltonian_drift_is_first_order_on_device(oracle):
    """SPEC.md acceptance 2 (:223,558): explicit Euler conserves H to first order in dt -- the drift
    |H(q(1),p(1)) - H(q0,p0)| at T = 400 is about half the drift at T = 200 (ratio in [0.4, 0.6]); both runs go
    through the device handle (trajectory capacity 400) and match the oracle's end states."""
    from paper_1907_04839_b200 import HamiltonianSystem

    n = 200
    q, p, *_ = synth_case(n, 3, 2025, spread=4.0)
    s = HamiltonianSystem(SIGMA, n, 3, "f64", max_timesteps=400)
    h0 = s.hamiltonian(q, p)
    drifts = []
    for T in (200, 400):
        tq, tp = s.integrate_forward(q, p, T)
        drifts.append(abs(s.hamiltonian(tq[-1], tp[-1]) - h0))
        otq, otp = oracle.integrate_forward("f64", q, p, SIGMA, T)
        assert rel_inf(tq[-1], otq[-1]) <= 1e-10 and rel_inf(tp[-1], otp[-1]) <= 1e-10
    # a gradient through all 400 stored snapshots: the adjoint sweep at the handle's capacity
    target = tq[-1] + 0.01
    r = s.compute_gradient(q, p, target, 10.0, 400)
    o = oracle.compute_gradient("f64", q, p, target, SIGMA, 10.0, 400)
    assert r.loss == pytest.approx(o[0], rel=1e-10) and rel_inf(r.grad, o[3]) <= 1e-10
    s.close()
    assert drifts[0] > 0 and 0.4 <= drifts[1] / drifts[0] <= 0.6, drifts


def test_result_document_of_a_registration_reproduces_the_warp(tmp_path):
    """register_landmarks -> schema-v1 result document -> load -> re-integrating the stored momenta gives the stored
    warped landmarks back (what warp_with_result relies on, registration.cpp:102-124,159-168)."""
    from paper_1907_04839_b200 import (HamiltonianSystem, ShootingConfig, load_result, register_landmarks,
                                       result_document_from, save_result)

    n, T = 400, 6
    rng = np.random.default_rng(8)
    q0 = rng.uniform(-8, 8, (n, 3))
    target = q0 + 0.4 * rng.normal(size=(n, 3))
    cfg = ShootingConfig(sigma=SIGMA, timesteps=T, lam=1e4, max_iter=15, precision="f64")
    reg = register_landmarks(q0, target, cfg)
    path = tmp_path / "result.json"
    save_result(result_document_from(reg, q0, target, cfg), path)
    doc = load_result(path)
    assert np.array_equal(doc.momenta.reshape(n, 3), reg.momenta) and np.array_equal(doc.warped, reg.warped)
    assert doc.config == cfg and doc.final_loss == reg.final_loss and doc.avg_after == reg.avg_after
    s = HamiltonianSystem(doc.config.sigma, n, 3, doc.config.precision, max_timesteps=doc.config.timesteps)
    tq, _ = s.integrate_forward(doc.template, doc.momenta.reshape(n, 3), doc.config.timesteps)
    s.close()
    # same inputs through the per-function path (tiled kernels; the registration itself ran the persistent kernel):
    # equal to rounding
    assert rel_inf(tq[-1], doc.warped) <= 1e-12
    assert doc.avg_after < doc.avg_before


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("world,n", [(2, 1500), (3, 2600), (4, 700), (2, 20000)])
def test_row_partition_peer_push_in_process(hs, oracle, prec, world, n):
    """The row partition over the peer-push transport (lms_p2p_*), world > 1 on ONE GPU: every rank is a handle
    with its own stream and host thread; the kernels' epilogues store each updated row into every rank's arena and
    only arrival flags are exchanged in stream order.  Same acceptance as the loopback test."""
    import threading

    from paper_1907_04839_b200 import HamiltonianSystem

    T, lam = 5, 100.0
    q, p, target, *_ = synth_case(n, 3, 900 + n + world, spread=10.0 if n < 10000 else 60.0)
    plain = hs(n, 3, prec, tiled_only=True)  # the partitioned ranks run the tiled kernels: compare like with like
    plain.bind_registration(q, target, lam, T)
    want_loss, want_grad = plain.objective(p)
    want_q = plain.final_q()
    ranks = [HamiltonianSystem(SIGMA, n, 3, prec, max_timesteps=T) for _ in range(world)]
    blobs, results, errors = [None] * world, [None] * world, []
    meet = threading.Barrier(world)

    def run(r):
        try:
            s = ranks[r]
            blobs[r] = s.p2p_export(r, world)
            meet.wait(timeout=120)  # the application's all-gather of the blobs
            s.p2p_connect(blobs)
            s.bind_registration(q, target, lam, T)
            meet.wait(timeout=120)
            evals = [s.objective(p) for _ in range(3)]  # later evaluations reuse the arenas the first one wrote
            results[r] = (evals, s.last_kinetic, s.last_mismatch, s.final_q())
        except Exception as e:  # pragma: no cover
            errors.append(e)
            meet.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    tol = 1e-12 if prec == "f64" else 2e-6
    for r in range(world):
        evals, kin, mm, fq = results[r]
        loss, grad = evals[0]
        assert loss == results[0][0][0][0] and np.array_equal(grad, results[0][0][0][1])  # identical on every rank
        for again in evals[1:]:
            assert again[0] == loss and np.array_equal(again[1], grad)                      # and run to run
        assert loss == pytest.approx(want_loss, rel=tol) and rel_inf(grad, want_grad) <= tol
        assert kin == pytest.approx(plain.last_kinetic, rel=tol) and mm == pytest.approx(plain.last_mismatch, rel=tol)
        assert rel_inf(fq, want_q) <= tol
    for s in ranks:
        s.close()


def _peer_push_worker(rank, world, prec, n, T, lam, seed, to_parent, from_parent):
    import numpy as np

    from paper_1907_04839_b200 import HamiltonianSystem

    try:
        rng = np.random.default_rng(seed)
        q = rng.uniform(-10, 10, (n, 3))
        p = 0.75 * rng.normal(size=(n, 3))
        target = q + 0.5 * rng.normal(size=(n, 3))
        s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
        to_parent.put((rank, "blob", s.p2p_export(rank, world)))
        blobs = from_parent.get(timeout=120)
        s.p2p_connect(blobs)
        s.bind_registration(q, target, lam, T)
        to_parent.put((rank, "bound", None))
        from_parent.get(timeout=120)
        first = s.objective(p)
        second = s.objective(p)
        to_parent.put((rank, "done", (first, second, s.final_q())))
        from_parent.get(timeout=120)  # keep the arena mapped until every rank has finished
        s.close()
    except Exception as e:  # pragma: no cover
        to_parent.put((rank, "error", repr(e)))


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_row_partition_peer_push_across_processes(hs, prec):
    """The production shape of the peer-push transport: one PROCESS per rank, arenas mapped through CUDA IPC
    (cudaIpcOpenMemHandle), flags through stream memory operations on the mapped memory.  Both ranks share the
    one GPU of this machine, which exercises everything but the NVLink wires."""
    import multiprocessing as mp

    world, n, T, lam, seed = 2, 1800, 4, 100.0, 77
    ctx = mp.get_context("spawn")
    to_parent = ctx.Queue()
    inboxes = [ctx.Queue() for _ in range(world)]
    procs = [ctx.Process(target=_peer_push_worker, args=(r, world, prec, n, T, lam, seed, to_parent, inboxes[r]))
             for r in range(world)]
    for pr in procs:
        pr.start()

    def collect(tag):
        got = {}
        while len(got) < world:
            rank, kind, payload = to_parent.get(timeout=240)
            assert kind != "error", payload
            assert kind == tag, (kind, tag)
            got[rank] = payload
        return [got[r] for r in range(world)]

    try:
        blobs = collect("blob")
        for box in inboxes:
            box.put(blobs)
        collect("bound")
        for box in inboxes:
            box.put("go")
        results = collect("done")
        for box in inboxes:
            box.put("bye")
    finally:
        for pr in procs:
            pr.join(timeout=60)
            if pr.is_alive():
                pr.kill()
    rng = np.random.default_rng(seed)
    q = rng.uniform(-10, 10, (n, 3))
    p = 0.75 * rng.normal(size=(n, 3))
    target = q + 0.5 * rng.normal(size=(n, 3))
    plain = hs(n, 3, prec, tiled_only=True)  # the partitioned ranks run the tiled kernels: compare like with like
    plain.bind_registration(q, target, lam, T)
    want_loss, want_grad = plain.objective(p)
    tol = 1e-12 if prec == "f64" else 2e-6
    for (first, second, fq) in results:
        assert first[0] == results[0][0][0] and np.array_equal(first[1], results[0][0][1])
        assert second[0] == first[0] and np.array_equal(second[1], first[1])
        assert first[0] == pytest.approx(want_loss, rel=tol) and rel_inf(first[1], want_grad) <= tol
        assert rel_inf(fq, plain.final_q()) <= tol
