"""GPU tests of the population-batch path (lms_batch_*): many independent registrations per launch."""
import numpy as np
import pytest

from conftest import rel_inf

pytestmark = pytest.mark.gpu
SIGMA = 1.5
TOL = {"f64": 1e-10, "f32": 1e-5}


def make_batch(batch, n, seed, dim=3):
    rng = np.random.default_rng(seed)
    q0 = rng.uniform(-7, 7, (batch, n, dim))
    p0 = 0.75 * rng.normal(size=(batch, n, dim))
    target = q0 + 0.5 * rng.normal(size=(batch, n, dim))
    return q0, p0, target


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("batch,n", [(1, 300), (5, 257), (12, 600), (40, 100)])
def test_batched_evaluation_matches_oracle_per_problem(oracle, prec, batch, n):
    from paper_1907_04839_b200 import BatchedRegistrations

    T, lam = 5, 10.0
    q0, p0, target = make_batch(batch, n, 100 + batch)
    br = BatchedRegistrations(SIGMA, n, batch, 3, prec, max_timesteps=T)
    br.bind(q0, target, lam, T)
    scalars, grad, div = br.evaluate(p0)
    finals = br.final_q()
    assert (div == -1).all()
    for b in range(batch):
        loss, kin, mm, g = oracle.compute_gradient(prec, q0[b], p0[b], target[b], SIGMA, lam, T)
        assert scalars[b, 0] == pytest.approx(loss, rel=TOL[prec])
        assert scalars[b, 1] == pytest.approx(kin, rel=TOL[prec])
        assert scalars[b, 2] == pytest.approx(mm, rel=TOL[prec])
        assert rel_inf(grad[b], g) <= TOL[prec]
        assert rel_inf(finals[b], oracle.integrate_forward(prec, q0[b], p0[b], SIGMA, T)[0][-1]) <= TOL[prec]
    # deterministic, and a second evaluation reuses the captured graph
    again = br.evaluate(p0)
    assert np.array_equal(again[0], scalars) and np.array_equal(again[1], grad)
    br.close()


def test_subset_evaluation_and_isolated_divergence(oracle):
    from paper_1907_04839_b200 import BatchedRegistrations

    batch, n, T, lam = 7, 200, 4, 10.0
    q0, p0, target = make_batch(batch, n, 9)
    br = BatchedRegistrations(SIGMA, n, batch, 3, "f64", max_timesteps=T)
    br.bind(q0, target, lam, T)
    full = br.evaluate(p0)
    ids = [5, 1, 3]
    sub = br.evaluate(p0, ids)
    for b in range(batch):
        if b in ids:
            assert np.allclose(sub[0][b], full[0][b], rtol=1e-13) and rel_inf(sub[1][b], full[1][b]) <= 1e-12
        else:
            assert not sub[0][b].any() and not sub[1][b].any()
    bad = p0.copy()
    bad[2, 7, 1] = np.nan
    scalars, grad, div = br.evaluate(bad)
    assert div[2] == 0 and (np.delete(div, 2) == -1).all()  # DivergedError(0) for problem 2 only
    for b in (0, 1, 3, 4, 5, 6):
        assert np.array_equal(scalars[b], full[0][b]) and np.array_equal(grad[b], full[1][b])
    br.close()


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_batched_registrations_match_single_runs(prec):
    from paper_1907_04839_b200 import BatchedRegistrations, LbfgsParams, ShootingConfig, register_landmarks

    batch, n, T, lam, iters = 6, 300, 5, 1e3, 12
    q0, _, target = make_batch(batch, n, 21)
    br = BatchedRegistrations(SIGMA, n, batch, 3, prec, max_timesteps=T)
    br.bind(q0, target, lam, T)
    res = br.register(LbfgsParams(max_iter=iters))
    br.close()
    assert (res.status == 0).all()
    # rounds ~ the longest single run, not the sum over problems: the calls really are coalesced
    assert res.rounds <= res.evaluations.max() + 1 and res.rounds < res.evaluations.sum()
    for b in range(batch):
        one = register_landmarks(q0[b], target[b], ShootingConfig(sigma=SIGMA, timesteps=T, lam=lam, max_iter=iters,
                                                                  precision=prec))
        assert res.initial_loss[b] == pytest.approx(one.initial_loss, rel=TOL[prec])
        if prec == "f64":
            assert res.iterations[b] == one.iterations and res.evaluations[b] == one.evaluations
            assert res.final_loss[b] == pytest.approx(one.final_loss, rel=1e-8)
            assert np.abs(res.warped[b] - one.warped).max() <= 1e-6
        else:
            assert np.abs(res.warped[b] - one.warped).max() <= 5e-3
        assert res.final_loss[b] < res.initial_loss[b]


@pytest.mark.parametrize("groups", [1, 2, 3])
def test_batch_register_in_alternating_groups(groups, monkeypatch):
    """From 32 problems on lms_batch_register evaluates the population in alternating groups (the host L-BFGS
    arithmetic of one group overlaps the device round of the other).  Every problem still runs the unchanged driver
    on its own evaluations: whatever the group count, fp64 results agree with single registrations to rounding and
    the rounds are coalesced per group."""
    from paper_1907_04839_b200 import BatchedRegistrations, LbfgsParams, ShootingConfig, register_landmarks

    monkeypatch.setenv("LMS_BATCH_GROUPS", str(groups))
    batch, n, T, lam, iters = 34, 120, 4, 1e3, 8
    q0, _, target = make_batch(batch, n, 77)
    br = BatchedRegistrations(SIGMA, n, batch, 3, "f64", max_timesteps=T)
    br.bind(q0, target, lam, T)
    res = br.register(LbfgsParams(max_iter=iters))
    br.close()
    assert (res.status == 0).all()
    assert res.rounds <= groups * (res.evaluations.max() + 1) and res.rounds < res.evaluations.sum()
    for b in (0, 11, 16, 17, 33):  # first / last problems of the groups
        one = register_landmarks(q0[b], target[b], ShootingConfig(sigma=SIGMA, timesteps=T, lam=lam, max_iter=iters,
                                                                  precision="f64"))
        assert res.iterations[b] == one.iterations and res.evaluations[b] == one.evaluations
        assert res.final_loss[b] == pytest.approx(one.final_loss, rel=1e-8)
        assert np.abs(res.warped[b] - one.warped).max() <= 1e-6


def test_batch_handle_rejects_single_problem_calls():
    from paper_1907_04839_b200 import BatchedRegistrations, StateError, _lib
    import ctypes

    br = BatchedRegistrations(SIGMA, 50, 3, 3, "f64", max_timesteps=3)
    q = np.zeros((50, 3))
    out = ctypes.c_double()
    dp = ctypes.POINTER(ctypes.c_double)
    rc = br.lib.lms_hamiltonian(br.handle, q.ctypes.data_as(dp), q.ctypes.data_as(dp), ctypes.byref(out))
    with pytest.raises(StateError):
        _lib.check(rc, br.handle)
    assert br.lib.lms_batch_size(br.handle) == 3
    br.close()


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_batched_two_dimensional(oracle, prec):
    from paper_1907_04839_b200 import BatchedRegistrations

    batch, n, T, lam = 4, 310, 6, 25.0
    q0, p0, target = make_batch(batch, n, 33, dim=2)
    br = BatchedRegistrations(SIGMA, n, batch, 2, prec, max_timesteps=T)
    br.bind(q0, target, lam, T)
    scalars, grad, div = br.evaluate(p0)
    for b in range(batch):
        loss, kin, mm, g = oracle.compute_gradient(prec, q0[b], p0[b], target[b], SIGMA, lam, T)
        assert scalars[b, 0] == pytest.approx(loss, rel=TOL[prec]) and rel_inf(grad[b], g) <= TOL[prec]
    br.close()


@pytest.mark.parametrize("batch,n,counts", [(8, 1000, [1, 3, 5, 7]), (128, 1000, [1, 17, 100, 127]),
                                            (128, 2000, [110, 64, 3])])
def test_every_subset_size_fits_the_partial_buffers(batch, n, counts):
    """Subsets re-plan the stream-K split (fewer row tiles -> more CTAs per row tile).  The partial-sum slots are
    indexed by CTA and sized once for the fullest grid, so no subset size can outgrow them (a smaller subset used
    to need MORE slots per row tile than the bind-time plan had reserved).  Every subset result must be bitwise the
    result of the same problems in any other subset of the same size, and match the full evaluation to rounding;
    a full evaluation afterwards must be bitwise the first one (nothing next to the buffers was corrupted)."""
    from paper_1907_04839_b200 import BatchedRegistrations

    T, lam = 4, 10.0
    q0, p0, target = make_batch(batch, n, 77 + batch + n)
    br = BatchedRegistrations(SIGMA, n, batch, 3, "f32", max_timesteps=T)
    br.bind(q0, target, lam, T)
    full = br.evaluate(p0)
    finals = br.final_q()
    rng = np.random.default_rng(5)
    for count in counts:
        ids = np.sort(rng.choice(batch, size=count, replace=False))
        sub = br.evaluate(p0, ids)
        assert (sub[2][ids] == -1).all()
        for b in ids:
            assert np.allclose(sub[0][b], full[0][b], rtol=1e-5)
            assert rel_inf(sub[1][b], full[1][b]) <= 1e-5  # different stream-K splits: fp32 rounding
        again = br.evaluate(p0, ids)
        assert np.array_equal(again[0], sub[0]) and np.array_equal(again[1], sub[1])
    after = br.evaluate(p0)
    assert np.array_equal(after[0], full[0]) and np.array_equal(after[1], full[1])
    assert np.array_equal(br.final_q(), finals)
    br.close()


def test_batch_register_with_problems_dropping_out():
    """lms_batch_register when the problems leave the rounds at different times (different iteration budgets are
    not available per problem, so: very different conditioning -> different line-search lengths and one problem
    that diverges at once): the later rounds run on shrinking subsets."""
    from paper_1907_04839_b200 import BatchedRegistrations, LbfgsParams

    batch, n, T, lam = 10, 1000, 4, 1e3
    q0, _, target = make_batch(batch, n, 404)
    for b in range(batch):  # problem b starts (b+1) x further from its target
        target[b] = q0[b] + (target[b] - q0[b]) * (0.2 + 0.4 * b)
    target[3, 11, 2] = np.inf  # x0 = (target - q0)/T is non-finite: DivergedError(0) at the first evaluation
    br = BatchedRegistrations(SIGMA, n, batch, 3, "f32", max_timesteps=T)
    br.bind(q0, target, lam, T)
    res = br.register(LbfgsParams(max_iter=6, grad_tol=1e-3))
    assert res.status[3] == 2 and (np.delete(res.status, 3) == 0).all()
    ok = np.delete(np.arange(batch), 3)
    assert (res.final_loss[ok] < res.initial_loss[ok]).all()
    assert res.rounds < res.evaluations[ok].sum()
    # the handle is still healthy: a full evaluation of the returned momenta is finite for the surviving problems
    scalars, grad, div = br.evaluate(np.where(np.isfinite(res.momenta), res.momenta, 0.0))
    assert np.isfinite(scalars[ok]).all() and np.isfinite(grad[ok]).all()
    br.close()
