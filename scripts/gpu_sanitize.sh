#!/bin/bash
# compute-sanitizer memcheck + racecheck over every kernel family: persistent small-N kernel, tiled kernels (R = 2 and
# R = 4 shapes), velocity / warp, batches with subsets, device-resident L-BFGS, registration metrics, peer-push layout.
set -x
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1907_04839_b200 import HamiltonianSystem, BatchedRegistrations, ShootingConfig, register_landmarks
rng = np.random.default_rng(0)
for prec in ("f32", "f64"):
    n, T = 700, 3
    q = rng.uniform(-6, 6, (n, 3)); p = rng.normal(size=(n, 3)); tg = q + 0.3 * rng.normal(size=(n, 3))
    for tiled in (False, True):  # the persistent one-launch kernel, then the tiled multi-launch path
        s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T, tiled_only=tiled)
        r = s.compute_gradient(q, p, tg, 10.0, T)
        print(prec, "tiled" if tiled else "persistent", s.last_eval_kernel_launches(), r.loss)
        s.velocities_at_step(q, p, rng.uniform(-6, 6, (333, 3)))
        s.warp_points(rng.uniform(-6, 6, (333, 3)))
        s.close()
    b = BatchedRegistrations(1.5, 300, 5, 3, prec, max_timesteps=T)
    q0 = rng.uniform(-6, 6, (5, 300, 3)); t5 = q0 + 0.3 * rng.normal(size=q0.shape)
    b.bind(q0, t5, 10.0, T); b.evaluate((t5 - q0) / T); b.evaluate((t5 - q0) / T, [3, 1]); b.close()
    # the large-N shapes (four rows per thread, column-major tiles) through a batch that is large as a whole, the
    # device-resident L-BFGS (cooperative two-loop kernel) with the device registration metrics, and the
    # exchange-arena layout of the peer-push row partition
    b = BatchedRegistrations(1.5, 1100, 30, 3, prec, max_timesteps=2)
    q0 = rng.uniform(-8, 8, (30, 1100, 3)); t30 = q0 + 0.3 * rng.normal(size=q0.shape)
    b.bind(q0, t30, 10.0, 2); b.evaluate((t30 - q0) / 2); b.close()
    n = 1100
    q = rng.uniform(-8, 8, (n, 3)); p = rng.normal(size=(n, 3)); tg = q + 0.3 * rng.normal(size=(n, 3))
    for dv in (False, True):
        reg = register_landmarks(q, tg, ShootingConfig(sigma=1.5, timesteps=T, lam=100.0, max_iter=4, precision=prec),
                                 device_vectors=dv)
        print("registration, device vectors" if dv else "registration, host driver", reg.final_loss, reg.avg_after)
    # the persistent kernel with two adjoint windows per step (fp32: above 4096 landmarks; fp64: above 2048)
    nw = 4600 if prec == "f32" else 2300
    qw = rng.uniform(-14, 14, (nw, 3)); pw = rng.normal(size=(nw, 3)); tw = qw + 0.3 * rng.normal(size=(nw, 3))
    s = HamiltonianSystem(1.5, nw, 3, prec, max_timesteps=2)
    print("two windows", s.compute_gradient(qw, pw, tw, 10.0, 2).loss, s.last_eval_kernel_launches()); s.close()
    # a mid-size problem on the tiled path: programmatic dependent launch, the combine's shared-memory landing zone
    n5 = 4500
    q5 = rng.uniform(-14, 14, (n5, 3)); p5 = rng.normal(size=(n5, 3)); t5k = q5 + 0.3 * rng.normal(size=(n5, 3))
    s = HamiltonianSystem(1.5, n5, 3, prec, max_timesteps=2, tiled_only=True)
    print("mid-size", s.compute_gradient(q5, p5, t5k, 10.0, 2).loss, s.last_eval_kernel_launches()); s.close()
    # the thin last row tile of the four-row shapes (variant 25): 4 and 2 column groups, alone and behind full tiles
    for nt in (30, 544, 700, 1056):
        qt = rng.uniform(-8, 8, (nt, 3)); pt = rng.normal(size=(nt, 3)); tt = qt + 0.3 * rng.normal(size=(nt, 3))
        s = HamiltonianSystem(1.5, nt, 3, prec, max_timesteps=2, variant=25, tiled_only=True)
        print("thin tile", nt, s.compute_gradient(qt, pt, tt, 10.0, 2).loss, s.last_eval_kernel_launches())
        s.derivatives(qt, pt); s.close()
    # (the in-process peer-push test is left out: compute-sanitizer serialises kernel launches of the process, so
    #  a rank's stream-ordered wait for its peer's flag blocks the very launch that would set it)
    s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
    blob = s.p2p_export(0, 1); s.p2p_connect([blob]); s.bind_registration(q, tg, 10.0, T)
    print("peer-push layout, one rank", s.objective(p)[0]); s.close()
PY
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 1 python /tmp/san.py > gpurun_out/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -4 gpurun_out/sanitizer_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 1 python /tmp/san.py > gpurun_out/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"
tail -4 gpurun_out/sanitizer_racecheck.log
