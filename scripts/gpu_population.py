"""BASELINE configs[3], one GPU's share end to end: B registrations of N landmarks, each an unchanged L-BFGS driver on
its own host thread, objective calls coalesced into one batched evaluation per round (lms_batch_register).
Reports wall time per registration batch, rounds, ms per round against the device time of one batched evaluation.
usage: python scripts/gpu_population.py [B] [N] [iters] [prec]"""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import BatchedRegistrations, HamiltonianSystem, LbfgsParams, make_template_points, rng_normals

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 30
prec = sys.argv[4] if len(sys.argv) > 4 else "f32"
T, sigma, lam = 10, 1.5, 5e5
base = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
gen = HamiltonianSystem(sigma, n, 3, "f64", max_timesteps=T)
q0 = np.empty((B, n, 3)); target = np.empty((B, n, 3))
for b in range(B):
    q0[b] = base
    target[b] = gen.integrate_forward(base, (0.75 * rng_normals(b, n * 3)).reshape(n, 3), T)[0][-1]
gen.close()
br = BatchedRegistrations(sigma, n, B, 3, prec, max_timesteps=T)
br.bind(q0, target, lam, T)
x0 = (target - q0) / T
for _ in range(3):
    br.evaluate(x0)
eval_ms = br.last_eval_device_ms()
t0 = time.perf_counter(); br.evaluate(x0); eval_wall = (time.perf_counter() - t0) * 1e3
for rep in range(2):
    t0 = time.perf_counter()
    res = br.register(LbfgsParams(max_iter=iters))
    wall = (time.perf_counter() - t0) * 1e3
    ev = np.asarray(res.evaluations)
    rounds = getattr(res, "rounds", None)
    print(f"{prec} B={B} N={n} iters={iters} run {rep}: {wall:.1f} ms wall, evaluations per problem {ev.min()}..{ev.max()}, "
          f"rounds {rounds}, batched evaluation {eval_ms:.2f} ms device / {eval_wall:.2f} ms wall -> "
          f"{wall / max(rounds or ev.max(), 1):.2f} ms per round; {B / (wall * 1e-3):.1f} registrations/s; "
          f"final loss median {np.median(res.final_loss):.4e}")
br.close()
