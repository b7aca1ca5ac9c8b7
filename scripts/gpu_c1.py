"""BASELINE configs[0]: N = 1000, T = 10, 100 L-BFGS iterations (the case the reference CPU runs): wall time of
the whole registration through the C ABI, host driver and device-resident driver, fp64 and fp32; best and median
of 7 runs after one warm-up, and the share of the wall time spent inside objective evaluations (host driver:
the rest is the reference-order sequential vector arithmetic of the L-BFGS two-loop recursion on the host)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, ShootingConfig, register_landmarks, make_synthetic_pair

n, T = 1000, 10
q0, target, _ = make_synthetic_pair(n, 1.5, T)
for prec in ("f64", "f32"):
    s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
    s.bind_registration(q0, target, 5e5, T)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    for _ in range(5):
        s.objective(x0)
    t0 = time.perf_counter()
    for _ in range(50):
        s.objective(x0)
    eval_wall = (time.perf_counter() - t0) / 50 * 1e3
    eval_dev = s.last_eval_device_ms()
    for dv in (False, True):
        cfg = ShootingConfig(sigma=1.5, timesteps=T, lam=5e5, max_iter=100, precision=prec)
        register_landmarks(q0, target, cfg, system=s, device_vectors=dv, already_bound=True)  # warm-up
        times = []
        for _ in range(7):
            t0 = time.perf_counter()
            r = register_landmarks(q0, target, cfg, system=s, device_vectors=dv, already_bound=True)
            times.append((time.perf_counter() - t0) * 1e3)
        ms, med = min(times), float(np.median(times))
        print(f"{prec} device_vectors={dv}: {r.iterations} iterations, {r.evaluations} evaluations, best {ms:.1f} ms "
              f"(median {med:.1f}), {ms / r.iterations:.3f} ms/iter, evaluations alone {r.evaluations * eval_wall:.1f} ms "
              f"({eval_wall:.3f} ms wall / {eval_dev:.3f} ms device each), loss {r.initial_loss:.4e} -> {r.final_loss:.6e}, "
              f"avg dist {r.avg_before:.4f} -> {r.avg_after:.2e} mm")
    s.close()
