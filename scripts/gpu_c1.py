"""BASELINE configs[0]: N = 1000, T = 10, 100 L-BFGS iterations (the case the reference CPU runs): wall time of
the whole registration through the C ABI, host driver and device-resident driver, fp64 and fp32."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, ShootingConfig, register_landmarks, make_synthetic_pair

n, T = 1000, 10
q0, target, _ = make_synthetic_pair(n, 1.5, T)
for prec in ("f64", "f32"):
    s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
    s.bind_registration(q0, target, 5e5, T)
    for dv in (False, True):
        cfg = ShootingConfig(sigma=1.5, timesteps=T, lam=5e5, max_iter=100, precision=prec)
        register_landmarks(q0, target, cfg, system=s, device_vectors=dv, already_bound=True)  # warm-up
        t0 = time.perf_counter()
        r = register_landmarks(q0, target, cfg, system=s, device_vectors=dv, already_bound=True)
        ms = (time.perf_counter() - t0) * 1e3
        print(f"{prec} device_vectors={dv}: {r.iterations} iterations, {r.evaluations} evaluations, {ms:.1f} ms total, "
              f"{ms / r.iterations:.3f} ms/iter, loss {r.initial_loss:.4e} -> {r.final_loss:.6e}, "
              f"avg dist {r.avg_before:.4f} -> {r.avg_after:.2e} mm")
    s.close()
