"""Where does an L-BFGS iteration's time go at N = 20 000?  total - evaluations x (ms per evaluation), for the host
driver (lms_register) and the device-resident one (lms_register_device), at several iteration counts."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, ShootingConfig, register_landmarks, make_synthetic_pair

n, T = int(sys.argv[1]) if len(sys.argv) > 1 else 20000, 10
q0, target, _ = make_synthetic_pair(n, 1.5, T, density_scaled=True)
for prec in ("f32",):
    s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
    s.bind_registration(q0, target, 5e5, T)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    for _ in range(3):
        s.objective(x0)
    t0 = time.perf_counter()
    for _ in range(10):
        s.objective(x0)
    ev_ms = (time.perf_counter() - t0) * 100
    print(f"{prec}: host-buffer evaluation {ev_ms:.3f} ms wall, device {s.last_eval_device_ms():.3f} ms")
    for iters in (10, 10, 30, 60):
        for dv in (False, True):
            cfg = ShootingConfig(sigma=1.5, timesteps=T, lam=5e5, max_iter=iters, precision=prec)
            t0 = time.perf_counter()
            r = register_landmarks(q0, target, cfg, system=s, device_vectors=dv, already_bound=True)
            ms = (time.perf_counter() - t0) * 1e3
            ov = ms - (r.evaluations + 1) * ev_ms
            print(f"  iters {r.iterations:3d} evals {r.evaluations:3d} device_vectors={dv}: total {ms:8.2f} ms, "
                  f"{ms / r.iterations:6.2f} ms/iter, non-evaluation time {ov:7.2f} ms = {ov / r.iterations:5.2f} ms/iter, "
                  f"loss {r.final_loss:.6e}")
    s.close()
