"""Exploration: how does L-BFGS behave at N=20k on the fixed-diameter and density-scaled problems?"""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, LbfgsParams, minimize, make_synthetic_pair

for density_scaled in (False, True):
    for prec in ("f64", "f32"):
        n, T = 20000, 10
        q0, target, p_true = make_synthetic_pair(n, 1.5, T, density_scaled=density_scaled)
        x0 = ((target - q0) / T).ravel()
        s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
        s.bind_registration(q0, target, 5e5, T)
        hist = []
        def obj(x):
            l, g = s.objective(x)
            hist.append(l)
            return l, g
        t0 = time.perf_counter()
        r = minimize(obj, x0, LbfgsParams(max_iter=8))
        dt = time.perf_counter() - t0
        print(f"density_scaled={density_scaled} {prec}: init {r.initial_loss:.4e} gnorm {r.initial_grad_inf_norm:.3e} "
              f"final {r.loss:.4e} iters {len(r.iterations)} evals {r.evaluations} reason {r.reason} "
              f"ms/iter {dt*1e3/max(len(r.iterations),1):.1f}")
        print("   evals:", ["%.3e" % v for v in hist[:12]])
        print("   steps:", [(f"{it[2]:.2e}", it[3]) for it in r.iterations])
        disp = np.linalg.norm(target - q0, axis=1)
        print("   mean |target-q0|", disp.mean(), "max", disp.max())
        s.close()
