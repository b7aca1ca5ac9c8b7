"""Where should variant 0 switch from the two-row to the four-row shapes?  Device ms per gradient, T = 10, fp32."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals
T = 10
for n in [int(a) for a in sys.argv[1:]]:
    q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
    target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    row = []
    for v in (0, 25):
        s = HamiltonianSystem(1.5, n, 3, "f32", max_timesteps=T, variant=v)
        s.bind_registration(q0, target, 5e5, T)
        ms = []
        for _ in range(25):
            s.objective(x0); ms.append(s.last_eval_device_ms())
        s.close()
        row.append(float(np.median(ms[5:])))
    print(f"N={n:6d}  R=2 {row[0]:8.3f} ms   R=4 {row[1]:8.3f} ms   ratio {row[1] / row[0]:.3f}", flush=True)
