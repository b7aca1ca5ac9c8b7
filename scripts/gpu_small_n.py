"""Small-N latency probe: one gradient at N (argv[1]), T = 10, fp32 (argv[2] = precision)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals
n = int(sys.argv[1]); prec = sys.argv[2] if len(sys.argv) > 2 else "f32"; T = 10
q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
x0 = np.ascontiguousarray(((target - q0) / T).ravel())
s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
s.bind_registration(q0, target, 5e5, T)
ms = []
for _ in range(30):
    s.objective(x0); ms.append(s.last_eval_device_ms())
print(n, prec, "device ms median", float(np.median(ms)))
s.close()
