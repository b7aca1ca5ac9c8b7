"""A/B of measurement builds of the persistent small-N kernel (LMS_LIB_PATH picks the library): device ms per gradient,
T = 10.  usage: LMS_LIB_PATH=... python scripts/small_variants.py [prec] [sizes...]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f32"
sizes = [int(v) for v in sys.argv[2:]] or [1000, 2000, 3000, 4000]
T = 10
out = []
for n in sizes:
    q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
    target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
    s.bind_registration(q0, target, 5e5, T)
    xd = torch.from_numpy(x0).cuda()
    gd = torch.empty_like(xd)
    for _ in range(5):
        s.objective_ptrs(xd.data_ptr(), gd.data_ptr(), device=True)
    ms = []
    for _ in range(30):
        s.objective_ptrs(xd.data_ptr(), gd.data_ptr(), device=True)
        ms.append(s.last_eval_device_ms())
    out.append(f"{n}: {np.median(ms):.4f} ({s.last_eval_kernel_launches()})")
    s.close()
print(prec, " | ".join(out))
