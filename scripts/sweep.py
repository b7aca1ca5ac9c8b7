"""BASELINE configs[4]: scaling sweep N = 1k .. 1M at T = 10, one gradient evaluation, fp32 and fp64,
as absolute time and as a fraction of the CUDA-core pipe roofline.  Writes gpurun_out/sweep.json."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals  # noqa: E402

SIGMA, LAM, T = 1.5, 5e5, 10
PEAK = {"f32": 148 * 128 * 1965e6, "f64": 148 * 64 * 1965e6}
SLOTS = {"f32": 61, "f64": 95}
out = []
sizes = [1000, 2000, 5000, 10000, 20000, 50000, 100000, 200000, 500000, 1000000]
max_n = {"f32": int(sys.argv[1]) if len(sys.argv) > 1 else 1000000, "f64": int(sys.argv[2]) if len(sys.argv) > 2 else 200000}
for n in sizes:
    q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
    # a target a small random displacement away: timing is data-independent, and this avoids an fp64 flow at 1M
    target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    for prec in ("f32", "f64"):
        if n > max_n[prec]:
            continue
        s = HamiltonianSystem(SIGMA, n, 3, prec, max_timesteps=T)
        s.bind_registration(q0, target, LAM, T)
        reps = 20 if n <= 20000 else (5 if n <= 100000 else (2 if n <= 200000 else 1))
        # device ms: x / grad resident in HBM (CUDA events around the evaluation); wall ms: the host-buffer call
        xd = torch.from_numpy(x0).cuda()
        gd = torch.empty_like(xd)
        for _ in range(3 if n <= 100000 else 1):
            s.objective(x0)
        ms, wall = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            s.objective(x0)
            wall.append((time.perf_counter() - t0) * 1e3)
            if n <= 20000:
                s.objective_ptrs(xd.data_ptr(), gd.data_ptr(), device=True)
            ms.append(s.last_eval_device_ms())
        s.close()
        dev = float(np.median(ms))
        units = 2.0 * T * n * n
        rec = {"n": n, "precision": prec, "device_ms": dev, "wall_ms": float(np.median(wall)), "evals_per_s": units / (dev * 1e-3),
               "roofline_frac": SLOTS[prec] * T * float(n) * n / (dev * 1e-3) / PEAK[prec], "reps": reps}
        out.append(rec)
        print(rec, flush=True)
json.dump(out, open("gpurun_out/sweep.json", "w"), indent=1)
