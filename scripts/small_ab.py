"""Small / mid-size single problems: the persistent one-launch kernel against the tiled multi-launch path, one
gradient at T = 10, fp32 and fp64 (device ms = CUDA events around the evaluation, wall ms = the whole host-buffer
C-ABI call).  Usage: python scripts/small_ab.py [out.json] [sizes...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals  # noqa: E402

SIGMA, LAM, T = 1.5, 5e5, 10
PEAK = {"f32": 148 * 128 * 1965e6, "f64": 148 * 64 * 1965e6}
SLOTS = {"f32": 61, "f64": 95}
out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/small_ab.json"
sizes = [int(v) for v in sys.argv[2:]] or [500, 1000, 1500, 2000, 3000, 4000, 5000, 7000, 9000]
os.environ["LMS_SMALL_MAX_N"] = "100000"  # let the persistent path take every size its register budget allows
out = []
for n in sizes:
    q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
    target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    for prec in ("f32", "f64"):
        rec = {"n": n, "precision": prec}
        for name, tiled in (("persistent", False), ("tiled", True)):
            s = HamiltonianSystem(SIGMA, n, 3, prec, max_timesteps=T, tiled_only=tiled)
            s.bind_registration(q0, target, LAM, T)
            # device ms: x / grad resident in HBM (CUDA events around the evaluation); wall ms: the host-buffer call
            xd = torch.from_numpy(x0).cuda()
            gd = torch.empty_like(xd)
            for _ in range(5):
                s.objective(x0)
                s.objective_ptrs(xd.data_ptr(), gd.data_ptr(), device=True)
            launches = s.last_eval_kernel_launches()
            ms, wall = [], []
            for _ in range(30):
                t0 = time.perf_counter()
                s.objective(x0)
                wall.append((time.perf_counter() - t0) * 1e3)
                s.objective_ptrs(xd.data_ptr(), gd.data_ptr(), device=True)
                ms.append(s.last_eval_device_ms())
            s.close()
            dev = float(np.median(ms))
            rec[name] = {"device_ms": dev, "wall_ms": float(np.median(wall)), "launches": launches,
                         "roofline_frac": SLOTS[prec] * T * float(n) * n / (dev * 1e-3) / PEAK[prec]}
        out.append(rec)
        print(json.dumps(rec), flush=True)
json.dump(out, open(out_path, "w"), indent=1)
