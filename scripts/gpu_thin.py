"""Thin last row tile (PairArgs::thin_split): device ms per gradient on the tiled path, T = 10, fp32, for
  R2 / R2t   two-row shapes (LMS_FORCE_ROWS=2) without / with the thin tile
  R4 / R4t   four-row shapes (LMS_FORCE_ROWS=4) without / with the thin tile
  ships      what the size rule of pick_kernels chooses (thin tile on)
usage: python scripts/gpu_thin.py N [N ...]"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
T = 10
if sys.argv[1] == "child":
    from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals

    n, v = int(sys.argv[2]), int(sys.argv[3])
    q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
    target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    s = HamiltonianSystem(1.5, n, 3, "f32", max_timesteps=T, variant=v, tiled_only=True)
    s.bind_registration(q0, target, 5e5, T)
    ms = []
    for _ in range(25):
        s.objective(x0)
        ms.append(s.last_eval_device_ms())
    print(json.dumps({"ms": float(np.median(ms[5:])), "kernels": s.lib.lms_system_kernel_names(s.handle).decode()}))
    sys.exit(0)
for n in [int(a) for a in sys.argv[1:]]:
    row = {}
    for name, env in (("R2", {"LMS_FORCE_ROWS": "2", "LMS_THIN": "0"}), ("R2t", {"LMS_FORCE_ROWS": "2"}),
                      ("R4", {"LMS_FORCE_ROWS": "4", "LMS_THIN": "0"}), ("R4t", {"LMS_FORCE_ROWS": "4"}), ("ships", {})):
        out = subprocess.run([sys.executable, __file__, "child", str(n), "0"], env=dict(os.environ, **env),
                             capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1]
        row[name] = json.loads(out)
    best = min(("R2t", "R4t"), key=lambda k: row[k]["ms"])
    print(f"N={n:6d}  R2 {row['R2']['ms']:7.3f}  R2t {row['R2t']['ms']:7.3f}  R4 {row['R4']['ms']:7.3f}  R4t {row['R4t']['ms']:7.3f}  "
          f"ships {'R4' if 'r4' in row['ships']['kernels'] else 'R2'} {row['ships']['ms']:7.3f}  best {best}  "
          f"ships/best {row['ships']['ms'] / row[best]['ms']:.4f}", flush=True)
