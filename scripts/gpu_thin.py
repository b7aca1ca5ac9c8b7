"""Thin last row tile (PairArgs::thin_split): device ms per gradient, T = 10, fp32, for
  A  variant 0 with LMS_THIN=0  (the size rule without the thin tile: two- or four-row shapes as before)
  B  variant 25 (four-row shapes), LMS_THIN=0
  C  variant 25, thin tile on (default phantom period)
  D  variant 0, thin tile on (what ships)
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
    for name, v, env in (("A", 0, {"LMS_THIN": "0"}), ("B", 25, {"LMS_THIN": "0"}), ("C", 25, {}), ("D", 0, {})):
        out = subprocess.run([sys.executable, __file__, "child", str(n), str(v)], env=dict(os.environ, **env),
                             capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1]
        row[name] = json.loads(out)
    r4 = "r4" in row["A"]["kernels"]
    print(f"N={n:6d}  A(old rule: {'R4' if r4 else 'R2'}) {row['A']['ms']:7.3f}  B(R4) {row['B']['ms']:7.3f}  "
          f"C(R4 thin) {row['C']['ms']:7.3f}  D(ships: {'R4' if 'r4' in row['D']['kernels'] else 'R2'}) {row['D']['ms']:7.3f}  "
          f"C/B {row['C']['ms'] / row['B']['ms']:.4f}  D/A {row['D']['ms'] / row['A']['ms']:.4f}", flush=True)
