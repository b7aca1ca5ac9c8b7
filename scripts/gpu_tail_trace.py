"""Hand-over chain of the CTAs that finish a shared row tile (stream-K combine), in microseconds, from the
-DLMS_TAIL_TRACE measurement build:
    LMS_BUILD_TAG=tail LMS_NVCC_EXTRA=-DLMS_TAIL_TRACE python -c "import __graft_entry__ as g; g.build()"
    gpurun -- python scripts/gpu_tail_trace.py [N]
phases: partial stores issued | fence | arrival (barrier + atomic + barrier) | segment loads and adds | epilogue."""
import os
import re
import subprocess
import sys
from collections import defaultdict

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals

    n, T = int(sys.argv[2]), 10
    q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
    target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    s = HamiltonianSystem(1.5, n, 3, "f32", max_timesteps=T, tiled_only=True)
    s.bind_registration(q0, target, 5e5, T)
    for _ in range(3):
        s.objective(x0)
    print("=== MARK", flush=True)
    s.objective(x0)
    print("device ms", s.last_eval_device_ms(), flush=True)
    s.close()
    sys.exit(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
env = dict(os.environ, LMS_LIB_PATH=os.path.join(ROOT, "paper_1907_04839_b200", "liblmshoot_b200_tail.so"))
out = subprocess.run([sys.executable, __file__, "child", str(n)], env=env, capture_output=True, text=True).stdout
out = out[out.index("=== MARK"):]
rows = defaultdict(list)
for m in re.finditer(r"TT mode (\d) step (\d+) cta (\d+) rt (\d+) nseg (\d+) : stores (-?\d+) fence (-?\d+) arrive (-?\d+) combine (-?\d+) epilogue (-?\d+)", out):
    mode, step, cta, rt, nseg, *ph = (int(g) for g in m.groups())
    rows[mode].append([nseg] + ph)
mhz = 1965.0
print(f"N = {n}: phases of the last-arriving CTA of a shared row tile, microseconds at {mhz:.0f} MHz (mean / max over tiles and steps)")
for mode, name in ((0, "forward"), (1, "adjoint")):
    a = np.array(rows[mode], dtype=float)
    if not len(a):
        continue
    us = a[:, 1:] / mhz
    names = ["stores", "fence", "arrive", "combine", "epilogue"]
    print(f"  {name}: {len(a)} tiles, segments per tile {a[:, 0].mean():.1f}; " +
          " | ".join(f"{nm} {us[:, i].mean():.2f} / {us[:, i].max():.2f}" for i, nm in enumerate(names)) +
          f" | total {us.sum(axis=1).mean():.2f} / {us.sum(axis=1).max():.2f}")
print(out[out.index("device ms"):].strip())
