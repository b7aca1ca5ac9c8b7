set -x
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1907_04839_b200 import HamiltonianSystem, BatchedRegistrations
rng = np.random.default_rng(0)
for prec in ("f32", "f64"):
    n, T = 700, 3
    q = rng.uniform(-6, 6, (n, 3)); p = rng.normal(size=(n, 3)); tg = q + 0.3 * rng.normal(size=(n, 3))
    s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
    r = s.compute_gradient(q, p, tg, 10.0, T)
    s.velocities_at_step(q, p, rng.uniform(-6, 6, (333, 3)))
    s.warp_points(rng.uniform(-6, 6, (333, 3)))
    s.close()
    b = BatchedRegistrations(1.5, 300, 5, 3, prec, max_timesteps=T)
    q0 = rng.uniform(-6, 6, (5, 300, 3)); t5 = q0 + 0.3 * rng.normal(size=q0.shape)
    b.bind(q0, t5, 10.0, T); b.evaluate((t5 - q0) / T); b.evaluate((t5 - q0) / T, [3, 1]); b.close()
    print(prec, r.loss)
PY
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 1 python /tmp/san.py > gpurun_out/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -4 gpurun_out/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 1 python /tmp/san.py > gpurun_out/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"
tail -4 gpurun_out/sanitizer_racecheck.log
