"""Bitwise run-to-run stress: thousands of evaluations of the same point through the persistent kernel (grid barrier,
TMA multicast, intra-CTA stream-K) and the tiled kernels (stream-K combine), every result compared with the first.
usage: python scripts/gpu_stress.py [reps]"""
import sys, time, hashlib
import numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
T = 10
bad = 0
for n, prec, r in ((257, "f32", reps), (1000, "f32", reps), (1000, "f64", reps), (3000, "f32", reps), (4096, "f32", reps // 3),
                   (2048, "f64", reps // 3), (3400, "f64", reps // 6), (5000, "f32", reps // 3), (8192, "f32", reps // 6),
                   (9000, "f32", reps // 6), (12400, "f32", reps // 10), (20000, "f32", reps // 15)):  # 9000 ... 20000: thin last row tile
    q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
    target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
    x0 = np.ascontiguousarray(((target - q0) / T).ravel())
    s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=T)
    s.bind_registration(q0, target, 5e5, T)
    loss0, g0 = s.objective(x0)
    h0 = hashlib.sha1(g0.tobytes()).hexdigest()
    t0 = time.perf_counter()
    mism = 0
    for _ in range(r):
        loss, g = s.objective(x0)
        if loss != loss0 or hashlib.sha1(g.tobytes()).hexdigest() != h0:
            mism += 1
    print(f"N={n} {prec}: {r} evaluations in {time.perf_counter() - t0:.1f} s, launches/eval {s.last_eval_kernel_launches()}, "
          f"mismatches {mism}", flush=True)
    bad += mism
    s.close()
print("stress ok" if bad == 0 else f"stress FAILED: {bad} mismatches")
sys.exit(0 if bad == 0 else 1)
