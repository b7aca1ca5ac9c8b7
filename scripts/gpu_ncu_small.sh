#!/bin/bash
# ncu --set full of the persistent small-N kernel.  usage: gpu_ncu_small.sh <tag> <n> [f32|f64]
tag=$1; n=${2:-2000}; prec=${3:-f32}
mkdir -p gpurun_out
cat > /tmp/one_small.py <<PY
import sys, numpy as np
sys.path.insert(0, ".")
from paper_1907_04839_b200 import HamiltonianSystem, make_template_points, rng_normals
n, T = $n, 10
q0 = make_template_points(n, 40.0 * float(np.sqrt(n / 1847.0)))
target = q0 + 0.5 * rng_normals(1, n * 3).reshape(n, 3)
x0 = np.ascontiguousarray(((target - q0) / T).ravel())
s = HamiltonianSystem(1.5, n, 3, "$prec", max_timesteps=T)
s.bind_registration(q0, target, 5e5, T)
for _ in range(6):
    s.objective(x0)
print(s.last_eval_device_ms())
PY
LMS_SMALL_MAX_N=100000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_eval -s 4 -c 1 -f -o gpurun_out/prof_small_${tag} python /tmp/one_small.py > gpurun_out/ncu_small_${tag}.log 2>&1
tail -3 gpurun_out/ncu_small_${tag}.log
