# usage: gpu_try_variants.sh "<f32 variants>" "<f64 variants>"  -- parity smoke + bench for experimental kernel variants
set -x
mkdir -p gpurun_out
cat > /tmp/vcheck.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
from oracle import load_oracle
from paper_1907_04839_b200 import HamiltonianSystem
prec, variant = sys.argv[1], int(sys.argv[2])
o = load_oracle(); rng = np.random.default_rng(0)
for n in (7, 257, 1000, 2300):
    q = rng.uniform(-7, 7, (n, 3)); p = 0.75 * rng.normal(size=(n, 3)); tg = q + 0.5 * rng.normal(size=(n, 3))
    s = HamiltonianSystem(1.5, n, 3, prec, max_timesteps=5, variant=variant)
    r = s.compute_gradient(q, p, tg, 10.0, 5); r2 = s.compute_gradient(q, p, tg, 10.0, 5)
    l, k, m, g = o.compute_gradient(prec, q, p, tg, 1.5, 10.0, 5)
    err = np.abs(r.grad - g).max() / np.abs(g).max()
    assert err < (1e-5 if prec == "f32" else 1e-10), (n, err)
    assert np.array_equal(r.grad, r2.grad)
    s.close()
print("variant", prec, variant, "parity ok")
PY
for v in $1; do timeout 120 python /tmp/vcheck.py f32 $v || echo "FAILED f32 $v"; done
for v in $2; do timeout 120 python /tmp/vcheck.py f64 $v || echo "FAILED f64 $v"; done
for v in 0 $1; do timeout 200 python bench.py --steps 10 --warmup 3 --no-extras --variant $v > gpurun_out/bench_v$v.log 2>&1; done
for v in 0 $2; do timeout 200 python bench.py --steps 5 --warmup 3 --no-extras --precision f64 --variant $v > gpurun_out/bench_f64_v$v.log 2>&1; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_v*.log'))+sorted(glob.glob('gpurun_out/bench_f64_v*.log')):
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l); r=d['roofline']
            print(f, d['config']['kernel_variant'], 'ms/step %.3f'%d['ms_per_step'], 'adj %.4f ms frac %.3f'%(r['avg_launch_ms'], r['frac']), 'fwd %.4f ms frac %.3f'%(r['forward_kernel']['avg_launch_ms'], r['forward_kernel']['frac']))
PY
