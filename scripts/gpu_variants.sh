set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "variants or full_size" > gpurun_out/pytest_variants.log 2>&1; tail -5 gpurun_out/pytest_variants.log
for v in "$@"; do
  timeout 300 python bench.py --steps 5 --warmup 3 --variant $v --no-extras > gpurun_out/bench_v$v.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_v*.log')):
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l); r=d['roofline']
            print(f, d['config']['kernel_variant'], 'ms/step %.3f'%d['ms_per_step'], 'adj %.4f ms frac %.3f'%(r['avg_launch_ms'], r['frac']), 'fwd %.4f ms frac %.3f'%(r['forward_kernel']['avg_launch_ms'], r['forward_kernel']['frac']), 'grad frac %.3f'%r['gradient']['frac'])
PY
