for v in 0 9 8; do for n in 14000 20000 50000 100000; do python bench.py --steps 5 --warmup 3 --no-extras --variant $v --n $n | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('v', d['config']['variant'], 'n', d['config']['n'], 'ms %.3f'%d['ms_per_step'], 'adj %.4f'%r['avg_launch_ms'], 'fwd %.4f'%r['forward_kernel']['avg_launch_ms'], 'grad frac %.3f'%r['gradient']['frac'])"; done; done
