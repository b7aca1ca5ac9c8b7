# A/B of kernel variants at large N: usage gpu_v9.sh "<variants>" "<N list>"
for v in $1; do for n in $2; do python bench.py --steps 5 --warmup 3 --no-extras --variant $v --n $n | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('v', d['config']['variant'], d['config']['kernel_variant'], 'n', d['config']['n'], 'ms %.3f'%d['ms_per_step'], 'adj %.4f'%r['avg_launch_ms'], 'fwd %.4f'%r['forward_kernel']['avg_launch_ms'], 'grad frac %.3f'%r['gradient']['frac'])"; done; done
