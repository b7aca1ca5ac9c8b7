set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 120 profiles/ubench/pipes gpurun_out/pipes_b200.json > gpurun_out/pipes.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
for v in 0 1 2 3; do
  timeout 300 python bench.py --steps 5 --warmup 3 --variant $v --no-extras > gpurun_out/bench_v$v.log 2>&1
done
timeout 300 python bench.py --steps 5 --warmup 3 --precision f64 --no-extras > gpurun_out/bench_f64.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.log 2>&1
tail -c 1500 gpurun_out/smoke.log
cat gpurun_out/pipes.log
