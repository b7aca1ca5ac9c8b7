# One full measurement session: GPU tests, smoke, bench (default + scalar A/B + fp64), ncu launch list and full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --variant 1 --no-extras > gpurun_out/bench_scalar.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --variant 11 --no-extras > gpurun_out/bench_r2.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --precision f64 --no-extras > gpurun_out/bench_f64.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1
bash scripts/gpu_ncu.sh v0 --variant 0
bash scripts/gpu_ncu.sh f64 --precision f64
timeout 300 python bench.py --batch 128 --steps 5 --warmup 3 > gpurun_out/bench_batch.log 2>&1
timeout 300 python bench.py --batch 128 --steps 5 --warmup 3 --precision f64 > gpurun_out/bench_batch_f64.log 2>&1
timeout 1200 python scripts/sweep.py > gpurun_out/sweep.log 2>&1
