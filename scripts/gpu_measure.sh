#!/bin/bash
# The round's remaining measurements: configs[4] sweep, configs[3] per-GPU batch share (fp32, fp64), configs[2] 1-GPU
# anchor, L-BFGS overhead per iteration.  usage: gpu_measure.sh [tag]
tag=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python scripts/sweep.py 1000000 200000 > gpurun_out/${tag}_sweep.log 2>&1; cp gpurun_out/sweep.json gpurun_out/${tag}_sweep.json; tail -3 gpurun_out/${tag}_sweep.log | cut -c1-200
timeout 600 python bench.py --batch 128 --landmarks 2000 --steps 10 --warmup 3 --no-extras > gpurun_out/${tag}_bench_batch.json 2> gpurun_out/${tag}_bench_batch.err; echo "batch rc=$?"
timeout 600 python bench.py --batch 128 --landmarks 2000 --steps 10 --warmup 3 --no-extras --precision f64 > gpurun_out/${tag}_bench_batch_f64.json 2>> gpurun_out/${tag}_bench_batch.err; echo "batch f64 rc=$?"
timeout 900 python bench.py --gpus 1 --landmarks 200000 --timesteps 20 --steps 3 --warmup 3 --no-extras > gpurun_out/${tag}_bench_c2_1gpu.json 2> gpurun_out/${tag}_bench_c2.err; echo "c2 rc=$?"
timeout 600 python scripts/gpu_lbfgs_overhead.py > gpurun_out/${tag}_lbfgs_overhead.log 2>&1; tail -12 gpurun_out/${tag}_lbfgs_overhead.log | cut -c1-220
