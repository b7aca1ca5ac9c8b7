#!/bin/bash
# One GPU session: the -m gpu tests, the default bench line, the 1-GPU anchor of configs[2], and a two-rank
# launcher / exchange check on the one GPU.  Everything lands in gpurun_out/.  Usage: gpurun -- bash scripts/gpu_session.sh [tag]
tag=${1:-r2}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/${tag}_pytest.log
tail -5 gpurun_out/${tag}_pytest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
cat gpurun_out/${tag}_bench.json | cut -c1-1500
python bench.py --gpus 1 --landmarks 200000 --timesteps 20 --steps 3 --warmup 3 --no-extras > gpurun_out/${tag}_bench_c2_1gpu.json 2> gpurun_out/${tag}_bench_c2.err; echo "c2 rc=$?"
cat gpurun_out/${tag}_bench_c2_1gpu.json | cut -c1-600
python bench.py --gpus 2 --landmarks 20000 --timesteps 10 --steps 3 --warmup 3 > gpurun_out/${tag}_bench_2rank_oversub.json 2> gpurun_out/${tag}_bench_2rank.err; echo "2rank rc=$?"
cat gpurun_out/${tag}_bench_2rank_oversub.json | cut -c1-1200
tail -3 gpurun_out/${tag}_bench_2rank.err
