#!/bin/bash
# One GPU session: -m gpu tests, default bench, fp64 bench, reference arm, configs[0], small-N A/B, ncu (fp32 + fp64).
tag=${1:-r2c}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/${tag}_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/${tag}_pytest.log; tail -4 gpurun_out/${tag}_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 10 --warmup 3 --precision f64 --no-extras > gpurun_out/${tag}_bench_f64.json 2>> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2>> gpurun_out/${tag}_bench.err; echo "ref rc=$?"
timeout 300 python scripts/gpu_c1.py > gpurun_out/${tag}_c1.log 2>&1; cat gpurun_out/${tag}_c1.log
timeout 600 python scripts/small_ab.py gpurun_out/${tag}_small_ab.json > gpurun_out/${tag}_small_ab.log 2>&1; tail -20 gpurun_out/${tag}_small_ab.log | cut -c1-400
bash scripts/gpu_ncu.sh ${tag}_f32 > /dev/null 2>&1
bash scripts/gpu_ncu.sh ${tag}_f64 --precision f64 > /dev/null 2>&1
ls -la gpurun_out | tail -30
