#!/bin/bash
# GPU session: tests, default bench, fp64 exp-table A/B, ncu launch lists + full captures (fp32, fp64), configs[0].
tag=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 10 --warmup 3 --precision f64 --no-extras > gpurun_out/${tag}_bench_f64.json 2>> gpurun_out/${tag}_bench.err
LMS_LIB_PATH=$PWD/paper_1907_04839_b200/liblmshoot_b200_exp6.so timeout 300 python bench.py --steps 10 --warmup 3 --precision f64 --no-extras > gpurun_out/${tag}_bench_f64_exp6.json 2>> gpurun_out/${tag}_bench.err
timeout 300 python scripts/gpu_c1.py > gpurun_out/${tag}_c1.log 2>&1; cat gpurun_out/${tag}_c1.log
bash scripts/gpu_ncu.sh ${tag}_f32 > /dev/null 2>&1
bash scripts/gpu_ncu.sh ${tag}_f64 --precision f64 > /dev/null 2>&1
ls -la gpurun_out | tail -20
