set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 38 -c 4 -f -o gpurun_out/prof_f64 \
    python bench.py --steps 1 --warmup 3 --no-extras --precision f64 > gpurun_out/ncu_full_f64.log 2>&1
tail -2 gpurun_out/ncu_full_f64.log | cut -c1-200
