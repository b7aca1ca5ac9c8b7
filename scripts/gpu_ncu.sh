# ncu captures for profiles/: launch list (shares) and one full capture of the pair kernels.
set -x
mkdir -p gpurun_out
V=${1:-0}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v$V.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --variant $V > gpurun_out/ncu_launch_v$V.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 38 -c 4 -f -o gpurun_out/prof_v$V \
    python bench.py --steps 1 --warmup 3 --no-extras --variant $V > gpurun_out/ncu_full_v$V.log 2>&1
tail -3 gpurun_out/ncu_full_v$V.log
ls -la gpurun_out
