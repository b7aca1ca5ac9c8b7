# ncu captures for profiles/: launch list (shares) and one full capture of the pair kernels.
# usage: gpu_ncu.sh <tag> [bench args...]      e.g.  gpu_ncu.sh v0 --variant 0   |   gpu_ncu.sh f64 --precision f64
set -x
mkdir -p gpurun_out
TAG=$1; shift
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-extras "$@" > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 49 -c 2 -f -o gpurun_out/prof_$TAG \
    python bench.py --steps 1 --warmup 3 --no-extras "$@" > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log | cut -c1-300
