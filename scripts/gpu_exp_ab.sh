# A/B of the fp64 exp table size (LMS_EXP_BITS = 4, 5, 6): builds three copies of the library here (CPU),
# then on the GPU swaps each in, checks parity (smoke + the fp64 exp accuracy test) and benches fp64.
# usage (here):   bash scripts/gpu_exp_ab.sh build      (GPU box):   bash scripts/gpu_exp_ab.sh run
set -x
LIB=paper_1907_04839_b200/liblmshoot_b200.so
if [ "$1" = build ]; then
  mkdir -p build_ab
  for b in 4 5 6; do
    (cd paper_1907_04839_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
       -DLMS_EXP_BITS=$b -o ../../build_ab/lib_exp$b.so system.cu capi.cu device_lbfgs.cu lbfgs_driver.cpp -ldl) &
  done
  wait
else
  mkdir -p gpurun_out
  cp $LIB /tmp/lib_orig.so
  for b in 4 5 6; do
    cp build_ab/lib_exp$b.so $LIB
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | grep f64
    timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "kernel_values or f64" 2>&1 | tail -1
    timeout 300 python bench.py --steps 5 --warmup 3 --precision f64 --no-extras > gpurun_out/bench_exp$b.log 2>&1
    grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_exp$b.log | head -1
    grep -o '"avg_launch_ms": [0-9.]*' gpurun_out/bench_exp$b.log
  done
  cp /tmp/lib_orig.so $LIB
fi
