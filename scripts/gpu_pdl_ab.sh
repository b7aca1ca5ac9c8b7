# A/B of programmatic dependent launch: parity smoke, sweep of small/mid N and the default bench, with LMS_PDL=0/1
set -x
mkdir -p gpurun_out
for pdl in 1 0; do
  export LMS_PDL=$pdl
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
  timeout 600 python scripts/sweep.py 20000 20000 > gpurun_out/sweep_pdl$pdl.log 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/bench_pdl$pdl.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
grep -h "'n'" gpurun_out/sweep_pdl1.log | cut -c1-150
grep -h "'n'" gpurun_out/sweep_pdl0.log | cut -c1-150
grep -h ms_per_step gpurun_out/bench_pdl*.log | cut -c1-200
