#!/bin/bash
# L2 prefetch of the next expert's weight tiles (ASYNCEP_PREFETCH_B=1) vs none.
mkdir -p gpurun_out
ASYNCEP_PREFETCH_B=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
rm -f gpurun_out/ab_libs.log
run() { echo "$1 $(timeout 300 env $2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $3 2>/dev/null | tail -1)" >> gpurun_out/ab_libs.log; }
for r in 1 2 3; do
  run pf0 "ASYNCEP_PREFETCH_B=0" ""
  run pf1 "ASYNCEP_PREFETCH_B=1" ""
done
for r in 1 2; do
  run pf0_8 "ASYNCEP_PREFETCH_B=0" "--fp8"
  run pf1_8 "ASYNCEP_PREFETCH_B=1" "--fp8"
done
