#!/bin/bash
# Token-major FP8 x quantisation kernel (ASYNCEP_QUANT_TOKENS=0 reverts): FP8 tests, FP8 A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
rm -f gpurun_out/ab_libs.log
run() { echo "$1 $(timeout 300 env $2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $3 2>/dev/null | tail -1)" >> gpurun_out/ab_libs.log; }
for r in 1 2; do
  run old8 "ASYNCEP_QUANT_TOKENS=0" "--fp8"
  run tok8 "ASYNCEP_QUANT_TOKENS=1" "--fp8"
done
