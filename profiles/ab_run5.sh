#!/bin/bash
# CTA-pair router (env ASYNCEP_ROUTER_PAIR=0 reverts it) and the unrolled FP8 x quantisation (_ab/lib_xq.so).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
rm -f gpurun_out/ab_libs.log
run() { echo "$1 $(timeout 300 env $2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $3 2>/dev/null | tail -1)" >> gpurun_out/ab_libs.log; }
for r in 1 2; do
  run r1cta "ASYNCEP_ROUTER_PAIR=0" ""
  run rpair "ASYNCEP_ROUTER_PAIR=1" ""
  run r1cta8 "ASYNCEP_ROUTER_PAIR=0" "--fp8"
  run xq8 "ASYNCEP_LIB=$PWD/_ab/lib_xq.so" "--fp8"
done
