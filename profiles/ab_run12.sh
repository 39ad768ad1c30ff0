#!/bin/bash
# Router tiles last-first (ASYNCEP_ROUTER_REVERSE=1) vs first-first.
mkdir -p gpurun_out
ASYNCEP_ROUTER_REVERSE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiny or router or 235b" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
rm -f gpurun_out/ab_libs.log
run() { echo "$1 $(timeout 300 env $2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $3 2>/dev/null | tail -1)" >> gpurun_out/ab_libs.log; }
for r in 1 2 3; do
  run fwd "ASYNCEP_ROUTER_REVERSE=0" ""
  run rev "ASYNCEP_ROUTER_REVERSE=1" ""
done
