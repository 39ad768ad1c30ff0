#!/bin/bash
# Router pair ring 8 deep (64-row W_r halves) vs 6: router tests + A/B.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
rm -f gpurun_out/ab_libs.log
ROUNDS=3 bash profiles/ab_libs.sh "base=_ab/lib_base.so" "r8=default"
