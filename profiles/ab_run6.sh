#!/bin/bash
# 8-warp stable ranks in the scatter + block-parallel expert scan: GPU tests, then base vs new.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
rm -f gpurun_out/ab_libs.log
ROUNDS=2 bash profiles/ab_libs.sh "base=_ab/lib_base.so" "new=default"
ROUNDS=1 BENCH_ARGS="--fp8" bash profiles/ab_libs.sh "base8=_ab/lib_base.so" "new8=default"
true
