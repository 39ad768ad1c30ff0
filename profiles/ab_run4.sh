#!/bin/bash
# Half-height tail tiles: GPU tests on the default build, then base (_ab/lib_prod2.so) vs default.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
rm -f gpurun_out/ab_libs.log
ROUNDS=2 bash profiles/ab_libs.sh "base=_ab/lib_prod2.so" "half=default"
ROUNDS=2 BENCH_ARGS="--fp8" bash profiles/ab_libs.sh "base8=_ab/lib_prod2.so" "half8=default"
true
