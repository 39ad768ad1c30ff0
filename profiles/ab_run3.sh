#!/bin/bash
# Full GPU tests on the default build; FP8 A/B of the register-cached x quantisation.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
rm -f gpurun_out/ab_libs.log
ROUNDS=3 BENCH_ARGS="--fp8" bash profiles/ab_libs.sh "oldq8=_ab/lib_prod2.so" "newq8=default"
true
