#!/bin/bash
# PROD2 (split A/B producers) check + A/B, and wait profiles of both.
mkdir -p gpurun_out
export ASYNCEP_LIB=$PWD/_ab/lib_prod2.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -m gpu -x -q > gpurun_out/pytest_prod2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_prod2.log
unset ASYNCEP_LIB
ASYNCEP_LIB=$PWD/_ab/lib_wp.so timeout 300 python profiles/prof_layer.py --iters 2 --fp8 > gpurun_out/wp_fp8_gather.log 2>&1
ASYNCEP_LIB=$PWD/_ab/lib_wp2.so timeout 300 python profiles/prof_layer.py --iters 2 --fp8 > gpurun_out/wp2_fp8_gather.log 2>&1
rm -f gpurun_out/ab_libs.log
ROUNDS=2 bash profiles/ab_libs.sh "new=default" "prod2=_ab/lib_prod2.so"
ROUNDS=2 BENCH_ARGS="--fp8" bash profiles/ab_libs.sh "new8=default" "prod2_8=_ab/lib_prod2.so"
true
