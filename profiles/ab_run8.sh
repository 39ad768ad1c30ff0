#!/bin/bash
# Separate A/B rings for the fused-dispatch GEMM1 (ARING=1, 8+4 and 7+5 stages) vs the shared 6-stage ring.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
ASYNCEP_LIB=$PWD/_ab/lib_aring84.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py tests/test_gpu_asyncep.py -m gpu -x -q > gpurun_out/pytest_aring.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_aring.log
rm -f gpurun_out/ab_libs.log
ROUNDS=2 bash profiles/ab_libs.sh "base=default" "ar84=_ab/lib_aring84.so" "ar75=_ab/lib_aring75.so"
ROUNDS=2 BENCH_ARGS="--fp8" bash profiles/ab_libs.sh "base8=default" "ar84_8=_ab/lib_aring84.so" "ar75_8=_ab/lib_aring75.so"
true
