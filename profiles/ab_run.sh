#!/bin/bash
# Same-box A/B: GPU tests on the default build, then base (_ab/lib_base.so) vs default, BF16 and FP8.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
rm -f gpurun_out/ab_libs.log
ROUNDS=${ROUNDS:-2} bash profiles/ab_libs.sh "base=_ab/lib_base.so" "new=default"
ROUNDS=${ROUNDS:-2} BENCH_ARGS="--fp8" bash profiles/ab_libs.sh "base8=_ab/lib_base.so" "new8=default"
[ -f _ab/lib_wp.so ] && ASYNCEP_LIB=$PWD/_ab/lib_wp.so timeout 300 python profiles/prof_layer.py --iters 2 --fp8 > gpurun_out/wp_fp8_gather.log 2>&1
true
