#!/bin/bash
# PLAIN_NSTG=2 (double-buffered GEMM2 epilogue staging) on the FP8 path.
mkdir -p gpurun_out
rm -f gpurun_out/ab_libs.log
ROUNDS=3 BENCH_ARGS="--fp8" bash profiles/ab_libs.sh "base8=default" "nstg2_8=_ab/lib_nstg2.so"
