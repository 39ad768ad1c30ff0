#!/bin/bash
# Barrier-wait breakdown of the grouped GEMMs (GEMM_WAITPROF=1 build in _ab/lib_wp.so):
# one 235B layer at 32K tokens, fused dispatch vs materialised X_perm, BF16 and FP8.
mkdir -p gpurun_out
export ASYNCEP_LIB=$PWD/_ab/lib_wp.so
timeout 300 python profiles/prof_layer.py --iters 3 > gpurun_out/wp_bf16_gather.log 2>&1
timeout 300 python profiles/prof_layer.py --iters 3 --flags 16 > gpurun_out/wp_bf16_xperm.log 2>&1
timeout 300 python profiles/prof_layer.py --iters 3 --fp8 > gpurun_out/wp_fp8_gather.log 2>&1
timeout 300 python profiles/prof_layer.py --iters 3 --fp8 --flags 16 > gpurun_out/wp_fp8_xperm.log 2>&1
