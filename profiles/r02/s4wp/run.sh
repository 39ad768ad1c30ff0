#!/bin/bash
# Session 4: barrier-wait breakdown of the current grouped GEMMs (GEMM_WAITPROF=1 build in
# _ab/lib_wp.so), one 235B layer at 32K tokens, default (materialised) dispatch, BF16 and FP8.
O=gpurun_out/s4wp; mkdir -p $O
export ASYNCEP_LIB=$PWD/_ab/lib_wp.so
timeout 300 python profiles/prof_layer.py --iters 3 > $O/wp_bf16.log 2>&1
timeout 300 python profiles/prof_layer.py --iters 3 --fp8 > $O/wp_fp8.log 2>&1
python profiles/waitprof_parse2.py $O/wp_bf16.log > $O/waitprof_bf16.txt
python profiles/waitprof_parse2.py $O/wp_fp8.log > $O/waitprof_fp8.txt
tail -n 4 $O/waitprof_*.txt
