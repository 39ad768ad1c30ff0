#!/bin/bash
# ncu --set full of the HBM-bound kernels of one 235B layer (BF16 and FP8): combine, permute, quantisation.
mkdir -p gpurun_out
K='regex:combine|perm_|quant'
timeout 900 ncu --set full --clock-control none -k "$K" -s 5 -c 5 -f -o gpurun_out/hbm_bf16 python profiles/prof_layer.py --iters 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k "$K" -s 6 -c 6 -f -o gpurun_out/hbm_fp8 python profiles/prof_layer.py --iters 2 --fp8 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
