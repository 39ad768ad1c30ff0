#!/bin/bash
# Session 4: ncu --set full of the HBM-bound kernels of one 235B layer at 32K tokens (second
# iteration of prof_layer): BF16 hist / scan / row-copy scatter / combine; FP8 adds the per-token
# quantisation-scatter and the intermediate's quantisation.
O=gpurun_out/s4hbm; mkdir -p $O
K='regex:combine|perm_|quant'
timeout 900 ncu --set full --clock-control none -k "$K" -s 4 -c 4 -f -o $O/hbm_bf16 python profiles/prof_layer.py --iters 2 > $O/bf16.log 2>&1
timeout 900 ncu --set full --clock-control none -k "$K" -s 6 -c 6 -f -o $O/hbm_fp8 python profiles/prof_layer.py --iters 2 --fp8 > $O/fp8.log 2>&1
ls -la $O
