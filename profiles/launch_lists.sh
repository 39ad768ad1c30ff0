#!/bin/bash
# ncu launch lists (gpu__time_duration per launch, our kernels only) of the bench command.
mkdir -p gpurun_out
K='regex:gemm_tc|combine|perm_|quant|gather_copy|router'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_bf16.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_fp8.csv \
  python bench.py --fp8 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
