#!/bin/bash
# Round-end evidence for profiles/: bench lines (BF16, FP8), ncu launch lists of the bench command,
# and one ncu --set full capture of the router / GEMM1 / GEMM2 launches of a 235B layer (BF16, FP8).
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/final_bf16.json 2> gpurun_out/final_bf16.err
timeout 400 python bench.py --fp8 > gpurun_out/final_fp8.json 2> gpurun_out/final_fp8.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_bf16.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_fp8.csv \
  python bench.py --fp8 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 3 -f \
  -o gpurun_out/gemm_full_bf16 python profiles/prof_layer.py --iters 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 3 -f \
  -o gpurun_out/gemm_full_fp8 python profiles/prof_layer.py --iters 2 --fp8 > /dev/null 2>&1
ls -la gpurun_out
