#!/bin/bash
# Round-end evidence with the current kernels: emulated 1/2/4/8-rank scaling (BF16, FP8),
# the Qwen3-30B layer shape, and the decoder stack with DP attention.
mkdir -p gpurun_out
bash profiles/scale_emulated.sh
timeout 400 python bench.py --shape 30b --tokens 16384 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_30b.json 2>/dev/null
timeout 400 python bench.py --attn --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_attn.json 2>/dev/null
