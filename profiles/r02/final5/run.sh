#!/bin/bash
# Validation after the MX path (session 3 of round 2): full GPU suite, smoke, BF16 / FP8 bench lines.
mkdir -p gpurun_out/final5
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final5/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final5/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final5/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final5/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/final5/bench_bf16.json 2> gpurun_out/final5/bench_bf16.err
timeout 400 python bench.py --fp8 > gpurun_out/final5/bench_fp8.json 2> gpurun_out/final5/bench_fp8.err
tail -3 gpurun_out/final5/pytest_gpu.log
