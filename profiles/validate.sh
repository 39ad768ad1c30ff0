#!/bin/bash
# Round validation on one B200: GPU tests, smoke, BF16/FP8 bench lines, reference arm.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
timeout 400 python bench.py --fp8 > gpurun_out/bench_fp8.json 2> gpurun_out/bench_fp8.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/pytest_gpu.log
