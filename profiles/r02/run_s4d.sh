#!/bin/bash
# Session 4 final validation: GPU suite (incl. the random-shape sweep), smoke, headline bench lines.
O=gpurun_out/s4d; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 400 python bench.py --steps 20 > $O/bench_bf16.json 2> $O/bench_bf16.err
timeout 400 python bench.py --steps 20 --fp8 --no-cpu-baseline > $O/bench_fp8.json 2> $O/bench_fp8.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
tail -n 2 $O/pytest_gpu.log; tail -n 1 $O/smoke.log
