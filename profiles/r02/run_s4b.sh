#!/bin/bash
# Session 4 validation after the bench re-measure rule: GPU suite, smoke, bench lines.
O=gpurun_out/s4b; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 400 python bench.py > $O/bench_bf16.json 2> $O/bench_bf16.err
timeout 400 python bench.py --fp8 --no-cpu-baseline > $O/bench_fp8.json 2> $O/bench_fp8.err
tail -n 2 $O/pytest_gpu.log; tail -n 1 $O/smoke.log
