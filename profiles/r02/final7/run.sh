#!/bin/bash
# Validation with the materialised dispatch default for both dtypes and the measured-sustained roofline
# peak (session 3): GPU suite, smoke, bench lines (20 steps), launch lists of the bench (our kernels).
O=gpurun_out/final7; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 400 python bench.py --steps 20 > $O/bench_bf16.json 2> $O/bench_bf16.err
timeout 400 python bench.py --steps 20 --fp8 > $O/bench_fp8.json 2> $O/bench_fp8.err
timeout 400 python bench.py --steps 20 --fused-dispatch --no-cpu-baseline > $O/bench_bf16_fused.json 2> $O/bench_bf16_fused.err
K='regex:gemm_tc|combine|perm_|quant|gather_copy|router'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file $O/launches_bf16.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file $O/launches_fp8.csv \
  python bench.py --fp8 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -3 $O/pytest_gpu.log
