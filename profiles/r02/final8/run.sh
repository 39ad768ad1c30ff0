#!/bin/bash
# Round-end validation (session 3): GPU suite, smoke, bench lines (BF16 / FP8 / reference arm /
# decoder / 30B), launch lists of the bench (our kernels), ncu --set full of the GEMMs.
O=gpurun_out/final8; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 400 python bench.py --steps 20 > $O/bench_bf16.json 2> $O/bench_bf16.err
timeout 400 python bench.py --steps 20 --fp8 > $O/bench_fp8.json 2> $O/bench_fp8.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 400 python bench.py --attn --steps 6 --no-cpu-baseline > $O/bench_decoder.json 2> $O/bench_decoder.err
timeout 400 python bench.py --shape 30b --tokens 16384 --steps 10 --no-cpu-baseline > $O/bench_30b.json 2> $O/bench_30b.err
K='regex:gemm_tc|combine|perm_|quant|gather_copy|router'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file $O/launches_bf16.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file $O/launches_fp8.csv \
  python bench.py --fp8 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 3 -f \
  -o $O/gemm_full_bf16 python profiles/prof_layer.py --iters 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 3 -f \
  -o $O/gemm_full_fp8 python profiles/prof_layer.py --iters 2 --fp8 > /dev/null 2>&1
tail -3 $O/pytest_gpu.log
