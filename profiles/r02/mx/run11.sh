# fused act quantisation (warp 2 of GEMM1) tests + A/B; launch lists of the bench (our kernels only)
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_mx.py -q -x > gpurun_out/r11_tests.log 2>&1; tail -2 gpurun_out/r11_tests.log
for T in 32768 16384; do
timeout 600 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 0 --flags-b 0x400 --pairs 8 > gpurun_out/ab11_faq_$T.json 2>> gpurun_out/ab11.err
timeout 600 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 0x400 --flags-b 0 --pairs 8 > gpurun_out/ab11_faq_rev_$T.json 2>> gpurun_out/ab11.err
done
K='regex:gemm_tc|combine|perm_|quant|gather_copy|router'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/r11_launches_bf16.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/r11_launches_fp8.csv \
  python bench.py --fp8 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
