# fused act quantisation after the reset-race fix: tests, isolated GEMM1 cycles, A/B (strict timeouts)
timeout 400 python -m pytest tests/test_gpu_fp8.py -q -x -k "act_quant or 235b" > gpurun_out/r13_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r13_tests.log; tail -2 gpurun_out/r13_tests.log
M=gpu__time_duration.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum
for f in 0 1024; do
timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc_kernel -s 3 -c 3 --csv --log-file gpurun_out/r13_cyc_$f.csv \
    python profiles/prof_layer.py --iters 2 --fp8 --flags $f > /dev/null 2>&1
done
timeout 300 python profiles/ab_flags.py --fp8 --tokens 32768 --flags-a 0 --flags-b 0x400 --pairs 6 > gpurun_out/ab13_faq_32768.json 2>> gpurun_out/ab13.err
timeout 300 python profiles/ab_flags.py --fp8 --tokens 32768 --flags-a 0x400 --flags-b 0 --pairs 6 > gpurun_out/ab13_faq_rev_32768.json 2>> gpurun_out/ab13.err
