set -x
M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum
run() { timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_tc_kernel -s 3 -c 3 --csv --log-file gpurun_out/r8_$2.csv \
    python profiles/prof_layer.py --iters 2 $1 > /dev/null 2>&1; }
run "--fp8 --flags 0" fp8_gather; run "--fp8 --flags 16" fp8_xperm; run "--flags 0" bf16_gather; run "--flags 16" bf16_xperm
run "--fp8 --flags 64" fp8_gather_noswap
