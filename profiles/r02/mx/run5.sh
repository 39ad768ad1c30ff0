set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv
M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum
run() { ASYNCEP_MX_DIAG=$2 timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_tc_kernel -s 3 -c 6 --csv --log-file gpurun_out/r5_$3.csv \
    python profiles/prof_layer.py --iters 3 --fp8 --flags $1 > /dev/null 2>&1; }
run 0 0 f8_1; run 256 0 mx_1; run 256 2 mxd2_1; run 256 0 mx_2; run 0 0 f8_2; run 256 2 mxd2_2
