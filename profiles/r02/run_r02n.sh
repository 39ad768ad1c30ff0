mkdir -p gpurun_out/r02n
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -x -q -p no:cacheprovider -k "swap or fused or fp8_layer" > gpurun_out/r02n/quick.log 2>&1; echo rc=$? >> gpurun_out/r02n/quick.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct
for pa in 0 1 2; do for pb in 1 0 2; do
  ASYNCEP_POL_A=$pa ASYNCEP_POL_B=$pb timeout 300 ncu --metrics $M --clock-control none --kernel-name-base demangled -k 'regex:gemm_tc_kernel<\(int\)1' -s 1 -c 1 --csv --log-file gpurun_out/r02n/pol_a${pa}_b${pb}.csv python profiles/prof_layer.py --iters 2 > /dev/null 2>&1
done; done
for T in 32768 16384; do
  timeout 400 python profiles/ab_flags.py --tokens $T --fp8 >> gpurun_out/r02n/ab_swap_fp8.jsonl 2>> gpurun_out/r02n/err.log
done
