mkdir -p gpurun_out/r02o
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct
for pa in 0 1 2; do for pb in 1 0; do
  ASYNCEP_POL_A=$pa ASYNCEP_POL_B=$pb timeout 300 ncu --metrics $M --clock-control none --kernel-name-base demangled -k 'regex:gemm_tc_kernel<\(int\)0' -s 1 -c 1 --csv --log-file gpurun_out/r02o/g2_pol_a${pa}_b${pb}.csv python profiles/prof_layer.py --iters 2 > /dev/null 2>&1
done; done
for pg in 1 0 1; do
  ASYNCEP_POL_GATHER=$pg timeout 300 ncu --metrics $M --clock-control none --kernel-name-base demangled -k 'regex:gemm_tc_kernel<\(int\)1' -s 1 -c 1 --csv --log-file gpurun_out/r02o/g1_gather$pg.csv python profiles/prof_layer.py --iters 2 > /dev/null 2>&1
  ASYNCEP_POL_GATHER=$pg timeout 300 ncu --metrics $M --clock-control none --kernel-name-base demangled -k 'regex:gemm_tc_kernel<\(int\)1' -s 1 -c 1 --csv --log-file gpurun_out/r02o/g1f8_gather$pg.csv python profiles/prof_layer.py --iters 2 --fp8 > /dev/null 2>&1
done
