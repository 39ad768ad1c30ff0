mkdir -p gpurun_out/r02s
M=gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second
for T in 32768 16384; do for pf in 0 1 2 4 0; do for f in "" "--fp8"; do
  n=bf16; [ -n "$f" ] && n=fp8
  ASYNCEP_GATHER_PF=$pf timeout 300 ncu --metrics $M --clock-control none --kernel-name-base demangled -k 'regex:gemm_tc_kernel<\(int\)1' -s 1 -c 1 --csv --log-file gpurun_out/r02s/g1_${n}_${T}_pf$pf.csv python profiles/prof_layer.py --iters 2 --tokens $T $f > /dev/null 2>&1
done; done; done
