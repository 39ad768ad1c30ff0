mkdir -p gpurun_out/r02j
for m in 240 0; do
  ASYNCEP_SWAP_MAX=$m timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_tc_kernel<\(int\)1" -s 2 -c 1 -o gpurun_out/r02j/g1_bf16_16k_swap$m python bench.py --layers 1 --tokens 16384 --steps 2 --warmup 3 --no-cpu-baseline --no-ab > gpurun_out/r02j/ncu_$m.log 2>&1
done
K='regex:gemm_tc_kernel|perm_hist|perm_scan|perm_scatter|combine_kernel|act_quant|quant_tokens|perm_quant|gather_copy'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 112 -c 224 --csv --log-file gpurun_out/r02j/launches_bf16.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02j/launch_bf16.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 144 -c 288 --csv --log-file gpurun_out/r02j/launches_fp8.csv python bench.py --fp8 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02j/launch_fp8.log 2>&1
