mkdir -p gpurun_out/r02i
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -x -q -p no:cacheprovider -k "not eight_layer and not 235b and not zipf" > gpurun_out/r02i/quick.log 2>&1; echo rc=$? >> gpurun_out/r02i/quick.log
for m in 240 0; do
  ASYNCEP_SWAP_MAX=$m timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel<1" -s 2 -c 1 -o gpurun_out/r02i/g1_bf16_16k_swap$m python bench.py --layers 1 --tokens 16384 --steps 2 --warmup 3 --no-cpu-baseline --no-ab > gpurun_out/r02i/ncu_$m.log 2>&1
done
