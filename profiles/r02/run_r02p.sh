mkdir -p gpurun_out/r02p
timeout 600 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fp8 or swap" > gpurun_out/r02p/fp8_tests.log 2>&1; echo rc=$? >> gpurun_out/r02p/fp8_tests.log
for i in 1 2; do
  ASYNCEP_FUSED_ACT_QUANT=1 timeout 300 python bench.py --fp8 --no-cpu-baseline > gpurun_out/r02p/fp8_fused_$i.json 2>> gpurun_out/r02p/err.log
  ASYNCEP_FUSED_ACT_QUANT=0 timeout 300 python bench.py --fp8 --no-cpu-baseline > gpurun_out/r02p/fp8_sep_$i.json 2>> gpurun_out/r02p/err.log
done
