mkdir -p gpurun_out/r02h
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -x -q -p no:cacheprovider -k "not eight_layer and not 235b and not zipf" > gpurun_out/r02h/quick.log 2>&1; echo rc=$? >> gpurun_out/r02h/quick.log
for T in 32768 16384 8192; do
  timeout 400 python profiles/ab_flags.py --tokens $T >> gpurun_out/r02h/ab_swap_bf16.jsonl 2>> gpurun_out/r02h/err.log
  timeout 400 python profiles/ab_flags.py --tokens $T --fp8 >> gpurun_out/r02h/ab_swap_fp8.jsonl 2>> gpurun_out/r02h/err.log
done
