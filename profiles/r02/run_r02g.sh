mkdir -p gpurun_out/r02g
for T in 32768 16384 8192; do
  timeout 400 python profiles/ab_flags.py --tokens $T >> gpurun_out/r02g/ab_swap_bf16.jsonl 2>> gpurun_out/r02g/err.log
  timeout 400 python profiles/ab_flags.py --tokens $T --fp8 >> gpurun_out/r02g/ab_swap_fp8.jsonl 2>> gpurun_out/r02g/err.log
done
