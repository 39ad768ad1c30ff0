mkdir -p gpurun_out/r02v
for T in 8192 16384 32768; do
  timeout 400 python profiles/ab_flags.py --tokens $T --fp8 --flags-a 0x80 --flags-b 0 >> gpurun_out/r02v/ab_fp8_g2swap.jsonl 2>> gpurun_out/r02v/err.log
  timeout 400 python profiles/ab_flags.py --tokens $T --flags-a 0x80 --flags-b 0 >> gpurun_out/r02v/ab_bf16_swap.jsonl 2>> gpurun_out/r02v/err.log
done
