#!/bin/bash
# Dispatch choice under the gather: materialised (default) vs fused, both stacks gathered (emulated
# N = 8 at 770 GB/s), BF16 / FP8, 32K and 24.5K tokens/GPU, both A/B orders.
mkdir -p gpurun_out/ctl4
for f in "" "--fp8"; do
  tag=bf16; [ -n "$f" ] && tag=fp8
  for T in 32768 24576; do
    timeout 500 python profiles/ab_flags.py $f --tokens $T --emulate 8 --flags-a 0 --flags-b 0x200 --pairs 6 > gpurun_out/ctl4/${tag}_$T.json 2>> gpurun_out/ctl4/ab.err
    timeout 500 python profiles/ab_flags.py $f --tokens $T --emulate 8 --flags-a 0x200 --flags-b 0 --pairs 6 > gpurun_out/ctl4/${tag}_rev_$T.json 2>> gpurun_out/ctl4/ab.err
  done
done
