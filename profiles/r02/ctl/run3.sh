#!/bin/bash
# After the materialised-dispatch default: FP8 swap-AB tails A/B (both orders) and the exposed
# AllGather with the resident control, emulated N = 8 at 770 GB/s, BF16 / FP8, 24.5K / 32K.
mkdir -p gpurun_out/ctl3
for T in 32768 16384; do
timeout 400 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 0 --flags-b 0x40 --pairs 6 > gpurun_out/ctl3/ab_swap_$T.json 2>> gpurun_out/ctl3/ab.err
timeout 400 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 0x40 --flags-b 0 --pairs 6 > gpurun_out/ctl3/ab_swap_rev_$T.json 2>> gpurun_out/ctl3/ab.err
done
for f in "" "--fp8"; do
  tag=bf16; [ -n "$f" ] && tag=fp8
  for T in 24576 32768; do
    timeout 900 python bench.py --steps 6 --warmup 2 --ab-steps 8 --no-cpu-baseline --emulate-gather 8 --link-gbs 770 \
        --tokens $T $f 2> gpurun_out/ctl3/${tag}_$T.err | tail -1 > gpurun_out/ctl3/${tag}_$T.json
  done
done
