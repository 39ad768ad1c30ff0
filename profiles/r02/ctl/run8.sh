#!/bin/bash
# Exposed AllGather vs tokens/GPU with the resident control, materialised dispatch (session 3 default),
# emulated N = 8 at 770 GB/s, BF16 and FP8.
mkdir -p gpurun_out/ctl8
for f in "--fp8" ""; do
  tag=bf16; [ -n "$f" ] && tag=fp8
  for T in 16384 24576 32768 49152; do
    timeout 600 python bench.py --steps 4 --warmup 2 --ab-steps 6 --no-cpu-baseline --emulate-gather 8 --link-gbs 770 \
        --tokens $T $f 2> gpurun_out/ctl8/${tag}_$T.err | tail -1 > gpurun_out/ctl8/${tag}_$T.json
  done
done
