#!/bin/bash
# Exposed AllGather with control + per-leg SM clocks; copy CTAs 148 vs 74; BF16 / FP8 32K.
mkdir -p gpurun_out/ctl2
for f in "" "--fp8"; do
  tag=bf16; [ -n "$f" ] && tag=fp8
  for c in 148 74; do
    ASYNCEP_GATHER_CTAS=$c timeout 900 python bench.py --steps 4 --warmup 2 --ab-steps 10 --no-cpu-baseline --emulate-gather 8 \
        --link-gbs 770 --tokens 32768 $f 2> gpurun_out/ctl2/${tag}_c$c.err | tail -1 > gpurun_out/ctl2/${tag}_c$c.json
  done
done
