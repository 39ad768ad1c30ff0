#!/bin/bash
# Exposed AllGather with the resident-vs-resident control (bench A/B: gathered, resident, resident
# control; leg order rotated), emulated N = 8 at 770 GB/s, BF16 and FP8, 24.5K / 32K tokens/GPU.
mkdir -p gpurun_out/ctl
timeout 300 python -m pytest tests/test_gpu_mx.py -q -k "sharded or deterministic" > gpurun_out/ctl/mx_new_tests.log 2>&1
for f in "" "--fp8"; do
  tag=bf16; [ -n "$f" ] && tag=fp8
  for T in 24576 32768; do
    timeout 900 python bench.py --steps 6 --warmup 2 --ab-steps 8 --no-cpu-baseline --emulate-gather 8 --link-gbs 770 \
        --tokens $T $f 2> gpurun_out/ctl/${tag}_$T.err | tail -1 > gpurun_out/ctl/${tag}_$T.json
  done
done
tail -2 gpurun_out/ctl/mx_new_tests.log
