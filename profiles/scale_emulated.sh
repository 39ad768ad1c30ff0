#!/bin/bash
# Per-GPU throughput of the AsyncEP stack with the N-rank gather emulated on one B200 (peer shards
# paced at 770 GB/s), N = 1, 2, 4, 8, BF16 and FP8 -> gpurun_out/scale_emulated.jsonl
out=${1:-gpurun_out/scale_emulated.jsonl}; mkdir -p $(dirname $out); : > $out
for f in "" "--fp8"; do
  timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $f 2>/dev/null | tail -1 >> $out
  for n in 2 4 8; do
    timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --emulate-gather $n --link-gbs 770 $f \
      2>/dev/null | tail -1 >> $out
  done
done
