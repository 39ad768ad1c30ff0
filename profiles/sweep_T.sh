#!/bin/bash
# Exposed-AllGather sweep around the saturation threshold T on one B200: 8-rank AsyncEP
# gather emulated with peer shards paced at 770 GB/s (NVLink 5 measured peer copy).
# usage: bash profiles/sweep_T.sh [bench args, e.g. --fp8 / --attn]
#        -> gpurun_out/sweep_T_<tag>.jsonl (tag = bf16, or the args without dashes/spaces)
tag=bf16; [ $# -gt 0 ] && tag=$(echo "$@" | tr -d ' -')
out=gpurun_out/sweep_T_$tag.jsonl; : > $out
for T in ${TOKENS:-4096 8192 16384 24576 32768 49152}; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --emulate-gather 8 --link-gbs 770 \
      --tokens $T "$@" 2>/dev/null | tail -1 >> $out
done
