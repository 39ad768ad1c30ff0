#!/bin/bash
# Same-box A/B of flash-attention kernel versions (ASYNCEP_FA_VER) on the attention layer.
# usage: ROUNDS=2 bash profiles/ab_attn.sh 2 3   -> gpurun_out/ab_attn.log
for r in $(seq 1 ${ROUNDS:-2}); do for v in "$@"; do for p in 4096 32768 1024; do
  echo "v$v $(ASYNCEP_FA_VER=$v timeout 120 python profiles/prof_attn.py --prompt $p 2>&1 | tail -1)" >> gpurun_out/ab_attn.log
done; done; done
