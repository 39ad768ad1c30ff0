#!/bin/bash
# Half-height tail tiles on / off: GEMM loop cycles (GEMM_WAITPROF build), BF16 and FP8.
mkdir -p gpurun_out
export ASYNCEP_LIB=$PWD/_ab/lib_wp.so
for hf in 0 1 0 1; do
  ASYNCEP_HALF_TILES=$hf timeout 300 python profiles/prof_layer.py --iters 2 > gpurun_out/wph${hf}_bf16.log 2>&1
  ASYNCEP_HALF_TILES=$hf timeout 300 python profiles/prof_layer.py --iters 2 --fp8 > gpurun_out/wph${hf}_fp8.log 2>&1
  for f in bf16 fp8; do echo "half=$hf $f"; python profiles/waitprof_parse.py gpurun_out/wph${hf}_$f.log | sed -n 5,6p; done
done
