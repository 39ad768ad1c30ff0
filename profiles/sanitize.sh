#!/bin/bash
# (Round 2: compute-sanitizer is closed on the GPU pool -- profiles/r02/sanitize/; tests/test_gpu_guard.py
# checks the product path for out-of-bounds writes with guard bands instead.)
# compute-sanitizer over small forwards (profiles/sanitize.py): the CUDA-core debug path under all
# three tools, then the tcgen05 product path (BF16 / FP8 / fused dispatch / MX) under memcheck.
O=${1:-gpurun_out}; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python profiles/sanitize.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_$tool.log
  tail -4 $O/sanitize_$tool.log
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python profiles/sanitize.py --tc > $O/sanitize_memcheck_tc.log 2>&1
echo "memcheck tc rc=$?" >> $O/sanitize_memcheck_tc.log
tail -12 $O/sanitize_memcheck_tc.log
