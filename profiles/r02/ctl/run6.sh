#!/bin/bash
# Gated gather (held on the host, released after the next forward's dispatch): test, timeline, then
# ungated vs gated (both stacks gathered, emulated N = 8 at 770 GB/s), both orders, FP8 / BF16.
mkdir -p gpurun_out/ctl6
timeout 300 python -m pytest tests/test_gpu_asyncep.py -q -x -k gated > gpurun_out/ctl6/tests.log 2>&1; echo "rc=$?" >> gpurun_out/ctl6/tests.log
tail -2 gpurun_out/ctl6/tests.log
timeout 200 python profiles/timeline.py --fp8 --gate > gpurun_out/ctl6/tl_gate_fp8.json 2> gpurun_out/ctl6/tl_gate_fp8.err
for f in "--fp8" ""; do
  tag=bf16; [ -n "$f" ] && tag=fp8
  for T in 32768 24576; do
    timeout 400 python profiles/ab_flags.py $f --tokens $T --emulate 8 --gate b --pairs 6 > gpurun_out/ctl6/${tag}_$T.json 2>> gpurun_out/ctl6/ab.err
    timeout 400 python profiles/ab_flags.py $f --tokens $T --emulate 8 --gate a --pairs 6 > gpurun_out/ctl6/${tag}_rev_$T.json 2>> gpurun_out/ctl6/ab.err
  done
done
