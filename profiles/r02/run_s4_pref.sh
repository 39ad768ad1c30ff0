#!/bin/bash
# Session 4: tile-id prefetch in the GEMM producer (SCHED_PREFETCH=1, the new default) vs the inline
# atomic (_ab/lib_nopref.so): ncu SM cycles of router / GEMM1 / GEMM2 at 32K tokens, BF16 and FP8,
# alternating libraries, 3 rounds; then the parity tests with the new default.
O=gpurun_out/s4pref; mkdir -p $O
M=gpu__time_duration.sum,sm__cycles_elapsed.max
for round in 1 2 3; do
  for d in bf16 fp8; do
    F=""; [ $d = fp8 ] && F="--fp8"
    for v in pref nopref; do
      L=""; [ $v = nopref ] && L=$PWD/_ab/lib_nopref.so
      ASYNCEP_LIB=$L timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_tc_kernel -s 3 -c 3 --csv \
        --log-file $O/${d}_${v}_${round}.csv python profiles/prof_layer.py --iters 2 $F > /dev/null 2>&1
    done
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py tests/test_gpu_shapes.py tests/test_gpu_guard.py tests/test_gpu_asyncep.py -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -n 2 $O/tests.log
