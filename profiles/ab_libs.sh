#!/bin/bash
# Same-box A/B of library variants (build.py -D ... --out _ab/lib_X.so): alternates the
# variants ROUNDS times and prints one summary line per run.
# usage: ROUNDS=2 BENCH_ARGS="--fp8" bash profiles/ab_libs.sh "label=lib_path|extra bench args" ...
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-2}); do
  for v in "$@"; do
    IFS='|' read lab extra <<< "$v"
    name=${lab%%=*}; lib=${lab#*=}
    if [ "$lib" = default ]; then unset ASYNCEP_LIB; else export ASYNCEP_LIB=$PWD/$lib; fi
    line=$(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $BENCH_ARGS $extra 2>/dev/null | tail -1)
    echo "$name $line" >> gpurun_out/ab_libs.log
  done
done
