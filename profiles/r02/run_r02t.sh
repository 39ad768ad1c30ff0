mkdir -p gpurun_out/r02t
timeout 300 python -m pytest tests/test_gpu_asyncep.py -q -x -p no:cacheprovider -k "graph or swap or timeline" > gpurun_out/r02t/tests.log 2>&1; echo rc=$? >> gpurun_out/r02t/tests.log
for T in 4096 8192 32768; do
  for g in "" "--graph"; do
    n=eager; [ -n "$g" ] && n=graph
    timeout 300 python bench.py --tokens $T --no-cpu-baseline $g > gpurun_out/r02t/bench_${n}_$T.json 2>> gpurun_out/r02t/err.log
  done
done
