mkdir -p gpurun_out/r02y
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -q -x -p no:cacheprovider -k "router or tiny or tcgen05 or deterministic or 30b or zipf or fp8_layer" > gpurun_out/r02y/t.log 2>&1; echo rc=$? >> gpurun_out/r02y/t.log
for r in 1 0 1 0; do
  ASYNCEP_ROUTER_SWAP=$r timeout 300 python bench.py --no-cpu-baseline --steps 6 > gpurun_out/r02y/bench_rs$r.json 2>> gpurun_out/r02y/err.log
  cat gpurun_out/r02y/bench_rs$r.json >> gpurun_out/r02y/all.jsonl
done
M=gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second
for r in 1 0; do
  ASYNCEP_ROUTER_SWAP=$r timeout 300 ncu --metrics $M --clock-control none --kernel-name-base demangled -k 'regex:router_swap|gemm_tc_kernel<\(int\)2' -s 1 -c 1 --csv --log-file gpurun_out/r02y/router_rs$r.csv python profiles/prof_layer.py --iters 2 > /dev/null 2>&1
done
