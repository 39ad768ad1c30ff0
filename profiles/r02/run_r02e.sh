mkdir -p gpurun_out/r02e
timeout 300 python -m pytest tests/test_gpu_parity.py -k "swap_tail or fused_dispatch or tiny or router_tile" -x -q -p no:cacheprovider > gpurun_out/r02e/swap_tests.log 2>&1; echo rc=$? >> gpurun_out/r02e/swap_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02e/gputest.log 2>&1; echo rc=$? >> gpurun_out/r02e/gputest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02e/bench_swap.json 2> gpurun_out/r02e/bench_swap.err
ASYNCEP_SWAP_MAX=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02e/bench_noswap.json 2>> gpurun_out/r02e/bench_swap.err
timeout 300 python bench.py --no-cpu-baseline --tokens 16384 > gpurun_out/r02e/bench_swap_16k.json 2>> gpurun_out/r02e/bench_swap.err
ASYNCEP_SWAP_MAX=0 timeout 300 python bench.py --no-cpu-baseline --tokens 16384 > gpurun_out/r02e/bench_noswap_16k.json 2>> gpurun_out/r02e/bench_swap.err
timeout 300 python bench.py --no-cpu-baseline --fp8 > gpurun_out/r02e/bench_swap_fp8.json 2>> gpurun_out/r02e/bench_swap.err
ASYNCEP_SWAP_MAX=0 timeout 300 python bench.py --no-cpu-baseline --fp8 > gpurun_out/r02e/bench_noswap_fp8.json 2>> gpurun_out/r02e/bench_swap.err
