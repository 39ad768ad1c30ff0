set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests/test_gpu_mx.py -x -q -s > gpurun_out/mx_tests.log 2>&1; echo "rc=$?" >> gpurun_out/mx_tests.log
tail -5 gpurun_out/mx_tests.log
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_parity.py -x -q > gpurun_out/regr.log 2>&1; echo "rc=$?" >> gpurun_out/regr.log
tail -3 gpurun_out/regr.log
timeout 600 python profiles/ab_flags.py --fp8 --flags-a 0 --flags-b 0x100 --pairs 8 > gpurun_out/ab_mx_32k.json 2> gpurun_out/ab_mx_32k.err
tail -5 gpurun_out/ab_mx_32k.json
