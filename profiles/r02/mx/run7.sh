set -x
timeout 600 python profiles/ab_flags.py --tokens 32768 --flags-a 0 --flags-b 0 --pairs 8 > gpurun_out/ab7_bf16_same.json 2>> gpurun_out/ab7.err
timeout 600 python profiles/ab_flags.py --tokens 32768 --flags-a 0 --flags-b 0 --pairs 8 --reverse-create > gpurun_out/ab7_bf16_same_rev.json 2>> gpurun_out/ab7.err
timeout 600 python profiles/ab_flags.py --fp8 --tokens 16384 --flags-a 0 --flags-b 0 --pairs 8 > gpurun_out/ab7_fp8_same.json 2>> gpurun_out/ab7.err
timeout 600 python profiles/ab_flags.py --fp8 --tokens 16384 --flags-a 0 --flags-b 0 --pairs 8 --reverse-create > gpurun_out/ab7_fp8_same_rev.json 2>> gpurun_out/ab7.err
