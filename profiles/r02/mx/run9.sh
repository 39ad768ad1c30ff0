for T in 32768 16384; do
timeout 600 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 0 --flags-b 16 --pairs 8 > gpurun_out/ab9_fp8_xperm_$T.json 2>> gpurun_out/ab9.err
timeout 600 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 16 --flags-b 0 --pairs 8 > gpurun_out/ab9_fp8_xperm_rev_$T.json 2>> gpurun_out/ab9.err
done
timeout 600 python profiles/ab_flags.py --tokens 32768 --flags-a 0 --flags-b 16 --pairs 8 > gpurun_out/ab9_bf16_xperm_32768.json 2>> gpurun_out/ab9.err
timeout 600 python profiles/ab_flags.py --tokens 32768 --flags-a 16 --flags-b 0 --pairs 8 > gpurun_out/ab9_bf16_xperm_rev_32768.json 2>> gpurun_out/ab9.err
