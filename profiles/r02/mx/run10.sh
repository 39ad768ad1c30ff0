# new scatter / quant kernels: BF16 and FP8 fused vs materialised, both orders; then the FP8/BF16 GPU tests touched
for T in 32768; do
timeout 600 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 0x200 --flags-b 0 --pairs 8 > gpurun_out/ab10_fp8_$T.json 2>> gpurun_out/ab10.err
timeout 600 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 0 --flags-b 0x200 --pairs 8 > gpurun_out/ab10_fp8_rev_$T.json 2>> gpurun_out/ab10.err
timeout 600 python profiles/ab_flags.py --tokens $T --flags-a 0 --flags-b 16 --pairs 8 > gpurun_out/ab10_bf16_$T.json 2>> gpurun_out/ab10.err
timeout 600 python profiles/ab_flags.py --tokens $T --flags-a 16 --flags-b 0 --pairs 8 > gpurun_out/ab10_bf16_rev_$T.json 2>> gpurun_out/ab10.err
done
timeout 600 python profiles/ab_flags.py --tokens 16384 --flags-a 0 --flags-b 16 --pairs 8 > gpurun_out/ab10_bf16_16384.json 2>> gpurun_out/ab10.err
timeout 600 python profiles/ab_flags.py --tokens 16384 --flags-a 16 --flags-b 0 --pairs 8 > gpurun_out/ab10_bf16_rev_16384.json 2>> gpurun_out/ab10.err
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_mx.py tests/test_gpu_parity.py -q -x > gpurun_out/ab10_tests.log 2>&1; tail -2 gpurun_out/ab10_tests.log
