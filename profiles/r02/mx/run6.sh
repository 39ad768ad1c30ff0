set -x
for T in 32768 16384; do
timeout 600 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 0x100 --flags-b 0x100 --pairs 8 > gpurun_out/ab6_same_$T.json 2>> gpurun_out/ab6.err
timeout 600 python profiles/ab_flags.py --fp8 --tokens $T --flags-a 0 --flags-b 0x100 --pairs 10 > gpurun_out/ab6_mx_$T.json 2>> gpurun_out/ab6.err
done
