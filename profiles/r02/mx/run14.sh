# swap-AB tails in both GEMMs (FLAG_SWAP_TAILS) vs the default, with the TMA-fed A (materialised dispatch)
mkdir -p gpurun_out/r14
for f in "" "--fp8"; do
  tag=bf16; [ -n "$f" ] && tag=fp8
  for T in 32768 16384; do
    timeout 400 python profiles/ab_flags.py $f --tokens $T --flags-a 0 --flags-b 0x80 --pairs 6 > gpurun_out/r14/${tag}_$T.json 2>> gpurun_out/r14/ab.err
    timeout 400 python profiles/ab_flags.py $f --tokens $T --flags-a 0x80 --flags-b 0 --pairs 6 > gpurun_out/r14/${tag}_rev_$T.json 2>> gpurun_out/r14/ab.err
  done
done
