mkdir -p gpurun_out/r02m
export ASYNCEP_LIB=$PWD/_ab/lib_wp.so
for T in 8192 32768; do
  for f in 128 64; do
    timeout 300 python profiles/prof_layer.py --iters 2 --tokens $T --flags $f > gpurun_out/r02m/wp_bf16_${T}_f$f.log 2>&1
    timeout 300 python profiles/prof_layer.py --iters 2 --tokens $T --flags $f --fp8 > gpurun_out/r02m/wp_fp8_${T}_f$f.log 2>&1
  done
done
