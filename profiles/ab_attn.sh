for r in 1 2; do for v in default _ab/lib_poly0.so _ab/lib_poly2.so _ab/lib_poly8.so; do
  if [ $v = default ]; then unset ASYNCEP_LIB; else export ASYNCEP_LIB=$PWD/$v; fi
  for p in 4096 32768; do echo "$v $(timeout 120 python profiles/prof_attn.py --prompt $p 2>&1 | tail -1)" >> gpurun_out/ab_attn.log; done
done; done
