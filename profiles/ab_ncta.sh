rm -f gpurun_out/ab_ncta.log
for r in 1 2; do
 for n in 2 1; do for a in "" "--xperm"; do
  echo "ncta$n$a $(ASYNCEP_GEMM_NCTA=$n timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --layers 4 $a 2>/dev/null | tail -1)" >> gpurun_out/ab_ncta.log
 done; done
done
