# Exposed AllGather (interleaved gathered - resident wall, bench.py's exposed_ag) around
# the saturation threshold T, N-rank gather emulated on one B200 at the NVLink-5 peer rate (770 GB/s).
mkdir -p gpurun_out/sweep
for T in 8192 16384 20480 24576 32768; do
  for N in 2 8; do
    timeout 400 python bench.py --emulate-gather $N --link-gbs 770 --tokens $T --steps 6 --no-cpu-baseline \
      >> gpurun_out/sweep/sweep_T_bf16.jsonl 2>> gpurun_out/sweep/err.log
  done
done
for T in 16384 24576 32768; do
  timeout 400 python bench.py --fp8 --emulate-gather 8 --link-gbs 770 --tokens $T --steps 6 --no-cpu-baseline \
    >> gpurun_out/sweep/sweep_T_fp8.jsonl 2>> gpurun_out/sweep/err.log
done
timeout 400 python bench.py --emulate-gather 4 --link-gbs 770 --steps 6 --no-cpu-baseline >> gpurun_out/sweep/sweep_T_bf16.jsonl 2>> gpurun_out/sweep/err.log
