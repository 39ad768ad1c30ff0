mkdir -p gpurun_out/r02w
for T in 8192 24576; do
  timeout 600 python bench.py --attn --emulate-gather 8 --link-gbs 770 --tokens $T --no-cpu-baseline >> gpurun_out/r02w/sweep_T_attn.jsonl 2>> gpurun_out/r02w/err.log
done
timeout 600 python bench.py --offload 2 --emulate-gather 8 --link-gbs 770 --no-cpu-baseline --no-ab > gpurun_out/r02w/bench_offload_w2_emu8.json 2>> gpurun_out/r02w/err.log
timeout 600 python bench.py --emulate-gather 8 --link-gbs 770 --tokens 16384 --no-cpu-baseline > gpurun_out/r02w/bench_emu8_16k_calib.json 2>> gpurun_out/r02w/err.log
