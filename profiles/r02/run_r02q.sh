mkdir -p gpurun_out/r02q
for th in 128 32 64 128; do
  ASYNCEP_GATHER_THREADS=$th timeout 600 python profiles/gather_interference.py --ctas 148 --pairs 12 > gpurun_out/r02q/bf16_t$th.jsonl 2>> gpurun_out/r02q/err.log
  ASYNCEP_GATHER_THREADS=$th timeout 600 python profiles/gather_interference.py --fp8 --ctas 148 --pairs 12 > gpurun_out/r02q/fp8_t$th.jsonl 2>> gpurun_out/r02q/err.log
done
