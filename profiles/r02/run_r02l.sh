mkdir -p gpurun_out/r02l
for g in 770 500 400; do
  timeout 600 python profiles/gather_interference.py --fp8 --ctas 148 --link-gbs $g --pairs 12 >> gpurun_out/r02l/pace_fp8_32k.jsonl 2>> gpurun_out/r02l/err.log
  timeout 600 python profiles/gather_interference.py --ctas 148 --link-gbs $g --pairs 12 >> gpurun_out/r02l/pace_bf16_32k.jsonl 2>> gpurun_out/r02l/err.log
done
