mkdir -p gpurun_out/r02f
for cfg in "240 0" "240 128" "240 240" "0 0"; do set -- $cfg
  ASYNCEP_SWAP_MAX=$1 ASYNCEP_SWAP_MAX_F8G2=$2 timeout 300 python bench.py --no-cpu-baseline --fp8 > gpurun_out/r02f/fp8_$1_$2.json 2>> gpurun_out/r02f/err.log
done
for m in 240 160 96 0 240; do
  ASYNCEP_SWAP_MAX=$m timeout 300 python bench.py --no-cpu-baseline --tokens 16384 > gpurun_out/r02f/bf16_16k_$m.json 2>> gpurun_out/r02f/err.log
done
for m in 240 160 0 240; do
  ASYNCEP_SWAP_MAX=$m timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02f/bf16_32k_$m.json 2>> gpurun_out/r02f/err.log
done
