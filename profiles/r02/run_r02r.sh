mkdir -p gpurun_out/r02r
timeout 300 python -m pytest tests/test_gpu_asyncep.py -x -q -p no:cacheprovider > gpurun_out/r02r/asyncep_tests.log 2>&1; echo rc=$? >> gpurun_out/r02r/asyncep_tests.log
for T in 32768 16384; do
  timeout 400 python profiles/timeline.py --tokens $T > gpurun_out/r02r/timeline_bf16_$T.json 2> gpurun_out/r02r/timeline_bf16_$T.txt
done
timeout 400 python profiles/timeline.py --fp8 --tokens 32768 > gpurun_out/r02r/timeline_fp8_32768.json 2> gpurun_out/r02r/timeline_fp8_32768.txt
