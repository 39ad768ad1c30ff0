set -x
mkdir -p gpurun_out/r02c
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/r02c/gputest.log 2>&1; echo rc=$? >> gpurun_out/r02c/gputest.log
timeout 900 python profiles/gather_interference.py --ctas 296,148,74,37 --pairs 8 > gpurun_out/r02c/interf_bf16.jsonl 2> gpurun_out/r02c/interf_bf16.err
timeout 900 python profiles/gather_interference.py --fp8 --ctas 296,148,74 --pairs 8 > gpurun_out/r02c/interf_fp8.jsonl 2> gpurun_out/r02c/interf_fp8.err
