mkdir -p gpurun_out/r02d
timeout 600 python profiles/gather_interference.py --ctas 148,96,296,148 --pairs 12 > gpurun_out/r02d/interf_bf16_p0.jsonl 2> gpurun_out/r02d/e1.err
timeout 600 python profiles/gather_interference.py --prio -1 --ctas 148,96,296,148 --pairs 12 > gpurun_out/r02d/interf_bf16_pm1.jsonl 2> gpurun_out/r02d/e2.err
timeout 600 python profiles/gather_interference.py --fp8 --prio -1 --ctas 148,296,148 --pairs 12 > gpurun_out/r02d/interf_fp8_pm1.jsonl 2> gpurun_out/r02d/e3.err
timeout 600 python profiles/gather_interference.py --fp8 --ctas 148,296,148 --pairs 12 > gpurun_out/r02d/interf_fp8_p0.jsonl 2> gpurun_out/r02d/e4.err
