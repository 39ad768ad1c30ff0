mkdir -p gpurun_out/r02k
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -x -q -p no:cacheprovider -k "not eight_layer and not 235b and not zipf" > gpurun_out/r02k/quick.log 2>&1; echo rc=$? >> gpurun_out/r02k/quick.log
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2605_02960_b200/csrc -o /tmp/probe_mma_n profiles/probe_mma_n.cu && timeout 120 /tmp/probe_mma_n > gpurun_out/r02k/probe_mma_n.jsonl 2>&1
bash profiles/r02/run_sweep_T.sh
