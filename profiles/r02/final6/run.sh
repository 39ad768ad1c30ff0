#!/bin/bash
# Validation with the materialised dispatch as the default (session 3): GPU suite, smoke, bench lines,
# HBM write-rate probe, launch lists of the bench command and ncu --set full of the GEMMs.
O=gpurun_out/final6; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 400 python bench.py --steps 20 > $O/bench_bf16.json 2> $O/bench_bf16.err
timeout 400 python bench.py --steps 20 --fp8 > $O/bench_fp8.json 2> $O/bench_fp8.err
timeout 120 python -c "
import torch, json
t = torch.empty(2 * 1024**3 // 2, dtype=torch.bfloat16, device='cuda'); s = torch.empty_like(t)
for name, fn in (('write', lambda: t.fill_(1.0)), ('copy', lambda: t.copy_(s))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    b = t.numel() * 2 * (1 if name == 'write' else 2)
    print(json.dumps({'op': name, 'bytes': b, 'ms': ms, 'gbs': b / ms / 1e6}))
" > $O/hbm_write_probe.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/launches_bf16.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/launches_fp8.csv \
  python bench.py --fp8 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 3 -f \
  -o $O/gemm_full_bf16 python profiles/prof_layer.py --iters 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 3 -f \
  -o $O/gemm_full_fp8 python profiles/prof_layer.py --iters 2 --fp8 > /dev/null 2>&1
tail -3 $O/pytest_gpu.log
