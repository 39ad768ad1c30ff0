#!/usr/bin/env python
"""Library (cuBLAS via torch) dense GEMM rates on this B200 with the SM clock sampled during the
timed loop: bf16 (torch.matmul) and e4m3 (torch._scaled_mm, per-tensor scales), square 8192^3 and
the grouped GEMM1's flat shape (M = 262,144 permuted rows, N = 3,072, K = 4,096).  Context for the
roofline: FLOP per clock per SM of the vendor GEMM (the practical per-clock ceiling), not a product
path.  python profiles/cublas_peaks.py > gpurun_out/cublas_peaks.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402

dev = torch.device("cuda", 0)
sms = torch.cuda.get_device_properties(dev).multi_processor_count


def rate(fn, flops, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ck = ClockSampler(0, period=0.005).start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    clk = ck.stop()
    s = e0.elapsed_time(e1) / 1e3 / iters
    mhz = clk.get("sm_mhz") or 0
    return {"tflops": flops / s / 1e12, "ms": s * 1e3, "sm_mhz": mhz, "reasons": clk.get("reasons"),
            "flop_per_clk_per_sm": flops / s / (mhz * 1e6) / sms if mhz else None}


for (M, N, K, tag) in ((8192, 8192, 8192, "square"), (262144, 3072, 4096, "gemm1_flat")):
    a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    b = torch.randn(N, K, device=dev, dtype=torch.bfloat16)
    flops = 2.0 * M * N * K
    iters = max(20, int(3e15 / flops))  # ~2 s per dtype: enough clock samples
    r = rate(lambda: torch.matmul(a, b.t()), flops, iters)
    print(json.dumps({"dtype": "bf16", "shape": tag, "M": M, "N": N, "K": K, **r}), flush=True)
    a8, b8 = a.to(torch.float8_e4m3fn), b.to(torch.float8_e4m3fn)
    one = torch.ones((), device=dev)
    try:
        r = rate(lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16), flops,
                 iters * 2)
        print(json.dumps({"dtype": "e4m3", "shape": tag, "M": M, "N": N, "K": K, **r}), flush=True)
    except Exception as ex:  # noqa: BLE001
        print(json.dumps({"dtype": "e4m3", "shape": tag, "error": str(ex)[:200]}), flush=True)
    del a, b, a8, b8
    torch.cuda.empty_cache()
