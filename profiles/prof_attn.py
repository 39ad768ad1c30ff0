#!/usr/bin/env python
"""NEXT-3 attention layer at the Qwen3-235B shape (H=4096, Hq=64, Hkv=4, d=128) on
--tokens tokens packed as prompts of --prompt tokens: times the whole layer with CUDA events
and the attention core alone, and prints one JSON line (tokens/s, TFLOP/s of the core
against its algorithmic causal FLOPs).  Also the light driver for ncu captures."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_02960_b200 import asyncep as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=32768)
ap.add_argument("--prompt", type=int, default=4096)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--H", type=int, default=4096)
ap.add_argument("--Hq", type=int, default=64)
ap.add_argument("--Hkv", type=int, default=4)
a = ap.parse_args()
d = 128
lengths = synth.prompt_lengths(a.tokens, a.prompt, 0, spread=0.0)
cu = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)
T = int(cu[-1])
cu_d = torch.from_numpy(cu).cuda()
w = synth.attn_weights(a.H, a.Hq, a.Hkv, d, 0, 0, device="cuda")
x = synth.tokens(T, a.H, 1, device="cuda")
cfg = A.make_attn_config(a.H, a.Hq, a.Hkv, d, max_tokens=T, max_prompts=len(lengths))
ws = torch.empty(A.asyncep_attn_workspace_size(cfg), dtype=torch.uint8, device="cuda")
xo, xn = torch.empty_like(x), torch.empty_like(x)

# attention core inputs (synthetic q/k/v of the same shape)
q = synth.normal((T, a.Hq, d), 0, 0xA1, 1.0, "cuda")
k = synth.normal((T, a.Hkv, d), 0, 0xA2, 1.0, "cuda")
vcu = np.concatenate([[0], np.cumsum([(n + 7) // 8 * 8 for n in lengths])]).astype(np.int32)
ldv = int(vcu[-1]) + 8
vt = synth.normal((a.Hkv, d, ldv), 0, 0xA3, 1.0, "cuda")
o = torch.empty_like(q)
vcu_d = torch.from_numpy(vcu).cuda()


def timed(fn):
    for _ in range(a.warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.iters


ms_layer = timed(lambda: A.asyncep_attn_layer(cfg, x, cu_d, w, xo, xn, ws))
ms_core = timed(lambda: A.asyncep_attention(cfg, q, k, vt, ldv, vcu_d, cu_d, o))
pairs = sum(n * (n + 1) // 2 for n in lengths)            # causal (query, key) pairs
core_flops = 4.0 * d * a.Hq * pairs                        # QK^T + PV, 2 d FLOPs each per pair
proj_flops = 2.0 * T * a.H * ((a.Hq + 2 * a.Hkv) * d + a.Hq * d)
print(json.dumps({
    "tokens": T, "prompts": len(lengths), "prompt_len": a.prompt,
    "layer_ms": ms_layer, "layer_tokens_per_s": T / ms_layer * 1e3,
    "layer_tflops": (core_flops + proj_flops) / ms_layer / 1e9,
    "core_ms": ms_core, "core_tflops": core_flops / ms_core / 1e9,
    "core_flops": core_flops, "proj_flops": proj_flops,
}))
