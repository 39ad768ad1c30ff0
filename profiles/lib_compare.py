#!/usr/bin/env python
"""Library MoE layers on the same B200, same layer, same tokens -- context for our kernels.

One Qwen3-235B-shape MoE layer (E=128, k=8, H=4096, h=1536, BF16) at 32,768 tokens, the
bench's per-layer workload.  Timed per layer (CUDA events, warm-up first):
  ours      asyncep_moe_forward through the C ABI (router + permute + GEMM1/SwiGLU + GEMM2 + combine)
  vllm      vLLM's fused MoE -- the kernels the paper's system runs (App. B): router
            logits (torch matmul) + fused_topk + fused_experts (Triton grouped GEMMs)
  grouped   torch._grouped_mm (PyTorch's CUTLASS grouped GEMM) with torch permute / combine
  flashinfer  flashinfer.fused_moe.cutlass_fused_moe (CUTLASS SM100 MoE), if it builds here
Every arm gets the same weights and tokens; outputs are cross-checked against ours
(err = max|y - y_ours| / max|y_ours|, expert part only).  Measurement only: nothing here is
on the product path, and the library arms never feed a parity claim."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from gpu_helpers import Workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=32768)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--arms", default="ours,vllm,grouped,flashinfer")
ap.add_argument("--fp8", action="store_true", help="FP8 experts (R17): ours vs vLLM fused_experts w8a8")
a = ap.parse_args()
if a.fp8:
    a.arms = ",".join(x for x in a.arms.split(",") if x in ("ours", "vllm"))
E, k, H, h, T = 128, 8, 4096, 1536, a.tokens
FLOP = 6.0 * k * H * h * T + 2.0 * H * E * T
wl = Workload(L=1, E=E, k=k, H=H, h=h, seed=0, fp8=a.fp8)
x = wl.tokens(T)
wr = wl.router(0)
if a.fp8:  # e4m3 codes + per-output-row fp32 scales
    g, u, d, gs, us, ds = wl.experts(0)
    g, u, d = (t.view(torch.float8_e4m3fn) for t in (g, u, d))
else:
    g, u, d = wl.experts(0)  # [E,h,H], [E,h,H], [E,H,h] bf16
dev = x.device


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


res = {"workload": f"one Qwen3-235B MoE layer, E={E} k={k} H={H} h={h}, {T} tokens, "
                   f"{'FP8 experts (per-row weight, per-token activation scales)' if a.fp8 else 'BF16'}, 1 B200",
       "flop_per_layer": FLOP, "arms": {}}
ref = None


def report(name, ms, y=None, note=""):
    global ref
    r = {"ms": ms, "tflops": FLOP / ms / 1e9, "note": note}
    if y is not None:
        if ref is None:
            ref = y.float()
        else:
            r["err_vs_ours"] = ((y.float() - ref).abs().max() / ref.abs().max()).item()
    res["arms"][name] = r
    print(name, json.dumps(r), flush=True)


arms = a.arms.split(",")
if "ours" in arms:
    st = wl.stack(max_tokens=T)
    y = torch.empty_like(x)
    ms = timed(lambda: st.forward(0, x, y=y), a.iters)
    st.forward(0, x, y=y)
    torch.cuda.synchronize()
    report("ours", ms, y.clone(), "asyncep_moe_forward (C ABI), all steps in our sm_100a kernels")
    del st
    torch.cuda.empty_cache()

# Timed library arms use a bf16 router linear, as vLLM's gate does; the output they are checked
# with is computed from fp32 logits (reading R3, as our router): bf16-rounded logits change the
# top-8 set of ~3 % of tokens, which alone moves the max error to ~0.2.
FP32_LOGITS = [False]
logits_fn = lambda: (torch.matmul(x.float(), wr.float().t()) if FP32_LOGITS[0] else torch.matmul(x, wr.t()).float())


def checked(fn):
    FP32_LOGITS[0] = True
    y = fn()
    FP32_LOGITS[0] = False
    return y

if "vllm" in arms:
    try:
        from vllm.model_executor.layers.fused_moe import fused_experts, fused_topk
        w1 = torch.cat([g, u], dim=1).contiguous()  # [E, 2h, H]: silu on the first half (gate)
        w2 = d.contiguous()
        qc = None
        if a.fp8:
            from vllm.model_executor.layers.fused_moe.config import fp8_w8a8_moe_quant_config
            qc = fp8_w8a8_moe_quant_config(torch.cat([gs, us], dim=1)[..., None].contiguous(), ds[..., None].contiguous(),
                                           per_act_token_quant=True, per_out_ch_quant=True)

        def vllm_layer():
            tw, ti, _ = fused_topk(x, logits_fn(), k, True)
            return fused_experts(x, w1, w2, tw, ti, quant_config=qc)
        ms = timed(vllm_layer, a.iters)
        report("vllm_fused_moe_triton", ms, checked(vllm_layer), "torch router matmul + vLLM fused_topk + fused_experts")
        del w1, w2
    except Exception as ex:  # record, do not fail the comparison
        res["arms"]["vllm_fused_moe_triton"] = {"error": f"{type(ex).__name__}: {str(ex)[:300]}"}
        print("vllm failed", ex, flush=True)
    torch.cuda.empty_cache()

if "grouped" in arms:
    try:
        wgu = torch.cat([g, u], dim=1).transpose(1, 2)      # [E, H, 2h] (K-major storage)
        wd = d.transpose(1, 2)                              # [E, h, H]

        def grouped_layer():
            lg = logits_fn()
            p = torch.softmax(lg, dim=-1)
            tw, ti = torch.topk(p, k, dim=-1)
            tw = tw / tw.sum(-1, keepdim=True)
            flat = ti.reshape(-1)
            order = torch.argsort(flat, stable=True)
            counts = torch.bincount(flat, minlength=E)
            offs = torch.cumsum(counts, 0).to(torch.int32)
            xp = x[order // k]
            gu = torch._grouped_mm(xp, wgu, offs=offs)
            act = torch.nn.functional.silu(gu[:, :h]) * gu[:, h:]
            yp = torch._grouped_mm(act, wd, offs=offs)
            out = torch.zeros_like(x, dtype=torch.float32)
            out.index_add_(0, order // k, yp.float() * tw.reshape(-1)[order, None])
            return out.to(torch.bfloat16)
        ms = timed(grouped_layer, a.iters)
        report("torch_grouped_mm", ms, checked(grouped_layer), "torch router/permute/combine + torch._grouped_mm (CUTLASS)")
        del wgu, wd
    except Exception as ex:
        res["arms"]["torch_grouped_mm"] = {"error": f"{type(ex).__name__}: {str(ex)[:300]}"}
        print("grouped failed", ex, flush=True)
    torch.cuda.empty_cache()

if "flashinfer" in arms:
    try:
        from flashinfer.fused_moe import cutlass_fused_moe
        fc1 = torch.cat([u, g], dim=1).contiguous()  # TRT-LLM Swiglu order: [up; gate]
        fc2 = d.contiguous()
        out = torch.empty_like(x)
        t0 = time.time()

        def fi_layer():
            tw, ti, _ = torch.topk(torch.softmax(logits_fn(), -1), k, dim=-1), None, None
            w_, i_ = tw
            w_ = w_ / w_.sum(-1, keepdim=True)
            return cutlass_fused_moe(x, i_.to(torch.int32), w_, fc1, fc2, torch.bfloat16, quant_scales=[], output=out)
        fi_layer()
        torch.cuda.synchronize()
        build_s = time.time() - t0
        ms = timed(fi_layer, a.iters)
        y = checked(fi_layer)
        y = y[0] if isinstance(y, (list, tuple)) else y
        report("flashinfer_cutlass_fused_moe", ms, y, f"torch router + flashinfer cutlass_fused_moe (first call {build_s:.0f} s)")
    except Exception as ex:
        res["arms"]["flashinfer_cutlass_fused_moe"] = {"error": f"{type(ex).__name__}: {str(ex)[:300]}"}
        print("flashinfer failed", ex, flush=True)

print("RESULT " + json.dumps(res))
