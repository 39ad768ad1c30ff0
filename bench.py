#!/usr/bin/env python
"""Benchmark: AsyncEP MoE-layer stack forward on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[2], the metric's config): Qwen3-235B-A22B MoE-layer
shape -- E=128 experts, top-8, H=4096, expert FFN h=1536 -- BF16, an 8-layer stack with
residual chaining (reading R9), 32,768 tokens per GPU (weak scaling: per-GPU work fixed).
One "step" = one pass of the whole hot path (router -> permute -> grouped GEMM with
SwiGLU -> combine) through all 8 layers over one batch of synthetic tokens.

  N = 1  : all layers resident (world_size 1, no gather).
  N > 1  : one process per GPU (torchrun), experts of layers >= 1 sharded 1/N by expert
           index, layer 0 replicated, NCCL AllGather of layer l+1 on a side stream while
           layer l computes.  No data-path collective.

Timing: W warm-up steps, then K steps bracketed by barrier + cuda synchronize, CUDA
events on the compute stream, max over ranks.  Inputs are larger than L2 (38.7 GB of
weights, 268 MB of activations per layer), so no explicit L2 flush.

--impl reference: the CPU oracle (oracle/, plain fp64 C) on the host cores, on a bounded
sample of the same workload (see cpu_baseline.sample in the JSON line).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s and MFU per B200, Qwen3-235B MoE layers, 1/2/4/8 GPUs; exposed AG time"
L_, E_, K_, H_, h_ = 8, 128, 8, 4096, 1536
T_LOC = 32768
FLOPS_TOK_LAYER = 2 * H_ * E_ + 6 * K_ * H_ * h_          # 303,038,464 (router + experts)
ATT_HQ, ATT_HKV = 64, 4                                    # Qwen3-235B-A22B attention (NEXT-3, R19)
COMBINE_BYTES_TOK = K_ * H_ * 2 + 2 * H_ * 2               # read k rows + residual, write y
GEMM1_FLOPS_TOK = 4 * K_ * H_ * h_                        # gate/up: 2 * k * H * 2h
GEMM2_FLOPS_TOK = 2 * K_ * H_ * h_
SPEC_BF16 = 2.25e15


def set_shape(name: str) -> None:
    """--shape 30b: BASELINE config 2 (Qwen3-30B-A3B MoE layer, H=2048, h=768, one layer,
    16K tokens, no sharding) instead of the headline Qwen3-235B stack."""
    global L_, H_, h_, T_LOC, FLOPS_TOK_LAYER, COMBINE_BYTES_TOK, GEMM1_FLOPS_TOK, GEMM2_FLOPS_TOK, ATT_HQ, ATT_HKV
    if name == "30b":
        L_, H_, h_, T_LOC = 1, 2048, 768, 16384
        ATT_HQ, ATT_HKV = 32, 4
    FLOPS_TOK_LAYER = 2 * H_ * E_ + 6 * K_ * H_ * h_
    COMBINE_BYTES_TOK = K_ * H_ * 2 + 2 * H_ * 2
    GEMM1_FLOPS_TOK = 4 * K_ * H_ * h_
    GEMM2_FLOPS_TOK = 2 * K_ * H_ * h_


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    def __init__(self, dev_index: int, period=0.1):
        self.dev_index, self.period = dev_index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
                "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
                "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for n, b in names.items():
                            if r & b and n != "gpu_idle":
                                self.reasons.add(n)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def ncu_traffic(fp8: bool = False):
    """DRAM bytes per launch of the dominant kernel (GEMM1) from the committed ncu
    --set full summary of the current kernel (profiles/r*/gemm_ncu_full*.json)."""
    import glob
    name = "gemm_ncu_full_fp8.json" if fp8 else "gemm_ncu_full.json"
    cands = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", name)))
    if not cands:
        return None
    try:
        for d in json.load(open(cands[-1])):
            if "<1," in d.get("kernel", ""):
                return {"bytes_per_launch": d.get("dram_bytes_per_launch"),
                        "source": os.path.relpath(cands[-1], ROOT),
                        "note": "ncu --set full, one launch (cold L2)"}
    except Exception:
        return None
    return None


# ------------------------------------------------------------------------------ oracle arm
class OracleSample:
    """The CPU oracle on a bounded sample of the workload: n_tokens through one of the
    Qwen3-235B-shape layers (the per-layer cost is identical for every layer)."""

    def __init__(self, layer: int = 0, seed: int = 0):
        import torch

        import oracle
        import synth
        dev = "cuda" if torch.cuda.is_available() else "cpu"  # synth is bit-identical on both
        self.dev, self.seed = dev, seed
        self.wr = synth.router_weight(E_, H_, seed, layer, device=dev).float().cpu().numpy()
        g, u, d = synth.expert_weights(E_, H_, h_, seed, layer, device=dev)
        self.g, self.u, self.d = (t.float().cpu().numpy() for t in (g, u, d))
        del g, u, d
        oracle.build()
        self.threads = oracle.num_threads()

    def run(self, n_tokens: int, sample: int = 0):
        import oracle
        import synth
        x = synth.tokens(n_tokens, H_, self.seed + 1000 + sample, device=self.dev).float().cpu().numpy()
        t0 = time.perf_counter()
        oracle.moe_layer(x, self.wr, self.g, self.u, self.d, K_)
        dt = time.perf_counter() - t0
        desc = (f"{n_tokens} tokens through 1 of the {L_} Qwen3-235B-shape layers (fp64 C oracle, "
                f"{self.threads} threads); stack tokens/s = layer tokens/s / {L_}")
        return n_tokens / dt / L_, dt, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n_tok = int(os.environ.get("ASYNCEP_REF_TOKENS", "256"))
    orc = OracleSample()
    vals = []
    desc = ""
    for i in range(args.warmup + args.steps):
        v, dt, desc = orc.run(n_tok, sample=i)
        if i >= args.warmup:
            vals.append((v, dt))
    dt_tot = sum(b for _, b in vals)
    v = n_tok * len(vals) / dt_tot / L_
    ms = dt_tot / len(vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "qwen3-235b-a22b moe-layer stack (E=128,k=8,H=4096,h=1536), 8 layers, "
                               f"bounded sample of {n_tok} tokens per step",
                   "tokens_per_gpu": T_LOC, "layers": L_},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": orc.threads, "kind": "oracle", "sample": desc},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU arm
def main():
    pre = argparse.ArgumentParser(add_help=False)
    pre.add_argument("--shape", choices=["235b", "30b"], default="235b")
    set_shape(pre.parse_known_args()[0].shape)
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", choices=["235b", "30b"], default="235b",
                    help="235b: headline Qwen3-235B 8-layer stack (config 3/4); 30b: Qwen3-30B layer (config 2)")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tokens", type=int, default=T_LOC, help="tokens per GPU")
    ap.add_argument("--replicate-layer0", type=int, default=1)
    ap.add_argument("--layers", type=int, default=L_)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--simt", action="store_true", help="CUDA-core GEMM (debug)")
    ap.add_argument("--xperm", action="store_true", help="materialise X_perm (unfused dispatch, FLAG_XPERM)")
    ap.add_argument("--emulate-gather", type=int, default=0, metavar="N",
                    help="1-GPU emulation of the N-rank AsyncEP gather (D2D copies of all N shards into "
                         "the slot on the comm stream); measures exposed wait + HBM interference")
    ap.add_argument("--link-gbs", type=float, default=0.0,
                    help="with --emulate-gather: pace the peer-shard copies at this GB/s (NVLink receive "
                         "bandwidth; B200_PROFILING.md measured peer copy: 770)")
    ap.add_argument("--gather", choices=["p2p", "nccl"], default="p2p",
                    help="N>1: the weight gather over NVLink copy engines on CUDA-IPC-mapped peer shards "
                         "(default; leaves every SM to the persistent GEMMs) or ncclAllGather")
    ap.add_argument("--ep", action="store_true",
                    help="contrast baseline: the same stack as synchronous DP x EP (two on-path AllToAlls "
                         "per layer, PAPER.md:196-199) instead of AsyncEP")
    ap.add_argument("--offload", type=int, default=0, metavar="W",
                    help="NEXT-2: expert shards in pinned host memory, a W-deep device window filled over PCIe")
    ap.add_argument("--zipf", type=float, default=0.0, metavar="S",
                    help="Zipf-skewed routing (reading R14, BASELINE config 5 uses S=0.35)")
    ap.add_argument("--attn", action="store_true",
                    help="NEXT-3: decoder layers = DP attention (KV-cache-free, Qwen3-235B heads) + MoE; the "
                         "gather of layer l+1 overlaps both")
    ap.add_argument("--prompt", type=int, default=4096,
                    help="prompt length of the packed batch with --attn (tokens/GPU split into prompts)")
    ap.add_argument("--fp8", action="store_true",
                    help="FP8 e4m3 experts (BASELINE config 4) instead of BF16 (config 3)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import synth
    from paper_2605_02960_b200 import asyncep as A
    from paper_2605_02960_b200.stack import MoEStack

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    # Test hooks for running N ranks on ONE GPU (NCCL refuses that): ASYNCEP_BENCH_DEVICE pins every
    # rank to one device, ASYNCEP_BENCH_BACKEND=gloo runs the control plane (barrier, max-over-ranks)
    # on gloo; the gather then must be the peer-copy transport (CUDA IPC works within one GPU).
    backend = os.environ.get("ASYNCEP_BENCH_BACKEND", "nccl")
    dev_idx = int(os.environ.get("ASYNCEP_BENCH_DEVICE", local))
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    comm = None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
            dist.all_reduce(torch.ones(1, device=dev))  # eager comm init
            comm = A.nccl_comm_ptr()
        else:
            dist.init_process_group(backend)
            if args.gather == "nccl" or args.ep:
                raise SystemExit("--gather nccl / --ep need the NCCL backend")
    L, T = args.layers, args.tokens
    seed = 0
    flags = A.FLAG_STAGE_TIMING | (A.FLAG_SIMT_GEMM if args.simt else 0) | (A.FLAG_XPERM if args.xperm else 0)
    gen = synth.expert_weights_fp8 if args.fp8 else synth.expert_weights
    if world > 1 and args.gather == "nccl":  # NCCL's SM-based AllGather needs SMs the GEMMs leave free
        os.environ.setdefault("ASYNCEP_RESERVE_SMS", "16")
    emu = args.emulate_gather if world == 1 else 0
    stack = MoEStack(L, E_, K_, H_, h_, T,
                     lambda l: synth.router_weight(E_, H_, seed, l, device=dev, zipf_s=args.zipf),
                     lambda l, ex: gen(E_, H_, h_, seed, l, device=dev, experts=ex),
                     world_size=emu or world, rank=rank, replicate_layer0=True, flags=flags, device=dev,
                     nccl_comm=comm, fp8=args.fp8, offload_window=args.offload)
    local_shards = stack.peer_shards() if emu > 1 else None
    gather_mode = "emulated" if emu > 1 else ("none" if world == 1 else args.gather)
    if world > 1 and args.gather == "p2p" and not args.ep:
        try:
            stack.enable_p2p_gather()
        except Exception as e:  # fall back to NCCL (recorded in the JSON line)
            gather_mode = f"nccl (p2p setup failed: {type(e).__name__}: {str(e)[:120]})"
            A.asyncep_set_peer_shards(stack.ctx, None)
    cu = None
    attn_flops_layer = 0.0
    if args.attn:
        lengths = synth.prompt_lengths(T, args.prompt, seed, spread=0.0)
        cu = torch.tensor([0] + list(np.cumsum(lengths)), dtype=torch.int32, device=dev)
        stack.enable_attention(lambda l: synth.attn_weights(H_, ATT_HQ, ATT_HKV, 128, seed, l, device=dev),
                               ATT_HQ, ATT_HKV, max_prompts=len(lengths))
        pairs = sum(n * (n + 1) // 2 for n in lengths)
        attn_flops_layer = 4.0 * 128 * ATT_HQ * pairs + 2.0 * T * H_ * ((ATT_HQ + 2 * ATT_HKV) * 128 + ATT_HQ * 128)
    if args.ep:  # contrast layer: every rank keeps its shard; tokens travel instead of weights
        _run = lambda xin, out: stack.run_ep(xin, out=out)
    else:
        _run = lambda xin, out: stack.run(xin, out=out, local_shards=local_shards, cu_seqlens=cu)
    if emu > 1 and args.link_gbs > 0:
        A.asyncep_set_link_emulation(stack.ctx, args.link_gbs * 1e9)
    # tokens: DP -- every rank its own batch
    x = synth.tokens(T, H_, seed + 17 + rank, device=dev, zipf_s=args.zipf)
    out = torch.empty_like(x)
    cs = stack.compute_stream

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[dev_idx])
            else:
                dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for _ in range(args.warmup):
        _run(x, out)
    barrier()
    A.asyncep_reset_stage_times(stack.ctx)
    launches0 = A.asyncep_kernel_launches(stack.ctx)
    clocks = ClockSampler(dev_idx).start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(cs)
    for _ in range(args.steps):
        _run(x, out)
    e1.record(cs)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    launches = A.asyncep_kernel_launches(stack.ctx) - launches0
    stages, nfwd = A.asyncep_stage_times(stack.ctx)
    ms_max = max_over_ranks(ms)
    ms_step = ms_max / args.steps
    value = world * T * args.steps / (ms_max / 1e3)     # whole-job tokens/s
    per_gpu = value / world
    mfu_flops = per_gpu * L * FLOPS_TOK_LAYER + (per_gpu / T) * L * attn_flops_layer

    # ---------------- e2e: public API with host buffers (pinned), copies in the timed region.
    # A serving pipeline: step i+1's input is copied host->device on one copy stream while step i
    # computes, and step i's output goes device->host on another (double-buffered both ways).
    xh = x.cpu().pin_memory()
    yh = [torch.empty_like(xh).pin_memory() for _ in range(2)]
    xd = [torch.empty_like(x) for _ in range(2)]
    od = [torch.empty_like(x) for _ in range(2)]
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def e2e_steps(n):
        with torch.cuda.stream(h2d):
            xd[0].copy_(xh, non_blocking=True)
            ev_in[0].record(h2d)
        for i in range(n):
            b = i % 2
            cs.wait_event(ev_in[b])
            if i >= 2:
                cs.wait_event(ev_out[b])         # od[b] of step i-2 has been read back
            _run(xd[b], od[b])
            ev_done[b].record(cs)
            if i + 1 < n:                         # prefetch the next step's input
                with torch.cuda.stream(h2d):
                    if i >= 1:
                        h2d.wait_event(ev_done[1 - b])   # step i-1 has finished reading xd[1-b]
                    xd[1 - b].copy_(xh, non_blocking=True)
                    ev_in[1 - b].record(h2d)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_done[b])
                yh[b].copy_(od[b], non_blocking=True)
                ev_out[b].record(d2h)
        cs.wait_event(ev_out[(n - 1) % 2])

    e2e_steps(2)
    barrier()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(cs)
    h2d.wait_event(f0)
    e2e_steps(args.steps)
    f1.record(cs)
    barrier()
    e2e_value = world * T * args.steps / (max_over_ranks(f0.elapsed_time(f1)) / 1e3)

    attn_info = None
    if args.attn:  # attention half alone (outside the timed region), for the layer breakdown
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        stack.attention(0, x, cu)
        barrier()
        a0.record(cs)
        for l in range(L):
            stack.attention(l, x, cu)
        a1.record(cs)
        barrier()
        a_ms = a0.elapsed_time(a1) / L
        attn_info = {"ms_per_layer": a_ms, "prompt_len": args.prompt, "prompts": int(cu.numel() - 1),
                     "q_heads": ATT_HQ, "kv_heads": ATT_HKV, "head_dim": 128,
                     "flops_per_layer": attn_flops_layer, "tflops": attn_flops_layer / (a_ms / 1e3) / 1e12,
                     "note": "RMSNorm + QKV GEMM + QK-norm/RoPE + causal flash attention + O GEMM + "
                             "residual/RMSNorm (reading R19); timed separately, included in the step"}

    peaks, peak_src = load_peaks()
    # dominant kernel: GEMM1 (gate/up + SwiGLU), stage-timed with CUDA events on the
    # compute stream around each launch inside the timed region
    g1_ms = stages["gemm1_gateup_swiglu"] / max(nfwd, 1)
    g1_flops = GEMM1_FLOPS_TOK * T
    g1_tflops = g1_flops / (g1_ms / 1e3) / 1e12 if g1_ms > 0 else 0.0  # 0: no stage events (--ep)
    peak_tf = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    peak_note = f"{peak_src} bf16_tflops_sustained (kernel timed inside a long step)"
    spec = SPEC_BF16
    if args.fp8:  # FP8 contraction: the bf16 measured peak x the nominal fp8/bf16 ratio (2x)
        peak_tf *= 2.0
        spec *= 2.0
        peak_note = f"{peak_src} bf16_tflops_sustained x 2 (nominal fp8:bf16 dense ratio)"
    traffic = ncu_traffic(args.fp8)
    per_layer_ms = {k: v / max(nfwd, 1) for k, v in stages.items()}
    # Eq. 1 (R11/R12): T in tokens/GPU with F = this run's grouped-GEMM
    # rate and the gather bandwidth of NVLink 5 (measured peer copy 770 GB/s, B200_PROFILING.md)
    gemm_ms = per_layer_ms["gemm1_gateup_swiglu"] + per_layer_ms["gemm2_down"]
    f_gemm = (GEMM1_FLOPS_TOK + GEMM2_FLOPS_TOK) * T / (gemm_ms / 1e3) if gemm_ms > 0 else 0.0
    n_for_T = world if world > 1 else (emu if emu > 1 else 8)
    bw = (args.link_gbs or 770.0) * 1e9
    tcfg = A.make_config(L, E_, K_, H_, h_, expert_dtype=A.FP8_E4M3 if args.fp8 else A.BF16,
                         world_size=n_for_T, max_tokens=T, gamma=1.2)
    t_tok, t_flops = A.asyncep_saturation_T(tcfg, f_gemm, bw) if f_gemm > 0 else (None, None)
    step_layer_ms = ms_step / L
    model = "qwen3-30b-a3b (config 2)" if args.shape == "30b" else "qwen3-235b-a22b"
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp8_e4m3" if args.fp8 else "bf16", "data": "synthetic",
        "config": {"workload": (f"{model} decoder-layer stack (DP attention Hq=64 Hkv=4 d=128, KV-cache-free, "
                                f"{args.prompt}-token prompts + MoE), " if args.attn else
                                f"{model} moe-layer stack, ") + f"{L} layers, E=128 k=8 H={H_} h={h_}, "
                               f"{T} tokens/GPU, {'FP8 e4m3 experts (bf16 router/activations)' if args.fp8 else 'BF16'}, "
                               "random-init weights" + (f", Zipf-skewed routing s={args.zipf} (R14)" if args.zipf else ""),
                   "tokens_per_gpu": T, "layers": L, "global_batch_tokens": T * world,
                   "parallelism": (f"dp{world}xep{world} contrast (2 on-path AllToAlls/layer)" if args.ep else
                                   f"dp{world}+asyncep{world}" if world > 1 else
                                   f"dp1, asyncep{emu} gather emulated on 1 GPU (D2D copies of the {emu} shards "
                                   "into the slot on the comm stream" +
                                   (f", peer shards paced at {args.link_gbs} GB/s" if args.link_gbs else "") + ")"
                                   if emu > 1 else "dp1 (all experts resident)") +
                                  (f", shards offloaded to pinned host memory, {args.offload}-deep device window "
                                   "(NEXT-2)" if args.offload else ""),
                   "gather": gather_mode,
                   "l2": (f"inputs larger than L2 ({L * E_ * 3 * H_ * h_ * (1 if args.fp8 else 2) / 1e9:.1f} GB expert "
                          f"weights + {T * K_ * H_ * 2 / 1e6:.0f} MB Y_perm per layer streamed each step, "
                          f"{T * H_ * 2 / 1e6:.0f} MB token activations); no flush")},
        "tokens_per_s_per_gpu": per_gpu,
        "layer_tokens_per_s_per_gpu": per_gpu * L,
        "mfu": {"vs_spec_dense": mfu_flops / spec, "spec_dense_flops": spec,
                "vs_measured_sustained": mfu_flops / (peak_tf * 1e12),
                "flops_per_token_layer": FLOPS_TOK_LAYER},
        "stage_ms_per_layer": per_layer_ms,
        "hbm": {  # achieved HBM bandwidth of the memory-bound steps (algorithmic bytes / stage time)
            "combine_gbs": (T * COMBINE_BYTES_TOK / (per_layer_ms["combine"] / 1e3) / 1e9
                            if per_layer_ms.get("combine") else None),
            "combine_bytes_per_token": COMBINE_BYTES_TOK,
            "peak_gbs": peaks.get("hbm_gbs"),
            "note": "combine reads k bf16 expert rows + the residual and writes y (81,920 B/token); the dispatch "
                    "writes only the row maps (the row copy is fused into GEMM1's A load)"},
        "attention": attn_info,
        "saturation_T": {"tokens_per_gpu": t_tok, "flops": t_flops, "N": n_for_T, "gamma": 1.2,
                         "flops_per_s": f_gemm, "ag_bytes_per_s": bw,
                         "note": "Eq. 1 per layer, F = measured grouped-GEMM rate of this run"},
        "layer_ms": step_layer_ms,
        "exposed_ag": {"ms_per_layer": per_layer_ms["gather_wait"],
                       "frac_of_layer": per_layer_ms["gather_wait"] / step_layer_ms if step_layer_ms and nfwd else None,
                       "note": ("stream wait before GEMM1 on gathered layers (0 when N=1)" if not emu else
                                f"emulated {emu}-rank gather (local D2D, no NVLink): exposed wait")},
        "roofline": {"kernel": "grouped GEMM1 gate/up + SwiGLU (tcgen05)", "bound": "tensor",
                     "achieved": g1_tflops, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": g1_tflops / peak_tf if g1_tflops else None,
                     "peak_source": peak_note,
                     "algorithmic_flops_per_launch": g1_flops, "ms_per_launch": g1_ms,
                     "traffic": traffic},
        "clocks": clk,
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": xh.numel() * 2,
                "d2h_bytes_per_step": yh[0].numel() * 2,
                "note": "public API (MoEStack.run over the C ABI); every step copies its input from pinned "
                        "host memory and its output back, on two copy streams overlapping the neighbouring "
                        "steps' compute (double-buffered); all copies inside the timed region"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_tok = int(os.environ.get("ASYNCEP_CPU_TOKENS", "4096"))
        del stack
        torch.cuda.empty_cache()
        orc = OracleSample()
        v, dt, desc = orc.run(n_tok)
        line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": orc.threads, "kind": "oracle",
                                "sample": desc + f"; {dt:.1f} s of CPU work"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
