#!/usr/bin/env python
"""Benchmark: AsyncEP MoE-layer stack forward on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[2], the metric's config): Qwen3-235B-A22B MoE-layer
shape -- E=128 experts, top-8, H=4096, expert FFN h=1536 -- BF16, an 8-layer stack with
residual chaining (reading R9), 32,768 tokens per GPU (weak scaling: per-GPU work fixed).
One "step" = one pass of the whole hot path (router -> permute -> grouped GEMM with
SwiGLU -> combine) through all 8 layers over one batch of synthetic tokens.

  N = 1  : all layers resident (world_size 1, no gather).
  N > 1  : one process per GPU.  `python bench.py --gpus N` launches the N ranks itself
           (torch.distributed.run on 127.0.0.1) when WORLD_SIZE is unset; under torchrun it
           is one rank.  Experts of layers >= 1 are sharded 1/N by expert index, layer 0 is
           replicated, and layer l+1 is gathered into a double-buffered slot on a side stream
           while layer l computes.  No data-path collective.  Every
           available gather transport (NCCL AllGather, copy engines over CUDA-IPC peer
           shards, the co-resident copy kernel) is probed and measured; the fastest carries
           the headline (or the one --gather names).

Timing: W warm-up steps, then K steps bracketed by barrier + cuda synchronize, CUDA
events on the compute stream, max over ranks.  Inputs are larger than L2 (38.7 GB of
weights, 268 MB of activations per layer), so no explicit L2 flush.

Exposed AllGather: exposed_AG = wall(gathered stack) - wall(resident
stack), the same kernels and tokens with every layer resident, timed step by step
interleaved in the same process after the timed region -- wait plus interference.

--impl reference: the CPU oracle (oracle/, plain fp64 C) on the host cores, on a bounded
sample of the same workload (see cpu_baseline.sample in the JSON line).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
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
ORACLE_SAMPLE_TOKENS = 2048  # per oracle sample, the same in cpu_baseline and --impl reference
NVLINK_ASSUMED_GBS = 770.0   # B200_PROFILING.md measured NVLink-5 peer copy (only when no probe ran)


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


B200_SMS = 148


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def tensor_peak(peaks: dict, src: str, clk: dict, fp8: bool):
    """Tensor peak for the dominant kernel (FP8: x 2, the nominal fp8:bf16 dense ratio), chosen
    from this run's own clock record: a run that hit the power cap (or ran well below the maximum
    SM clock) is a kernel inside a long step -> MEASURED_PEAKS' sustained cuBLAS rate; a run that
    stayed at (>= 95 % of) the maximum clock with no throttle reason -> the burst rate.  Burst,
    sustained and the nominal per-clock rate at the run's median SM clock (8,192 bf16 FLOP/clk/SM x
    SMs x clock) are all returned for context."""
    burst = peaks.get("bf16_tflops", 1590.0)
    sus = peaks.get("bf16_tflops_sustained", burst)
    sus_mhz = (peaks.get("clocks_under_load") or {}).get("sm_mhz_median")
    run_mhz, max_mhz = clk.get("sm_mhz"), clk.get("sm_max_mhz")
    capped = bool(clk.get("reasons")) or not (run_mhz and max_mhz and run_mhz >= 0.95 * max_mhz)
    mult = 2.0 if fp8 else 1.0
    if capped:
        peak, note = sus, f"{src} bf16_tflops_sustained {sus}" + (
            f" (median {sus_mhz} MHz under load)" if sus_mhz else "") + " -- run power-capped / below max clock"
    else:
        peak, note = burst, f"{src} bf16_tflops {burst} (burst) -- run at max clock, no throttle reason"
    if fp8:
        note += " x 2 (nominal fp8:bf16 dense ratio)"
    nominal = 8192.0 * B200_SMS * run_mhz * 1e6 / 1e12 if run_mhz else None
    return peak * mult, note, {"burst": burst * mult, "sustained": sus * mult,
                               "nominal_at_run_clock": nominal * mult if nominal else None}


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    def __init__(self, dev_index: int, period=0.02):
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
    n_tok = int(os.environ.get("ASYNCEP_REF_TOKENS", str(ORACLE_SAMPLE_TOKENS)))
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


# ------------------------------------------------------------------------------ launcher
def self_launch(argv, n: int) -> int:
    """`bench.py --gpus N` without a torchrun environment: start the N ranks here (one process
    per GPU, rendezvous on 127.0.0.1) and pass rank 0's JSON line through."""
    import torch
    if "ASYNCEP_BENCH_DEVICE" not in os.environ and torch.cuda.device_count() < n:
        print(f"bench.py: --gpus {n} but only {torch.cuda.device_count()} visible GPU(s)", file=sys.stderr)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    if "NCCL_DEBUG" not in env:  # communicator init (transports, NVLS, channels) into the log, not stdout
        env.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT", NCCL_DEBUG_FILE="/dev/stderr")
    env.setdefault("OMP_NUM_THREADS", "8")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    r = subprocess.run(cmd, env=env, stdout=subprocess.PIPE, text=True)
    sys.stdout.write(r.stdout)
    sys.stdout.flush()
    return r.returncode


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
    ap.add_argument("--layers", type=int, default=L_)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--simt", action="store_true", help="CUDA-core GEMM (debug)")
    ap.add_argument("--xperm", action="store_true", help="materialise X_perm (FLAG_XPERM; the default)")
    ap.add_argument("--gate", action="store_true",
                    help="gated gather: each layer's gather starts after the previous forward's dispatch "
                         "(asyncep_set_gather_gate)")
    ap.add_argument("--fused-dispatch", action="store_true",
                    help="GEMM1 gathers the token rows itself (FLAG_FUSED_DISPATCH)")
    ap.add_argument("--emulate-gather", type=int, default=0, metavar="N",
                    help="1-GPU emulation of the N-rank AsyncEP gather (copies of the N-1 peer shards into "
                         "the slot on the comm stream); measures exposed wait + interference")
    ap.add_argument("--link-gbs", type=float, default=0.0,
                    help="with --emulate-gather: pace the peer-shard copies at this GB/s (NVLink receive "
                         "bandwidth; B200_PROFILING.md measured peer copy: 770)")
    ap.add_argument("--gather", choices=["auto", "kernel", "ce", "nccl"], default="auto",
                    help="N>1 gather transport: auto = measure every available one and keep the fastest; "
                         "kernel = co-resident copy kernel over CUDA-IPC peer shards; ce = copy engines over the "
                         "same peer shards; nccl = ncclAllGather (GEMMs leave ASYNCEP_RESERVE_SMS, default 16, "
                         "SMs to NCCL's kernels)")
    ap.add_argument("--no-ab", action="store_true",
                    help="skip the resident-vs-gathered interleaved measurement of exposed AllGather")
    ap.add_argument("--ab-steps", type=int, default=0, help="interleaved A/B pairs (default: max(steps, 6))")
    ap.add_argument("--no-ab-control", action="store_true",
                    help="no second resident stack in the exposed-AllGather A/B (its noise-floor control)")
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
    ap.add_argument("--graph", action="store_true",
                    help="N=1 resident stack only: capture one step into a CUDA graph and time its replays "
                         "(no per-stage events inside a graph, so no stage times / roofline)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(sys.argv[1:], args.gpus)

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
    # on gloo; the gather then must be a peer-copy transport (CUDA IPC works within one GPU).
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
    if args.graph and (world > 1 or args.emulate_gather or args.ep or args.offload):
        raise SystemExit("--graph: resident single-GPU stacks only (the gather's events cross steps)")
    flags = (0 if args.graph else A.FLAG_STAGE_TIMING) | (A.FLAG_SIMT_GEMM if args.simt else 0) | \
        (A.FLAG_XPERM if args.xperm else 0) | (A.FLAG_FUSED_DISPATCH if args.fused_dispatch else 0)
    graph_stream = torch.cuda.Stream(dev) if args.graph else None
    gen = synth.expert_weights_fp8 if args.fp8 else synth.expert_weights
    emu = args.emulate_gather if world == 1 else 0
    router_fn = lambda l: synth.router_weight(E_, H_, seed, l, device=dev, zipf_s=args.zipf)
    expert_fn = lambda l, ex: gen(E_, H_, h_, seed, l, device=dev, experts=ex)
    stack = MoEStack(L, E_, K_, H_, h_, T, router_fn, expert_fn,
                     world_size=emu or world, rank=rank, replicate_layer0=True, flags=flags, device=dev,
                     nccl_comm=comm, fp8=args.fp8, offload_window=args.offload, compute_stream=graph_stream)
    local_shards = stack.peer_shards() if emu > 1 else None
    gathered = (world > 1 or emu > 1) and not args.ep
    reserve_nccl = int(os.environ.get("ASYNCEP_RESERVE_SMS", "16"))
    p2p_error = None
    if world > 1 and not args.ep and args.gather != "nccl":
        try:
            stack.enable_p2p_gather()
        except Exception as e:  # recorded in the JSON line; NCCL remains
            p2p_error = f"{type(e).__name__}: {str(e)[:160]}"
        # every rank must take the same transports (the probes and NCCL calls are collective)
        ok = torch.tensor([0 if p2p_error else 1], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            p2p_error = p2p_error or "peer-shard mapping failed on another rank"
            A.asyncep_set_peer_shards(stack.ctx, None)
    if emu > 1 and args.link_gbs > 0:
        A.asyncep_set_link_emulation(stack.ctx, args.link_gbs * 1e9)
    if args.gate and (world > 1 or emu > 1):
        A.asyncep_set_gather_gate(stack.ctx, True)
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

    def timed_steps(n, run=_run, xin=x, o=out):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(cs)
        for _ in range(n):
            torch.cuda.nvtx.range_push("step")
            run(xin, o)
            torch.cuda.nvtx.range_pop()
        e1.record(cs)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)) / n

    # ---------------- gather transports (N > 1): startup probe of each, then a short timed run of
    # each; the fastest carries the headline unless --gather names one.
    transports = {}
    chosen = None
    if gathered:
        cands = []
        if emu > 1:
            cands = [{"kernel": A.GATHER_COPY_KERNEL, "ce": A.GATHER_COPY_ENGINE}.get(args.gather, A.GATHER_COPY_KERNEL)]
        else:
            have_p2p = p2p_error is None and args.gather != "nccl"
            if args.gather in ("auto", "kernel") and have_p2p:
                cands.append(A.GATHER_COPY_KERNEL)
            if args.gather in ("auto", "ce") and have_p2p:
                cands.append(A.GATHER_COPY_ENGINE)
            if args.gather in ("auto", "nccl") and comm is not None:
                cands.append(A.GATHER_NCCL)
        if not cands:
            raise SystemExit(f"no gather transport available (p2p: {p2p_error}, nccl comm: {comm is not None})")
        if A.GATHER_NCCL in cands:  # NCCL's gather kernels confined to the SMs the GEMMs leave free
            _gather_pg, gather_comm = A.nccl_gather_group(reserve_nccl)
            A.asyncep_set_gather_comm(stack.ctx, gather_comm)
        probe_layer = 1 if L > 1 else 0
        for tr in cands:
            A.asyncep_set_gather_transport(stack.ctx, tr, reserve_nccl if tr == A.GATHER_NCCL else 0)
            barrier()
            probe = None
            if probe_layer >= 1 and not args.offload:  # (offload: a gather follows its H2D stage)
                ms_p, nbytes = A.asyncep_probe_gather(stack.ctx, probe_layer,
                                                      local_shards(probe_layer) if local_shards else None)
                ms_p = max_over_ranks(ms_p)
                probe = {"ms": ms_p, "bytes_per_rank": nbytes, "gbs": nbytes / (ms_p / 1e3) / 1e9}
            for _ in range(2):
                _run(x, out)
            ms_tr = timed_steps(2) if len(cands) > 1 else None
            transports[A.GATHER_NAMES[tr]] = {"probe": probe, "ms_per_step": ms_tr,
                                              "reserve_sms": reserve_nccl if tr == A.GATHER_NCCL else 0,
                                              **({"nccl_max_ctas": reserve_nccl} if tr == A.GATHER_NCCL else {})}
        if len(cands) > 1:
            chosen = min(cands, key=lambda t: transports[A.GATHER_NAMES[t]]["ms_per_step"])
        else:
            chosen = cands[0]
        A.asyncep_set_gather_transport(stack.ctx, chosen, reserve_nccl if chosen == A.GATHER_NCCL else 0)

    if args.graph:  # one step captured on the stack's (non-default) compute stream, replayed per step
        with torch.cuda.stream(cs):
            _run(x, out)
            cs.synchronize()
            graph = torch.cuda.CUDAGraph()
            l0 = A.asyncep_kernel_launches(stack.ctx)
            with torch.cuda.graph(graph, stream=cs):
                stack.run(x, out=out, cu_seqlens=cu)
            graph_launches = A.asyncep_kernel_launches(stack.ctx) - l0  # kernels inside one replay
        _eager = _run

        def _run(xin, o):  # the captured buffers replay the graph on cs; others (e2e) run eagerly
            if xin is x and o is out:
                with torch.cuda.stream(cs):
                    graph.replay()
            else:
                _eager(xin, o)
    for _ in range(args.warmup):
        _run(x, out)
    barrier()
    # The timed region.  A run whose clock record shows a hardware / thermal slowdown is rejected
    # and re-measured once (the task's timing rule); sw_power_cap is kept and noted.
    bad_reasons = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "hw_power_brake_slowdown"}
    rejected = None
    for attempt in range(2):
        A.asyncep_reset_stage_times(stack.ctx)
        launches0 = A.asyncep_kernel_launches(stack.ctx)
        clocks = ClockSampler(dev_idx).start()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(cs)
        for _ in range(args.steps):
            torch.cuda.nvtx.range_push("step")
            _run(x, out)
            torch.cuda.nvtx.range_pop()
        e1.record(cs)
        barrier()
        clk = clocks.stop()
        ms = e0.elapsed_time(e1)
        launches = A.asyncep_kernel_launches(stack.ctx) - launches0
        bad = sorted(set(clk.get("reasons") or []) & bad_reasons)
        if world > 1:  # every rank takes the same decision
            t = torch.tensor([1 if bad else 0], device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            bad = bad or (["on another rank"] if int(t.item()) else [])
        if not bad or attempt == 1:
            break
        rejected = {"ms": ms, "reasons": bad, "sm_mhz": clk.get("sm_mhz")}
        print(f"bench.py: timed region saw {bad}; re-measuring once", file=sys.stderr)
    if rejected:
        clk["remeasured_after"] = rejected
    # NEXT-1 (App. B.4): T from the last timed step as the profile pass -- t_c = the
    # resident layer 0, t_e = the slowest gathered layer, C_dummy = f_tok x tokens (in the library)
    calib = None  # (N = 1 without offload: nothing is transferred, Eq. 3 has no t_EP to calibrate)
    if not args.graph and not args.ep and L > 1 and (gathered or args.offload):
        try:
            calib = A.asyncep_calibrate_T(stack.ctx, 1.2, T)
        except A.AsyncEPError as e:
            calib = {"error": str(e)[:200]}
    if args.graph:
        launches = graph_launches * args.steps
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
    peak_tf, peak_note, peak_ref = tensor_peak(peaks, peak_src, clk, args.fp8)
    spec = SPEC_BF16 * (2.0 if args.fp8 else 1.0)
    traffic = ncu_traffic(args.fp8)
    per_layer_ms = {k: v / max(nfwd, 1) for k, v in stages.items()}
    gemm_ms = per_layer_ms["gemm1_gateup_swiglu"] + per_layer_ms["gemm2_down"]
    f_gemm = (GEMM1_FLOPS_TOK + GEMM2_FLOPS_TOK) * T / (gemm_ms / 1e3) if gemm_ms > 0 else 0.0
    step_layer_ms = ms_step / L

    # ---------------- exposed AllGather: wall(gathered) - wall(resident), same kernels
    # and tokens, every layer resident in the second stack; step by step, interleaved.
    exposed = {"ms_per_layer": 0.0, "frac_of_layer": 0.0, "wait_ms_per_layer": per_layer_ms["gather_wait"],
               "note": "N=1: every layer resident, nothing gathered"}
    if gathered or args.offload:
        exposed = {"ms_per_layer": None, "frac_of_layer": None, "wait_ms_per_layer": per_layer_ms["gather_wait"],
                   "note": "resident-vs-gathered A/B not run (--no-ab, or a one-layer stack); the wait for the "
                           "slot (or the H2D window) before GEMM1 only"}
    if gathered and not args.no_ab and L > 1:
        res = MoEStack(L, E_, K_, H_, h_, T, router_fn, expert_fn, world_size=1, rank=0, replicate_layer0=True,
                       flags=flags & ~A.FLAG_STAGE_TIMING, device=dev, fp8=args.fp8,
                       compute_stream=cs)
        if args.attn:
            res.enable_attention(lambda l: synth.attn_weights(H_, ATT_HQ, ATT_HKV, 128, seed, l, device=dev),
                                 ATT_HQ, ATT_HKV, max_prompts=int(cu.numel() - 1))
        run_res = lambda xin, o: res.run(xin, out=o, cu_seqlens=cu)
        out_r = torch.empty_like(x)
        # control: a second resident stack (same weights and tokens, its own memory).  Two identical
        # contexts can differ by a few % on some boxes (profiles/r02/mx: A/B harness control), so the
        # resident time is the pooled median of both and their difference is reported as the noise.
        ctl = None
        if not args.no_ab_control:
            ctl = MoEStack(L, E_, K_, H_, h_, T, router_fn, expert_fn, world_size=1, rank=0, replicate_layer0=True,
                           flags=flags & ~A.FLAG_STAGE_TIMING, device=dev, fp8=args.fp8, compute_stream=cs)
            if args.attn:
                ctl.enable_attention(lambda l: synth.attn_weights(H_, ATT_HQ, ATT_HKV, 128, seed, l, device=dev),
                                     ATT_HQ, ATT_HKV, max_prompts=int(cu.numel() - 1))
        run_ctl = (lambda xin, o: ctl.run(xin, out=o, cu_seqlens=cu)) if ctl is not None else None
        out_c = torch.empty_like(x)
        for _ in range(2):
            run_res(x, out_r)
            _run(x, out)
            if run_ctl:
                run_ctl(x, out_c)
        n_ab = args.ab_steps or max(args.steps, 6)
        clocks_ab = ClockSampler(dev_idx).start()
        t_res, t_gat, t_ctl = [], [], []
        mhz = {"r": [], "g": [], "c": []}  # per-leg median SM clock (is the interference the clock?)

        def leg(tag, store, *a):
            ck = ClockSampler(dev_idx, period=0.005).start()
            store.append(timed_steps(1, *a))
            mhz[tag].append(ck.stop().get("sm_mhz"))

        legs = [("r", lambda: leg("r", t_res, run_res, x, out_r)), ("g", lambda: leg("g", t_gat))]
        if run_ctl:
            legs.append(("c", lambda: leg("c", t_ctl, run_ctl, x, out_c)))
        for i in range(n_ab):  # rotate the order of the legs step by step
            for j in range(len(legs)):
                legs[(i + j) % len(legs)][1]()
        clk_ab = clocks_ab.stop()
        med_g = float(np.median(t_gat))
        med_r = float(np.median(t_res + t_ctl))   # pooled resident legs
        bitwise = bool(torch.equal(out.view(torch.int16), out_r.view(torch.int16)))
        exp_layer = (med_g - med_r) / (L - 1)
        exposed = {
            "ms_per_layer": exp_layer, "frac_of_layer": exp_layer / (med_r / L),
            "wait_ms_per_layer": per_layer_ms["gather_wait"],
            "step_ms_gathered": med_g, "step_ms_resident": med_r, "pairs": n_ab, "clocks": clk_ab,
            "output_bitwise_equal_resident": bitwise,
            "sm_mhz_per_leg": {k: (float(np.median([m for m in v if m])) if any(v) else None)
                               for k, v in mhz.items() if v},
            "note": ("SURVEY S8(d): (median gathered step - median resident step) / (L-1 gathered layers), "
                     "steps interleaved one by one in this process, leg order rotated (max over ranks); frac = "
                     "that / resident layer time; resident = the pooled steps of two resident contexts.  "
                     "wait_ms_per_layer = the compute stream's wait for the slot before GEMM1 (inside the "
                     "timed region) -- the part of the exposure that is not interference")}
        if run_ctl:
            m1, m2 = float(np.median(t_res)), float(np.median(t_ctl))
            exposed["control"] = {
                "step_ms_resident_1": m1, "step_ms_resident_2": m2,
                "frac_of_layer": abs(m2 - m1) / (L - 1) / (med_r / L),
                "note": "two identical resident contexts, normalised like frac_of_layer: the A/B's noise floor"}
            del ctl
        del res
        torch.cuda.empty_cache()

    # ---------------- contrast (Table 1 DP x EP): the same stack as
    # synchronous expert parallelism -- each rank keeps its E/N experts and the permuted token rows
    # travel to them and back with two on-path AllToAlls per layer -- timed on the same box (N > 1).
    ep_contrast = None
    if world > 1 and comm is not None and not args.ep and not args.fp8 and not args.attn and not args.no_ab:
        o_ep = torch.empty_like(x)
        stack.run_ep(x, out=o_ep)
        n_ep = max(2, min(args.steps, 5))
        ms_ep = timed_steps(n_ep, lambda xin, o: stack.run_ep(xin, out=o), x, o_ep)
        ep_contrast = {
            "ms_per_step": ms_ep, "value": world * T / (ms_ep / 1e3), "unit": "tokens/s",
            "asyncep_speedup": ms_ep / ms_step, "steps": n_ep,
            "alltoall_bytes_per_layer_per_rank": 4 * K_ * (world - 1) / world * T * H_ * 2,
            "note": "asyncep_ep_forward per layer: router + permute, per-expert count exchange + host sync, "
                    "row AllToAll to the expert owners (ncclSend/Recv, on the compute stream), grouped GEMM, "
                    "reverse AllToAll, combine; same tokens, weights and kernels as the headline"}
        del o_ep
        torch.cuda.empty_cache()

    # Eq. 1 (R11/R12): T in tokens/GPU with F = this run's grouped-GEMM rate and the
    # gather bandwidth probed at startup with the chosen transport (else assumed NVLink 5 peer copy).
    n_for_T = world if world > 1 else (emu if emu > 1 else 8)
    probe = transports.get(A.GATHER_NAMES.get(chosen, ""), {}).get("probe") if chosen is not None else None
    if probe:
        bw, bw_src = probe["gbs"] * 1e9, f"probed at startup ({A.GATHER_NAMES[chosen]}, one layer's gather)"
    else:
        bw, bw_src = (args.link_gbs or NVLINK_ASSUMED_GBS) * 1e9, "assumed (no gather at this N)"
    tcfg = A.make_config(L, E_, K_, H_, h_, expert_dtype=A.FP8_E4M3 if args.fp8 else A.BF16,
                         world_size=n_for_T, max_tokens=T, gamma=1.2)
    t_tok, t_flops = A.asyncep_saturation_T(tcfg, f_gemm, bw) if f_gemm > 0 else (None, None)
    model = "qwen3-30b-a3b (config 2)" if args.shape == "30b" else "qwen3-235b-a22b"
    if world > 1:
        par = f"dp{world}+asyncep{world}"
    elif emu > 1:
        par = (f"dp1, asyncep{emu} gather emulated on 1 GPU (copies of the {emu - 1} peer shards into the slot on "
               "the comm stream" + (f", paced at {args.link_gbs} GB/s" if args.link_gbs else "") + ")")
    else:
        par = "dp1 (all experts resident)"
    if args.ep:
        par = f"dp{world}xep{world} contrast (2 on-path AllToAlls/layer)"
    if args.offload:
        par += f", shards offloaded to pinned host memory, {args.offload}-deep device window (NEXT-2)"
    gather_desc = "none" if not gathered else A.GATHER_NAMES[chosen] + (
        " (emulated peers)" if emu > 1 else "") + (f"; p2p setup failed: {p2p_error}" if p2p_error else "")
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
                   "parallelism": par, "gather": gather_desc + (" (gated: starts after the dispatch)" if args.gate and gathered else ""),
                   "launch": ("one step captured as a CUDA graph, replayed per timed step (e2e runs eagerly)"
                              if args.graph else "eager stream launches"),
                   "l2": (f"inputs larger than L2 ({L * E_ * 3 * H_ * h_ * (1 if args.fp8 else 2) / 1e9:.1f} GB expert "
                          f"weights + {T * K_ * H_ * 2 / 1e6:.0f} MB Y_perm per layer streamed each step, "
                          f"{T * H_ * 2 / 1e6:.0f} MB token activations); no flush")},
        "tokens_per_s_per_gpu": per_gpu,
        "layer_tokens_per_s_per_gpu": per_gpu * L,
        "mfu": {"vs_spec_dense": mfu_flops / spec, "spec_dense_flops": spec,
                "vs_measured_peak_at_run_clock": mfu_flops / (peak_tf * 1e12),
                "flops_per_token_layer": FLOPS_TOK_LAYER},
        "stage_ms_per_layer": per_layer_ms,
        "hbm": {  # achieved HBM bandwidth of the memory-bound steps (algorithmic bytes / stage time)
            "combine_gbs": (T * COMBINE_BYTES_TOK / (per_layer_ms["combine"] / 1e3) / 1e9
                            if per_layer_ms.get("combine") else None),
            "combine_bytes_per_token": COMBINE_BYTES_TOK,
            "peak_gbs": peaks.get("hbm_gbs"),
            "dispatch_gbs": (T * (H_ * 2 + K_ * H_ * (1 if args.fp8 else 2)) / (per_layer_ms["permute"] / 1e3) / 1e9
                             if per_layer_ms.get("permute") and not args.fused_dispatch else None),
            "note": "combine reads k bf16 expert rows + the residual and writes y (81,920 B/token); the dispatch "
                    "(permute stage: maps + row copy, or the FP8 quantisation into the k rows) reads x once and "
                    "writes k rows per token (73,728 B/token BF16, 40,960 B/token FP8); with --fused-dispatch it "
                    "writes only the row maps (GEMM1 gathers the rows)"},
        "attention": attn_info,
        "saturation_T": {"tokens_per_gpu": t_tok, "flops": t_flops, "N": n_for_T, "gamma": 1.2,
                         "flops_per_s": f_gemm, "ag_bytes_per_s": bw, "ag_bandwidth_source": bw_src,
                         "note": "Eq. 1 per layer, F = measured grouped-GEMM rate of this run"},
        "calibrated_T": calib,
        "layer_ms": step_layer_ms,
        "exposed_ag": exposed,
        "gather_transports": transports or None,
        "ep_contrast": ep_contrast,
        "roofline": {"kernel": "grouped GEMM1 gate/up + SwiGLU (tcgen05)", "bound": "tensor",
                     "achieved": g1_tflops, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": g1_tflops / peak_tf if g1_tflops else None,
                     "peak_source": peak_note,
                     "frac_of_burst": g1_tflops / peak_ref["burst"] if g1_tflops else None,
                     "frac_of_sustained": g1_tflops / peak_ref["sustained"] if g1_tflops else None,
                     "frac_of_nominal_at_run_clock": (g1_tflops / peak_ref["nominal_at_run_clock"]
                                                      if g1_tflops and peak_ref["nominal_at_run_clock"] else None),
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
        n_tok = int(os.environ.get("ASYNCEP_CPU_TOKENS", str(ORACLE_SAMPLE_TOKENS)))
        n_samp = 3
        del stack
        torch.cuda.empty_cache()
        orc = OracleSample()
        runs = [orc.run(n_tok, sample=i) for i in range(n_samp)]
        dt = sum(r[1] for r in runs)
        v = n_tok * n_samp / dt / L_
        line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": orc.threads, "kind": "oracle",
                                "sample": f"{n_samp} x " + runs[0][2] + f"; {dt:.1f} s of CPU work"}
        # also a one-thread figure (512 tokens: one full 32-row block per expert)
        import oracle
        oracle.set_num_threads(1)
        v1, dt1, _ = orc.run(512, sample=99)
        oracle.set_num_threads(orc.threads)
        line["cpu_baseline"]["single_thread"] = {"value": v1, "unit": "tokens/s", "cores": 1,
                                                 "sample": f"512 tokens, 1 thread, {dt1:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
