"""Exposed AllGather under SURVEY S8(d)'s definition on one B200, swept over the co-resident copy
kernel's configuration: wall(gathered stack, N-rank gather emulated at the NVLink rate) -
wall(resident stack), same kernels and tokens, step by step interleaved in one process.

    python profiles/gather_interference.py [--fp8] [--tokens 32768] [--N 8] [--ctas 296,148,74]
                                           [--link-gbs 770] [--pairs 8]

One JSON line per configuration: medians of the step times, the exposed ms per gathered layer and
its fraction of the resident layer time, per-stage times of both stacks, clocks.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_2605_02960_b200 import asyncep as A  # noqa: E402
from paper_2605_02960_b200.stack import MoEStack  # noqa: E402

L, E, K, H, h = 8, 128, 8, 4096, 1536


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fp8", action="store_true")
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--N", type=int, default=8)
    ap.add_argument("--ctas", default="296,148,74")
    ap.add_argument("--link-gbs", type=float, default=770.0)
    ap.add_argument("--pairs", type=int, default=8)
    ap.add_argument("--prio", type=int, default=0, help="compute-stream priority (0 = default, -1/-2 higher)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    T = args.tokens
    gen = synth.expert_weights_fp8 if args.fp8 else synth.expert_weights
    rf = lambda l: synth.router_weight(E, H, 0, l, device=dev)
    ef = lambda l, ex: gen(E, H, h, 0, l, device=dev, experts=ex)
    flags = A.FLAG_STAGE_TIMING
    cs = torch.cuda.Stream(dev, priority=args.prio) if args.prio else torch.cuda.current_stream(dev)
    torch.cuda.set_stream(cs)
    res = MoEStack(L, E, K, H, h, T, rf, ef, world_size=1, flags=flags, device=dev, fp8=args.fp8, compute_stream=cs)
    gat = MoEStack(L, E, K, H, h, T, rf, ef, world_size=args.N, rank=0, flags=flags, device=dev, fp8=args.fp8,
                   compute_stream=cs)
    shards = gat.peer_shards()
    A.asyncep_set_link_emulation(gat.ctx, args.link_gbs * 1e9)
    x = synth.tokens(T, H, 17, device=dev)
    o_r, o_g = torch.empty_like(x), torch.empty_like(x)

    def step_ms(fn):
        cs = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(cs)
        fn()
        e1.record(cs)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    run_r = lambda: res.run(x, out=o_r)
    run_g = lambda: gat.run(x, out=o_g, local_shards=shards)
    for _ in range(3):
        run_r()
        run_g()
    for ctas in [int(c) for c in args.ctas.split(",")]:
        A.asyncep_set_gather_copy_ctas(gat.ctx, ctas)
        for _ in range(2):
            run_r()
            run_g()
        A.asyncep_reset_stage_times(res.ctx)
        A.asyncep_reset_stage_times(gat.ctx)
        ck = ClockSampler(0).start()
        tr, tg = [], []
        for _ in range(args.pairs):
            tr.append(step_ms(run_r))
            tg.append(step_ms(run_g))
        clk = ck.stop()
        sr, nr = A.asyncep_stage_times(res.ctx)
        sg, ng = A.asyncep_stage_times(gat.ctx)
        mr, mg = float(np.median(tr)), float(np.median(tg))
        exp_layer = (mg - mr) / (L - 1)
        print(json.dumps({
            "fp8": args.fp8, "tokens": T, "N": args.N, "link_gbs": args.link_gbs, "copy_ctas": ctas,
            "compute_priority": args.prio,
            "step_ms_resident": mr, "step_ms_gathered": mg, "exposed_ms_per_layer": exp_layer,
            "exposed_frac_of_layer": exp_layer / (mr / L),
            "bitwise_equal": bool(torch.equal(o_r.view(torch.int16), o_g.view(torch.int16))),
            "stage_ms_resident": {k: v / max(nr, 1) for k, v in sr.items()},
            "stage_ms_gathered": {k: v / max(ng, 1) for k, v in sg.items()},
            "all_resident": tr, "all_gathered": tg, "clocks": clk}), flush=True)

if __name__ == "__main__":
    main()
