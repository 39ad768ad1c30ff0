"""Same-process interleaved A/B of two library configurations that differ only in asyncep_config.flags
(e.g. swap-AB tail tiles on / off): two 8-layer Qwen3-235B stacks over the same weights and tokens,
steps alternated one by one, medians of the step time and of each stage.  Removes the box-to-box and
run-to-run clock drift of separate bench runs (the part runs power-capped).

    python profiles/ab_flags.py --flags-b 0x40 [--fp8] [--tokens 16384] [--pairs 10]
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
    ap.add_argument("--flags-a", type=lambda v: int(v, 0), default=0)
    ap.add_argument("--flags-b", type=lambda v: int(v, 0), default=A.FLAG_NO_SWAP_TAILS)
    ap.add_argument("--pairs", type=int, default=10)
    ap.add_argument("--reverse-create", action="store_true", help="create context b before context a")
    ap.add_argument("--emulate", type=int, default=1, help="N > 1: both stacks gathered, N ranks emulated")
    ap.add_argument("--link-gbs", type=float, default=770.0, help="emulated link rate (with --emulate)")
    ap.add_argument("--gate", default="none", choices=["none", "a", "b", "both"],
                    help="gated gather (asyncep_set_gather_gate) in context a / b / both (with --emulate)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    T = args.tokens
    gen = synth.expert_weights_fp8 if args.fp8 else synth.expert_weights
    rf = lambda l: synth.router_weight(E, H, 0, l, device=dev)
    ef = lambda l, ex: gen(E, H, h, 0, l, device=dev, experts=ex)
    order = (("b", args.flags_b), ("a", args.flags_a)) if args.reverse_create else (("a", args.flags_a), ("b", args.flags_b))
    N = args.emulate
    st = {n: MoEStack(L, E, K, H, h, T, rf, ef, flags=A.FLAG_STAGE_TIMING | f, device=dev, fp8=args.fp8,
                      **({"world_size": N, "rank": 0} if N > 1 else {}))
          for n, f in order}
    shards = {}
    for n in st:  # N > 1: the N-rank gather emulated on this GPU (peer shards, paced copy kernel)
        shards[n] = st[n].peer_shards() if N > 1 else None
        if N > 1 and args.link_gbs > 0:
            A.asyncep_set_link_emulation(st[n].ctx, args.link_gbs * 1e9)
        if N > 1 and args.gate in (n, "both"):
            A.asyncep_set_gather_gate(st[n].ctx, True)
    x = synth.tokens(T, H, 17, device=dev)
    out = {n: torch.empty_like(x) for n in st}
    cs = torch.cuda.current_stream()

    def step(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(cs)
        st[n].run(x, out=out[n], local_shards=shards[n])
        e1.record(cs)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(3):
        step("a")
        step("b")
    for n in st:
        A.asyncep_reset_stage_times(st[n].ctx)
    ck = ClockSampler(0).start()
    t = {"a": [], "b": []}
    for i in range(args.pairs):  # ABBA order: a fixed order biased the second config by ~3 % on one box
        for n in (("a", "b") if i % 2 == 0 else ("b", "a")):
            t[n].append(step(n))
    clk = ck.stop()
    stages = {}
    for n in st:
        s, f = A.asyncep_stage_times(st[n].ctx)
        stages[n] = {k: v / max(f, 1) for k, v in s.items()}
    ma, mb = float(np.median(t["a"])), float(np.median(t["b"]))
    print(json.dumps({"fp8": args.fp8, "tokens": T, "emulate": N, "gate": args.gate, "flags_a": args.flags_a, "flags_b": args.flags_b,
                      "step_ms_a": ma, "step_ms_b": mb, "speedup_a_over_b": mb / ma,
                      "tokens_per_s_a": T / (ma / 1e3), "tokens_per_s_b": T / (mb / 1e3),
                      "stage_ms_a": stages["a"], "stage_ms_b": stages["b"], "all_a": t["a"], "all_b": t["b"],
                      "clocks": clk}), flush=True)


if __name__ == "__main__":
    main()
