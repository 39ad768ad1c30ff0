"""Per-layer event timeline of one step of the 8-layer Qwen3-235B stack with the N-rank gather
emulated on one B200 (asyncep_timeline_begin / _read: the view an nsys trace would give).  For each
layer: forward start, GEMM1 start (after the wait for the gathered slot), end; and the gather of
that layer on the comm stream.  JSON to stdout, plus an ASCII chart on stderr ('=' compute,
'.' waiting for the gathered slot, '|' GEMM1 start, '#' the gather).

    python profiles/timeline.py [--fp8] [--tokens 32768] [--N 8] [--link-gbs 770]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2605_02960_b200 import asyncep as A  # noqa: E402
from paper_2605_02960_b200.stack import MoEStack  # noqa: E402

L, E, K, H, h = 8, 128, 8, 4096, 1536


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fp8", action="store_true")
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--N", type=int, default=8)
    ap.add_argument("--link-gbs", type=float, default=770.0)
    ap.add_argument("--gate", action="store_true", help="gated gather (asyncep_set_gather_gate)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    gen = synth.expert_weights_fp8 if args.fp8 else synth.expert_weights
    st = MoEStack(L, E, K, H, h, args.tokens, lambda l: synth.router_weight(E, H, 0, l, device=dev),
                  lambda l, ex: gen(E, H, h, 0, l, device=dev, experts=ex), world_size=args.N, rank=0,
                  flags=A.FLAG_STAGE_TIMING, device=dev, fp8=args.fp8)
    shards = st.peer_shards()
    A.asyncep_set_link_emulation(st.ctx, args.link_gbs * 1e9)
    if args.gate:
        A.asyncep_set_gather_gate(st.ctx, True)
    x = synth.tokens(args.tokens, H, 17, device=dev)
    out = torch.empty_like(x)
    for _ in range(3):
        st.run(x, out=out, local_shards=shards)
    torch.cuda.synchronize()
    A.asyncep_timeline_begin(st.ctx)
    st.run(x, out=out, local_shards=shards)
    torch.cuda.synchronize()
    recs = A.asyncep_timeline_read(st.ctx)
    fwd = {l: (a, b, c, d) for k, l, a, b, c, d in recs if k == "forward"}
    gat = {l: (a, b) for k, l, a, b, _, _ in recs if k == "gather"}
    layers = []
    for l in range(L):
        f = fwd[l]
        g = gat.get(l)
        layers.append({"layer": l, "forward_start": f[0], "dispatch_done": f[1], "gemm1_start": f[2],
                       "forward_end": f[3], "gather_start": g[0] if g else None, "gather_end": g[1] if g else None,
                       "wait_ms": f[2] - f[1]})
    print(json.dumps({"fp8": args.fp8, "tokens": args.tokens, "N": args.N, "link_gbs": args.link_gbs, "gate": args.gate,
                      "step_ms": fwd[L - 1][3] - fwd[0][0], "layers": layers}), flush=True)
    scale = 100.0 / (fwd[L - 1][3] + 1e-9)
    for d in layers:
        row = [" "] * 101
        for t in range(int(d["forward_start"] * scale), int(d["forward_end"] * scale) + 1):
            row[min(t, 100)] = "="
        for t in range(int(d["dispatch_done"] * scale), int(d["gemm1_start"] * scale) + 1):
            row[min(t, 100)] = "."
        row[min(int(d["gemm1_start"] * scale), 100)] = "|"
        print(f"L{d['layer']} fwd {''.join(row)}", file=sys.stderr)
        if d["gather_start"] is not None:
            row = [" "] * 101
            for t in range(int(d["gather_start"] * scale), int(d["gather_end"] * scale) + 1):
                row[min(t, 100)] = "#"
            print(f"L{d['layer']} ag  {''.join(row)}", file=sys.stderr)


if __name__ == "__main__":
    main()
