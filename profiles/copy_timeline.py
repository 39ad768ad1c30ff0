#!/usr/bin/env python
"""Timeline of the gather-transport copies (asyncep_gather_copy, 64 MiB chunks) issued on a side
stream while the MoE stack runs: completion time of every chunk relative to the stack's start
(CUDA events), to see whether the copies progress during the persistent GEMMs or only in gaps."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from gpu_helpers import Workload  # noqa: E402
from paper_2605_02960_b200 import asyncep as A  # noqa: E402

CH = 64 << 20
fp8 = "--fp8" in sys.argv
wl = Workload(L=2, E=128, k=8, H=4096, h=1536, seed=0, fp8=fp8)
st = wl.stack(max_tokens=32768, flags=A.FLAG_STAGE_TIMING | (A.FLAG_XPERM if "--xperm" in sys.argv else 0))
x = wl.tokens(32768)
nbytes = 2400 << 20
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
side = torch.cuda.Stream()
main = torch.cuda.current_stream()
st.run(x)
torch.cuda.synchronize()
ev0 = torch.cuda.Event(enable_timing=True)
ev0.record(main)
side.wait_event(ev0)
evs = []
for o in range(0, nbytes, CH):   # copies enqueued FIRST, then the stack
    A.asyncep_gather_copy(dst[o:], src[o:], min(CH, nbytes - o), side)
    e = torch.cuda.Event(enable_timing=True)
    e.record(side)
    evs.append(e)
m1 = torch.cuda.Event(enable_timing=True)
st.run(x)
m1.record(main)
torch.cuda.synchronize()
t = [round(ev0.elapsed_time(e), 3) for e in evs]
print(json.dumps({"fp8": fp8, "xperm": "--xperm" in sys.argv, "chunk_done_ms": t, "stack_ms": round(ev0.elapsed_time(m1), 3),
                  "stages": A.asyncep_stage_times(st.ctx)[0]}))
