#!/usr/bin/env python
"""How fast do the 1-GPU gather emulation's copies run next to the MoE layer?  Times 2.4 GB
(an FP8 layer's 8 shards) and 4.8 GB (BF16) of 64 MiB device-to-device copies on a side
stream: alone, and concurrently with the persistent GEMMs of the layer stack on the compute
stream.  Prints one JSON line per case (GB/s)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from gpu_helpers import Workload  # noqa: E402

CH = 64 << 20


MODE = "ce" if "--ce" in sys.argv else "torch"


def copies(dst, src, nbytes, stream):
    from paper_2605_02960_b200 import asyncep as A
    with torch.cuda.stream(stream):
        for o in range(0, nbytes, CH):
            n = min(CH, nbytes - o)
            if MODE == "ce":  # the library's gather transport (copy-engine hint)
                A.asyncep_gather_copy(dst[o:], src[o:], n, stream)
            else:
                dst[o:o + n].copy_(src[o:o + n], non_blocking=True)


def timed(fn, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


fp8 = "--fp8" in sys.argv
wl = Workload(L=2, E=128, k=8, H=4096, h=1536, seed=0, fp8=fp8)
st = wl.stack(max_tokens=32768)
x = wl.tokens(32768)
nbytes = (2400 if fp8 else 4800) << 20
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
side = torch.cuda.Stream()
main = torch.cuda.current_stream()
for _ in range(2):
    copies(dst, src, nbytes, side)
    st.run(x)
torch.cuda.synchronize()
alone = timed(lambda: copies(dst, src, nbytes, side), side)
stack_alone = timed(lambda: st.run(x), main)
# concurrent: start both, time the copies on the side stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.run(x)                      # the stack is enqueued first ...
e0.record(side)                # ... then the copies, which start right away on the side stream
copies(dst, src, nbytes, side)
e1.record(side)
torch.cuda.synchronize()
conc = e0.elapsed_time(e1)
print(json.dumps({"mode": MODE, "fp8": fp8, "bytes": nbytes, "copy_alone_ms": alone, "copy_alone_gbs": nbytes / alone / 1e6,
                  "stack_2layers_ms": stack_alone, "copy_concurrent_ms": conc,
                  "copy_concurrent_gbs": nbytes / conc / 1e6}))
