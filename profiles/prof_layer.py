#!/usr/bin/env python
"""One Qwen3-235B-shape layer (E=128,k=8,H=4096,h=1536) at 32,768 tokens, run --iters
times -- a light driver for ncu captures of the hot kernels (the bench's launch config)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from gpu_helpers import Workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--tokens", type=int, default=32768)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--H", type=int, default=4096)
ap.add_argument("--h", type=int, default=1536)
ap.add_argument("--fp8", action="store_true")
a = ap.parse_args()
wl = Workload(L=1, E=128, k=8, H=a.H, h=a.h, seed=0, fp8=a.fp8)
st = wl.stack(max_tokens=a.tokens, flags=a.flags)
x = wl.tokens(a.tokens)
y = torch.empty_like(x)
torch.cuda.synchronize()
for _ in range(a.iters):
    st.forward(0, x, residual=x, y=y)
torch.cuda.synchronize()
print("done")
