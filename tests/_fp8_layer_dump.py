"""Helper for test_gpu_fp8.test_fused_act_quant_bitwise: one FP8 layer (three forwards, so the
per-slice counters and amax must re-arm) in a fresh process; the environment selects the fused or
the separate intermediate quantisation.  Writes the three outputs to argv[1] (.npy)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gpu_helpers import Workload  # noqa: E402

flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = Workload(L=1, E=64, k=6, H=1024, h=512, seed=23, fp8=True)
st = wl.stack(max_tokens=4096, flags=flags)
outs = []
for T in (3000, 700, 3000):
    x = wl.tokens(T)
    y = torch.empty_like(x)
    st.forward(0, x, residual=x, y=y)
    torch.cuda.synchronize()
    outs.append(y.view(torch.int16).cpu().numpy().ravel())
np.save(sys.argv[1], np.concatenate(outs))
