"""Small forwards for compute-sanitizer (memcheck / racecheck / synccheck): the permute, combine and
quantisation kernels with the CUDA-core GEMM/router (FLAG_SIMT_*; the sanitizer does not model
tcgen05/TMA), BF16 and FP8-dispatch shapes, ragged token counts."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from gpu_helpers import Workload  # noqa: E402

for (E, k, H, h, T) in ((8, 2, 64, 128, 300), (128, 8, 256, 256, 700), (64, 12, 256, 256, 129)):
    wl = Workload(L=1, E=E, k=k, H=H, h=h, seed=3)
    st = wl.stack(max_tokens=T, flags=2 | 8)
    x = wl.tokens(T)
    y = torch.empty_like(x)
    st.forward(0, x, residual=x, y=y)
    torch.cuda.synchronize()
    print("ok", E, k, H, h, T, float(y.float().abs().mean()))
