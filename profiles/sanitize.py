"""Small forwards for compute-sanitizer (memcheck / racecheck / synccheck).

Default: the permute, combine and quantisation kernels with the CUDA-core GEMM/router
(FLAG_SIMT_*; the sanitizer does not model tcgen05/TMA), BF16 shapes, ragged token counts.
--tc: the product path instead (tcgen05 router and grouped GEMMs, materialised dispatch incl. the
register-resident row copy at H = 2048, swap-AB tails, BF16 and FP8 with the act quantisation, the
fused dispatch and the MX intermediate) -- memcheck then checks every ordinary load / store of
those kernels (the TMA / tcgen05 traffic itself is not instrumented)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from gpu_helpers import Workload  # noqa: E402

TC = "--tc" in sys.argv
if not TC:
    cases = [(E, k, H, h, T, False, 2 | 8) for (E, k, H, h, T) in
             ((8, 2, 64, 128, 300), (128, 8, 256, 256, 700), (64, 12, 256, 256, 129))]
else:
    cases = [
        (8, 2, 256, 256, 300, False, 0),          # BF16, ragged experts, swap-AB tails
        (128, 8, 256, 256, 700, False, 0),        # many near-empty experts
        (16, 4, 2048, 256, 257, False, 0),        # register-resident row copy (H = 2048)
        (16, 4, 512, 256, 333, False, 0x200),     # fused dispatch (cp.async gather)
        (16, 4, 512, 256, 333, True, 0),          # FP8: per-token quantisation + act quantisation
        (16, 4, 2048, 256, 129, True, 0),         # FP8, register-resident quantisation-scatter
        (16, 4, 512, 256, 333, True, 0x100),      # FP8 MX intermediate
        (16, 4, 512, 256, 333, True, 0x200),      # FP8 fused dispatch
    ]
for (E, k, H, h, T, fp8, flags) in cases:
    wl = Workload(L=1, E=E, k=k, H=H, h=h, seed=3, fp8=fp8)
    st = wl.stack(max_tokens=T, flags=flags)
    x = wl.tokens(T)
    y = torch.empty_like(x)
    st.forward(0, x, residual=x, y=y)
    torch.cuda.synchronize()
    print("ok", "fp8" if fp8 else "bf16", hex(flags), E, k, H, h, T, float(y.float().abs().mean()))
