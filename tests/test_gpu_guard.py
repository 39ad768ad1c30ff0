"""Out-of-bounds write check without compute-sanitizer (closed on this GPU pool): every buffer the
library writes -- the workspace, both gather slots, the output y and the router outputs -- is placed
between 1 MiB guard bands filled with a byte pattern, a context is created on those buffers through
the C ABI (asyncep_init), and forwards of every kernel path (BF16 / FP8 experts, swap-AB tails,
the fused dispatch, the MX intermediate, the register-resident row copy at H = 2048) at ragged token
counts must leave every guard byte untouched and produce the same output, bit for bit, as the
same layer run on an ordinary stack."""
import pytest
import torch

from gpu_helpers import Workload
from paper_2605_02960_b200 import asyncep as A

pytestmark = pytest.mark.gpu

GUARD = 1 << 20
PAT = 0xA5


def _guarded(nbytes, dev="cuda"):
    """(view of nbytes, whole buffer); the view starts GUARD bytes in (256-B aligned)."""
    n = (nbytes + 255) // 256 * 256
    buf = torch.full((n + 2 * GUARD,), PAT, dtype=torch.uint8, device=dev)
    return buf[GUARD:GUARD + nbytes], buf, nbytes


def _guards_intact(entry):
    _, buf, nbytes = entry
    n = (nbytes + 255) // 256 * 256
    head, tail = buf[:GUARD], buf[GUARD + nbytes:]
    assert tail.numel() == n - nbytes + GUARD
    return bool((head == PAT).all()) and bool((tail == PAT).all())


CASES = [
    # (E, k, H, h, fp8, flags, T list)
    (16, 4, 512, 256, False, 0, [1, 129, 700]),
    (16, 4, 512, 256, False, A.FLAG_SWAP_TAILS, [5, 333]),
    (16, 4, 512, 256, False, A.FLAG_FUSED_DISPATCH, [1, 333]),
    (16, 4, 2048, 256, False, 0, [257]),
    (16, 4, 512, 256, True, 0, [1, 129, 700]),
    (16, 4, 512, 256, True, A.FLAG_MX_ACT, [333]),
    (16, 4, 512, 256, True, A.FLAG_FUSED_DISPATCH, [333]),
    (16, 4, 2048, 256, True, 0, [129]),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{'fp8' if c[4] else 'bf16'}-H{c[2]}-f{c[5]:#x}")
@pytest.mark.parametrize("N", [1, 2])
def test_forward_writes_stay_inside_their_buffers(case, N):
    E, k, H, h, fp8, flags, Ts = case
    Tmax = max(Ts)
    wl = Workload(L=2, E=E, k=k, H=H, h=h, seed=51, fp8=fp8)
    ref_st = wl.stack(max_tokens=Tmax, flags=flags)  # resident reference
    ranks = [wl.stack(max_tokens=Tmax, flags=flags, world_size=N, rank=r) for r in range(N)] if N > 1 else [ref_st]
    st = ranks[0]
    cfg = st.cfg
    ws = _guarded(A.asyncep_workspace_size(cfg))
    slots = [_guarded(A.asyncep_slot_bytes(cfg)) for _ in range(2)] if N > 1 else [None, None]
    cs = torch.cuda.current_stream()
    comm = torch.cuda.Stream() if N > 1 else None
    ctx = A.asyncep_init(cfg, None, cs, comm, st.router_w, st.shards, slots[0][0] if N > 1 else None,
                         slots[1][0] if N > 1 else None, ws[0])
    entries = [ws] + ([slots[0], slots[1]] if N > 1 else [])
    try:
        for T in Ts:
            x = wl.tokens(T)
            y = _guarded(T * H * 2)
            ids = _guarded(T * k * 4)
            w = _guarded(T * k * 4)
            counts = _guarded(E * 4)
            yv = y[0].view(torch.bfloat16).view(T, H)
            for l in range(2):
                if l >= 1 and N > 1:
                    A.asyncep_prefetch_layer_local(ctx, l, [ranks[r].shards[l] for r in range(N)])
                A.asyncep_moe_forward(ctx, l, x, residual=x, y=yv, topk_ids_out=ids[0].view(torch.int32),
                                      topk_w_out=w[0].view(torch.float32), expert_counts_out=counts[0].view(torch.int32))
                ref = ref_st.forward(l, x, residual=x)
                torch.cuda.synchronize()
                assert torch.equal(yv.view(torch.int16), ref.view(torch.int16)), (T, l)
                for e in entries + [y, ids, w, counts]:
                    assert _guards_intact(e), (T, l)
    finally:
        A.asyncep_destroy(ctx)
