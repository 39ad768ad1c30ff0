"""NEXT-3 wired into the AsyncEP stack: decoder layers (DP attention, KV-cache-free, then
MoE; reading R19) with the next layer's expert gather overlapping both halves.

The components are pinned against the oracle elsewhere (tests/test_gpu_attn.py,
tests/test_gpu_parity.py); here the stack's composition and its gather schedule are
checked bitwise: stack(l) == MoE_l(RMSNorm(x'), residual x') with x' = x + Attn_l(x), and
the N-rank gathered stack (1-GPU rank emulation) == the resident stack."""
import numpy as np
import pytest
import torch

import synth
from gpu_helpers import Workload
from paper_2605_02960_b200 import asyncep as A

pytestmark = pytest.mark.gpu

Hq, Hkv = 8, 2


def _bits(t):
    return t.view(torch.int16)


def _decoder_stack(wl, T, **kw):
    st = wl.stack(max_tokens=T, **kw)
    st.enable_attention(lambda l: synth.attn_weights(wl.H, Hq, Hkv, 128, 5, l, device="cuda"), Hq, Hkv)
    return st


def _cu(lengths):
    return torch.from_numpy(np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)).cuda()


@pytest.mark.parametrize("fp8", [False, True], ids=["bf16_experts", "fp8_experts"])
def test_decoder_stack_composition_bitwise(fp8):
    wl = Workload(L=3, E=16, k=4, H=512, h=256, seed=21, fp8=fp8)
    lengths = [700, 1, 300, 129]
    T = sum(lengths)
    cu = _cu(lengths)
    x = wl.tokens(T)
    st = _decoder_stack(wl, T)
    out = st.run(x, cu_seqlens=cu).clone()
    # the same layers composed by hand through the two ABI entry points
    cur = x.clone()
    for l in range(wl.L):
        xa = torch.empty_like(cur)
        xn = torch.empty_like(cur)
        A.asyncep_attn_layer(st.attn_cfg, cur, cu, st.attn_w[l], xa, xn, st.attn_ws)
        y = torch.empty_like(cur)
        st.forward(l, xn, residual=xa, y=y)
        cur = y
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    assert torch.equal(_bits(out), _bits(cur))


@pytest.mark.parametrize("N", [2, 4])
def test_decoder_stack_gathered_equals_resident(N):
    wl = Workload(L=4, E=16, k=4, H=512, h=256, seed=22)
    lengths = [512, 400, 88]
    T = sum(lengths)
    cu = _cu(lengths)
    x = wl.tokens(T)
    ref = _decoder_stack(wl, T).run(x, cu_seqlens=cu).clone()
    st = _decoder_stack(wl, T, world_size=N)
    sh = st.peer_shards()
    for _ in range(2):  # the second pass reuses both slots
        out = st.run(x, cu_seqlens=cu, local_shards=sh).clone()
        torch.cuda.synchronize()
        assert torch.equal(_bits(out), _bits(ref))
