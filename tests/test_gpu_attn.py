"""NEXT-3 parity on B200: the tcgen05 flash-attention core and the full DP attention layer
(reading R19) through the C ABI, against the fp64 oracle (oracle/attn_oracle.c).

Tolerance: the R7 metric err = max|y - y*| / max|y*| <= 2e-2 (the north_star BF16 bound);
the attention core alone is held to 1e-2 (its only roundings are the bf16 P and output)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import f32
from parity import output_error
from paper_2605_02960_b200 import asyncep as A

pytestmark = pytest.mark.gpu


def _err(got, ref):
    return output_error(got, ref)["err"]


def _cu(lengths):
    return np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)


def _core(lengths, Hq, Hkv, seed, rows=None, scale_q=1.0):
    cu = _cu(lengths)
    T = int(cu[-1])
    d = 128
    q = synth.normal((T, Hq, d), seed, 0xA1, scale_q, "cuda")
    k = synth.normal((T, Hkv, d), seed, 0xA2, 1.0, "cuda")
    v = synth.normal((T, Hkv, d), seed, 0xA3, 1.0, "cuda")
    # V^T with every prompt starting on a multiple of 8 columns (the ABI's alignment rule)
    vcu = np.concatenate([[0], np.cumsum([(n + 7) // 8 * 8 for n in lengths])]).astype(np.int32)
    ldv = int(vcu[-1]) + 8
    vt = torch.zeros((Hkv, d, ldv), dtype=torch.bfloat16, device="cuda")
    for b, n in enumerate(lengths):
        vt[:, :, vcu[b]:vcu[b] + n] = v[cu[b]:cu[b + 1]].permute(1, 2, 0)
    o = torch.full((T, Hq, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    cfg = A.make_attn_config(256, Hq, Hkv, d, max_tokens=T)  # hidden unused by the core
    A.asyncep_attention(cfg, q, k, vt, ldv, torch.from_numpy(vcu).cuda(), torch.from_numpy(cu).cuda(), o)
    torch.cuda.synchronize()
    sel = np.arange(T) if rows is None else np.asarray(rows)
    ref = oracle.attention(f32(q)[sel], f32(k), f32(v), cu, rows=None if rows is None else sel)
    return f32(o)[sel], ref


@pytest.mark.parametrize("lengths", [[1], [128], [129], [127, 1, 300], [64, 257, 128, 5, 700], [1000, 24]])
def test_attention_core_parity(lengths):
    got, ref = _core(lengths, Hq=8, Hkv=2, seed=3)
    assert np.isfinite(got).all()
    err = _err(got.reshape(got.shape[0], -1), ref.reshape(ref.shape[0], -1))
    assert err <= 1e-2, err


def test_attention_core_peaked_scores():
    # larger score spread (q scaled 4x): exercises the running-max rescale of O in TMEM
    got, ref = _core([900, 400], Hq=4, Hkv=1, seed=5, scale_q=4.0)
    err = _err(got.reshape(got.shape[0], -1), ref.reshape(ref.shape[0], -1))
    assert err <= 1e-2, err


def test_attention_core_qwen3_heads_sampled():
    """Qwen3-235B attention heads (Hq=64, Hkv=4) over 4 prompts of 2,048 tokens; 48 sampled rows."""
    lengths = [2048] * 4
    rows = np.unique(np.concatenate([[0, 127, 128, 2047, 2048, 8191],
                                     np.random.default_rng(1).choice(8192, 42, replace=False)]))
    got, ref = _core(lengths, Hq=64, Hkv=4, seed=7, rows=rows)
    err = _err(got.reshape(got.shape[0], -1), ref.reshape(ref.shape[0], -1))
    assert err <= 1e-2, err


@pytest.mark.parametrize("lengths", [[32768], [4096] * 8], ids=["one_32k_prompt", "eight_4k_prompts"])
def test_attention_core_bench_shapes_sampled(lengths):
    """The bench's attention configurations at full size (32,768 tokens, Qwen3-235B heads):
    sampled rows near tile / prompt boundaries and at random, against the oracle."""
    T = sum(lengths)
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([[0, 127, 128, 255, 256, 4095, 4096, T - 1], rng.choice(T, 16, replace=False)]))
    got, ref = _core(lengths, Hq=64, Hkv=4, seed=17, rows=rows)
    err = _err(got.reshape(got.shape[0], -1), ref.reshape(ref.shape[0], -1))
    assert err <= 1e-2, err


def _layer(H, Hq, Hkv, lengths, seed, rows=None):
    d = 128
    cu = _cu(lengths)
    T = int(cu[-1])
    ws_w = synth.attn_weights(H, Hq, Hkv, d, seed, 0, device="cuda")
    x = synth.tokens(T, H, seed + 1, device="cuda")
    cfg = A.make_attn_config(H, Hq, Hkv, d, max_tokens=T)
    ws = torch.empty(A.asyncep_attn_workspace_size(cfg), dtype=torch.uint8, device="cuda")
    xo = torch.empty_like(x)
    xn2 = torch.empty_like(x)
    A.asyncep_attn_layer(cfg, x, torch.from_numpy(cu).cuda(), ws_w, xo, xn2, ws)
    torch.cuda.synchronize()
    hw = [f32(w) for w in ws_w]
    ref_x, ref_n = oracle.attn_layer(f32(x), cu, Hq, Hkv, d, *hw, rows=rows)
    sel = slice(None) if rows is None else np.asarray(rows)
    return f32(xo)[sel], f32(xn2)[sel], ref_x, ref_n, f32(x)[sel]


def test_attn_layer_parity_small():
    got_x, got_n, ref_x, ref_n, x = _layer(512, 8, 2, [300, 1, 129, 250], seed=11)
    # the attention contribution x' - x is checked on its own scale as well as the sum
    assert _err(got_x - x, ref_x - x) <= 2e-2
    assert _err(got_x, ref_x) <= 2e-2
    assert _err(got_n, ref_n) <= 2e-2


def test_attn_layer_parity_qwen3_shape_sampled():
    rows = np.array([0, 1, 127, 128, 600, 1023, 1024, 1500, 2047])
    got_x, got_n, ref_x, ref_n, x = _layer(4096, 64, 4, [1024, 1024], seed=13, rows=rows)
    assert _err(got_x - x, ref_x - x) <= 2e-2
    assert _err(got_n, ref_n) <= 2e-2


def test_attn_layer_deterministic_and_empty():
    H, Hq, Hkv, d = 512, 8, 2, 128
    lengths = [700, 300]
    cu = torch.from_numpy(_cu(lengths)).cuda()
    w = synth.attn_weights(H, Hq, Hkv, d, 2, 0, device="cuda")
    x = synth.tokens(1000, H, 3, device="cuda")
    cfg = A.make_attn_config(H, Hq, Hkv, d, max_tokens=1000)
    ws = torch.empty(A.asyncep_attn_workspace_size(cfg), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(2):
        xo, xn = torch.empty_like(x), torch.empty_like(x)
        A.asyncep_attn_layer(cfg, x, cu, w, xo, xn, ws)
        outs.append((xo.clone(), xn.clone()))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
    assert torch.equal(outs[0][1].view(torch.int16), outs[1][1].view(torch.int16))
    # T = 0 is a no-op; T > max_tokens is rejected
    A.asyncep_attn_layer(cfg, x[:0], torch.zeros(2, dtype=torch.int32, device="cuda"), w, xo[:0], xn[:0], ws)
    with pytest.raises(A.AsyncEPError):
        big = synth.tokens(1001, H, 3, device="cuda")
        A.asyncep_attn_layer(cfg, big, torch.tensor([0, 1001], dtype=torch.int32, device="cuda"), w,
                             torch.empty_like(big), torch.empty_like(big), ws)


def test_attention_concurrent_streams_bitwise():
    """Two attention calls in flight at once on two streams (each with its own scheduler
    counter) give bitwise the outputs of serial calls (a shared global counter let
    one launch take the other's work items)."""
    lengths = [3000, 1100, 700]
    cu = _cu(lengths)
    T, d, Hq, Hkv = int(cu[-1]), 128, 16, 4
    vcu = np.concatenate([[0], np.cumsum([(n + 7) // 8 * 8 for n in lengths])]).astype(np.int32)
    ldv = int(vcu[-1]) + 8
    cfg = A.make_attn_config(256, Hq, Hkv, d, max_tokens=T)
    cu_d, vcu_d = torch.from_numpy(cu).cuda(), torch.from_numpy(vcu).cuda()
    ins = []
    for seed in (11, 12):
        q = synth.normal((T, Hq, d), seed, 0xA1, 1.0, "cuda")
        k = synth.normal((T, Hkv, d), seed, 0xA2, 1.0, "cuda")
        vt = synth.normal((Hkv, d, ldv), seed, 0xA3, 1.0, "cuda")
        ins.append((q, k, vt))
    serial = []
    for q, k, vt in ins:
        o = torch.empty((T, Hq, d), dtype=torch.bfloat16, device="cuda")
        A.asyncep_attention(cfg, q, k, vt, ldv, vcu_d, cu_d, o)
        serial.append(o)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty((T, Hq, d), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    for rep in range(3):
        for (q, k, vt), o, s in zip(ins, outs, streams):
            o.fill_(float("nan"))
        torch.cuda.synchronize()
        for (q, k, vt), o, s in zip(ins, outs, streams):
            A.asyncep_attention(cfg, q, k, vt, ldv, vcu_d, cu_d, o, stream=s)
        torch.cuda.synchronize()
        for o, ref in zip(outs, serial):
            assert torch.equal(o.view(torch.int16), ref.view(torch.int16))
