"""Pins of the NEXT-3 attention oracle (oracle/attn_oracle.c) against closed forms, textbook
reductions and invariants -- not against itself (S2).  CPU only."""
import numpy as np
import pytest

import oracle
import synth


def _rng(s=0):
    return np.random.default_rng(s)


# ------------------------------------------------------------------ RMSNorm
def test_rmsnorm_unit_rms_and_scale_invariance():
    x = _rng(1).standard_normal((7, 96)).astype(np.float32)
    eps = 1e-6
    y = oracle.rmsnorm(x, None, eps)
    ms = (x.astype(np.float64) ** 2).mean(1)
    # closed form: mean(y^2) = ms / (ms + eps)
    np.testing.assert_allclose((y ** 2).mean(1), ms / (ms + eps), rtol=1e-12)
    # eps = 0: invariant to a positive scale of the row
    np.testing.assert_allclose(oracle.rmsnorm(4.0 * x, None, 0.0), oracle.rmsnorm(x, None, 0.0), rtol=1e-12)
    # the weight multiplies column-wise
    w = _rng(2).standard_normal(96).astype(np.float32)
    np.testing.assert_allclose(oracle.rmsnorm(x, w, eps), y * w, rtol=1e-12)


# ------------------------------------------------------------------ RoPE
def test_rope_identity_at_zero_and_norm_preserving():
    x = _rng(3).standard_normal((5, 3, 64))
    np.testing.assert_array_equal(oracle.rope(x, np.zeros(5), 1e6), x)
    y = oracle.rope(x, np.arange(5) * 977, 1e6)
    pairs = lambda a: a[..., :32] ** 2 + a[..., 32:] ** 2  # noqa: E731  rotate-half pairs (i, i + d/2)
    np.testing.assert_allclose(pairs(y), pairs(x), rtol=1e-12, atol=1e-12)


def test_rope_d2_is_complex_rotation():
    # d = 2: inv_freq_0 = theta^0 = 1, so the pair rotates by pos radians: (a + ib) e^{i pos}
    x = _rng(4).standard_normal((6, 1, 2))
    pos = np.array([0, 1, 2, 5, 100, 31337])
    z = (x[:, 0, 0] + 1j * x[:, 0, 1]) * np.exp(1j * pos)
    y = oracle.rope(x, pos, 1e6)
    np.testing.assert_allclose(y[:, 0, 0], z.real, atol=1e-12)
    np.testing.assert_allclose(y[:, 0, 1], z.imag, atol=1e-12)


def test_rope_scores_depend_on_relative_position_only():
    q = _rng(5).standard_normal((1, 1, 128))
    k = _rng(6).standard_normal((1, 1, 128))
    s = [float((oracle.rope(q, [m + sh], 1e6) * oracle.rope(k, [n + sh], 1e6)).sum())
         for (m, n, sh) in ((10, 3, 0), (10, 3, 1000), (10, 3, 54321))]
    np.testing.assert_allclose(s, s[0], rtol=1e-9)


# ------------------------------------------------------------------ attention
def _qkv(T, Hq, Hkv, d, seed):
    r = _rng(seed)
    return (r.standard_normal((T, Hq, d)), r.standard_normal((T, Hkv, d)), r.standard_normal((T, Hkv, d)))


def test_attention_uniform_scores_give_prefix_means():
    cu = [0, 5, 12, 13]
    T = cu[-1]
    q, k, v = _qkv(T, 4, 2, 8, 7)
    q[:] = 0.0  # every score 0 -> uniform softmax over the visible keys
    o = oracle.attention(q, k, v, cu, causal=True)
    for b in range(3):
        s, e = cu[b], cu[b + 1]
        pref = np.cumsum(v[s:e], 0) / np.arange(1, e - s + 1)[:, None, None]  # [n, Hkv, d]
        np.testing.assert_allclose(o[s:e], np.repeat(pref, 2, axis=1), rtol=1e-12, atol=1e-12)
    onc = oracle.attention(q, k, v, cu, causal=False)  # non-causal: full-prompt mean
    for b in range(3):
        s, e = cu[b], cu[b + 1]
        np.testing.assert_allclose(onc[s:e], np.repeat(v[s:e].mean(0, keepdims=True), 2, 1).repeat(e - s, 0),
                                   rtol=1e-12, atol=1e-12)


def test_attention_single_token_prompts_return_v():
    cu = np.arange(6)
    q, k, v = _qkv(5, 8, 2, 16, 8)
    o = oracle.attention(q, k, v, cu)
    np.testing.assert_allclose(o, np.repeat(v, 4, axis=1), rtol=1e-14)


def test_attention_hard_selection():
    # orthogonal keys, a query aligned with key m at large scale -> o ~= v_m
    T, d = 16, 16
    k = (np.eye(d)[:T] * 1.0)[:, None, :]
    v = _rng(9).standard_normal((T, 1, d))
    q = np.zeros((T, 1, d))
    for t in range(T):
        q[t, 0, t // 2] = 60.0  # the query at t picks key t // 2 (visible: t // 2 <= t)
    o = oracle.attention(q, k, v, [0, T], scale=1.0)
    np.testing.assert_allclose(o[:, 0], v[np.arange(T) // 2, 0], atol=1e-20 + 1e-12 * np.abs(v).max())


def test_attention_causality_packing_gqa_shift_rows():
    cu = np.array([0, 37, 38, 100, 161])
    T = int(cu[-1])
    q, k, v = _qkv(T, 8, 2, 32, 10)
    o = oracle.attention(q, k, v, cu)
    # causality: perturbing token 70 and later of prompt 2 leaves its earlier rows unchanged
    k2, v2, q2 = k.copy(), v.copy(), q.copy()
    k2[70:100] += 3.0
    v2[70:100] -= 1.0
    q2[70:100] *= 2.0
    o2 = oracle.attention(q2, k2, v2, cu)
    assert np.array_equal(o2[:70], o[:70]) and np.array_equal(o2[100:], o[100:])
    assert not np.allclose(o2[70:100], o[70:100])
    # packing order: prompts reversed in the pack give the same per-prompt rows
    segs = [(int(cu[b]), int(cu[b + 1])) for b in range(4)][::-1]
    perm = np.concatenate([np.arange(s, e) for s, e in segs])
    cu_r = np.concatenate([[0], np.cumsum([e - s for s, e in segs])])
    o_r = oracle.attention(q[perm], k[perm], v[perm], cu_r)
    assert np.array_equal(o_r, o[perm])
    # GQA == MHA with each kv head repeated over its query group
    o_m = oracle.attention(q, np.repeat(k, 4, 1), np.repeat(v, 4, 1), cu)
    assert np.array_equal(o_m, o)
    # adding one vector to every key shifts each query's scores by a constant -> same output
    o_s = oracle.attention(q, k + _rng(11).standard_normal((1, 2, 32)), v, cu)
    np.testing.assert_allclose(o_s, o, rtol=1e-9, atol=1e-11)
    # a row subset evaluates exactly those rows
    rows = np.array([0, 36, 37, 99, 160])
    assert np.array_equal(oracle.attention(q[rows], k, v, cu, rows=rows), o[rows])


# ------------------------------------------------------------------ the layer
def _layer_weights(H, Hq, Hkv, d, seed=0):
    return [a.float().numpy() for a in synth.attn_weights(H, Hq, Hkv, d, seed, 0)]


def test_attn_layer_zero_output_projection_and_single_token_prompts():
    H, Hq, Hkv, d = 64, 4, 2, 16
    w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2 = _layer_weights(H, Hq, Hkv, d)
    x = synth.tokens(9, H, 3).float().numpy()
    cu = [0, 4, 9]
    # W_o = 0: the residual passes through exactly and xn2 = RMSNorm(x; w_ln2)
    xo, xn2 = oracle.attn_layer(x, cu, Hq, Hkv, d, w_ln1, w_qkv, w_qn, w_kn, np.zeros_like(w_o), w_ln2)
    assert np.array_equal(xo, x)
    np.testing.assert_allclose(xn2, oracle.rmsnorm(x, w_ln2), rtol=1e-6)
    # single-token prompts: attention returns v, so the layer is dense linear algebra:
    # x' = x + W_o . repeat_groups(W_v . RMSNorm(x; w_ln1))   (norms/RoPE on q, k drop out)
    cu1 = np.arange(10)
    xo1, _ = oracle.attn_layer(x, cu1, Hq, Hkv, d, w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2)
    xn = oracle.rmsnorm(x, w_ln1)
    vv = xn @ w_qkv[(Hq + Hkv) * d:].astype(np.float64).T            # [T, Hkv d]
    o = np.repeat(vv.reshape(9, Hkv, d), Hq // Hkv, axis=1).reshape(9, Hq * d)
    np.testing.assert_allclose(xo1, x + o @ w_o.astype(np.float64).T, rtol=1e-5, atol=1e-5)


def test_attn_layer_wiring_and_row_subset():
    """The layer equals its definition assembled from independently pinned parts: numpy
    matmuls for the projections, oracle RMSNorm / RoPE / attention for the rest."""
    H, Hq, Hkv, d = 64, 4, 2, 16
    w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2 = _layer_weights(H, Hq, Hkv, d, 1)
    cu = np.array([0, 7, 20, 21, 33])
    T = int(cu[-1])
    x = synth.tokens(T, H, 4).float().numpy()
    xo, xn2 = oracle.attn_layer(x, cu, Hq, Hkv, d, w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2)
    pos = np.concatenate([np.arange(cu[b + 1] - cu[b]) for b in range(len(cu) - 1)])
    qkv = oracle.rmsnorm(x, w_ln1) @ w_qkv.astype(np.float64).T
    q = qkv[:, :Hq * d].reshape(T, Hq, d)
    k = qkv[:, Hq * d:(Hq + Hkv) * d].reshape(T, Hkv, d)
    v = qkv[:, (Hq + Hkv) * d:].reshape(T, Hkv, d)
    q = oracle.rope(oracle.rmsnorm(q.astype(np.float32), w_qn).reshape(T, Hq, d), pos)
    k = oracle.rope(oracle.rmsnorm(k.astype(np.float32), w_kn).reshape(T, Hkv, d), pos)
    o = oracle.attention(q, k, v, cu).reshape(T, Hq * d)
    ref = x + o @ w_o.astype(np.float64).T
    # (the fp32 casts above round q, k before their norms: tolerance covers that)
    np.testing.assert_allclose(xo, ref, rtol=1e-4, atol=1e-4)
    np.testing.assert_allclose(xn2, oracle.rmsnorm(ref.astype(np.float32), w_ln2), rtol=1e-4, atol=1e-4)
    rows = np.array([0, 6, 19, 20, 32])
    xs, ns = oracle.attn_layer(x, cu, Hq, Hkv, d, w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2, rows=rows)
    assert np.array_equal(xs, xo[rows]) and np.array_equal(ns, xn2[rows])
