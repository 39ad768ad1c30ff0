"""Pins for the CPU oracle (oracle/), checked against things other than itself:
brute force, closed forms, textbook special cases, invariants and the paper's/SPEC's
worked numbers.  No GPU needed.  Each test names the passage it pins."""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand(shape, std, seed):
    # bf16-representable values (round fp32 to bf16 by truncating mantissa with RNE)
    a = np.random.default_rng(seed).standard_normal(shape).astype(np.float32) * np.float32(std)
    u = a.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def _layer(T=64, H=64, E=8, k=2, h=128, seed=0):
    x = _rand((T, H), 1.0, seed)
    wr = _rand((E, H), 1 / math.sqrt(H), seed + 1)
    wg = _rand((E, h, H), 1 / math.sqrt(H), seed + 2)
    wu = _rand((E, h, H), 1 / math.sqrt(H), seed + 3)
    wd = _rand((E, H, h), 1 / math.sqrt(h), seed + 4)
    return x, wr, wg, wu, wd


# ------------------------------------------------------------------ router (R1-R3)

@pytest.mark.parametrize("T,H,E,k", [(256, 64, 8, 2), (2000, 256, 128, 8), (50, 32, 16, 16)])
def test_topk_matches_brute_force_sort(T, H, E, k):
    x = _rand((T, H), 1.0, 11)
    wr = _rand((E, H), 1 / math.sqrt(H), 12)
    r = oracle.router(x, wr, k)
    lg = x.astype(np.float64) @ wr.astype(np.float64).T  # library matmul, not the oracle loop
    np.testing.assert_allclose(r["logits"], lg, rtol=0, atol=1e-12)
    # brute force: full stable sort by (-logit, id)
    order = np.lexsort((np.broadcast_to(np.arange(E), lg.shape), -lg), axis=1)[:, :k]
    far = r["gap"] > 1e-9
    assert np.array_equal(r["ids"][far], order[far])
    assert np.array_equal(r["counts"], np.bincount(r["ids"].ravel(), minlength=E))
    assert r["counts"].sum() == T * k


def test_routing_weights_sum_to_one_and_match_softmax():
    x, wr, *_ = _layer(T=300, H=64, E=16, k=4)
    r = oracle.router(x, wr, 4)
    np.testing.assert_allclose(r["w"].sum(1), 1.0, atol=1e-12)
    # norm_topk: w equals softmax over the k selected logits (R1 equivalence)
    sel = np.take_along_axis(r["logits"], r["ids"].astype(np.int64), 1)
    ref = np.exp(sel - sel.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    np.testing.assert_allclose(r["w"], ref, atol=1e-12)
    # full softmax over E sums to one and un-normalised weights are its top-k entries
    r0 = oracle.router(x, wr, 4, norm_topk=False)
    p = np.exp(r["logits"] - r["logits"].max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    np.testing.assert_allclose(p.sum(1), 1.0, atol=1e-12)
    np.testing.assert_allclose(r0["w"], np.take_along_axis(p, r["ids"].astype(np.int64), 1), atol=1e-12)
    assert np.all(r0["w"].sum(1) <= 1 + 1e-12)


def test_weights_invariant_to_logit_shift():
    x, wr, *_ = _layer(T=200, H=64, E=8, k=2)
    x = x.copy()
    x[:, 0] = 1.0
    wr2 = wr.copy()
    wr2[:, 0] += np.float32(0.5)  # every logit + 0.5 exactly
    a, b = oracle.router(x, wr, 2), oracle.router(x, wr2, 2)
    assert np.array_equal(a["ids"], b["ids"])
    np.testing.assert_allclose(a["w"], b["w"], atol=1e-12)


def test_tie_breaks_to_lower_expert_id():
    H, E = 8, 6
    wr = _rand((E, H), 0.3, 5)
    wr[4] = wr[1]  # experts 1 and 4 always tie
    wr[1] += 5.0
    wr[4] += 5.0   # ... and are always the top two
    x = np.abs(_rand((10, H), 1.0, 6)) + 0.1
    r = oracle.router(x.astype(np.float32), wr.astype(np.float32), 1)
    assert np.all(r["ids"][:, 0] == 1)
    r2 = oracle.router(x.astype(np.float32), wr.astype(np.float32), 2)
    assert np.all(r2["ids"] == [1, 4])


def test_ids_override_recomputes_weights():
    x, wr, *_ = _layer(T=50, H=64, E=8, k=2)
    forced = np.tile(np.array([[7, 0]], np.int32), (50, 1))
    r = oracle.router(x, wr, 2, ids_in=forced)
    assert np.array_equal(r["ids"], forced)
    sel = np.take_along_axis(r["logits"], forced.astype(np.int64), 1)
    ref = np.exp(sel - sel.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    np.testing.assert_allclose(r["w"], ref, atol=1e-12)


# ------------------------------------------------------------------ layer (R4, R5, R9)

def test_hand_worked_layer():
    g = json.load(open(os.path.join(GOLD, "hand_tiny_layer.json")))
    arr = lambda n: np.array(g[n], np.float32)
    for res, key in ((True, "expected_y_residual"), (False, "expected_y_no_residual")):
        r = oracle.moe_layer(arr("x"), arr("wr"), arr("wg"), arr("wu"), arr("wd"), g["k"], residual=res)
        assert r["ids"].tolist() == g["expected_ids"]
        np.testing.assert_allclose(r["w"], g["expected_w"], rtol=1e-15)
        np.testing.assert_allclose(r["y"], g[key], rtol=1e-15)
        np.testing.assert_allclose(r["gap"], g["expected_gap"], rtol=1e-15)


def test_single_expert_reduces_to_dense_swiglu_ffn():
    """E=1, k=1: the layer is the textbook dense SwiGLU FFN y = x + Wd(silu(Wg x) * Wu x)."""
    x, wr, wg, wu, wd = _layer(T=40, H=64, E=1, k=1, h=96)
    r = oracle.moe_layer(x, wr, wg, wu, wd, 1)
    X = x.astype(np.float64)
    G, U = X @ wg[0].astype(np.float64).T, X @ wu[0].astype(np.float64).T
    A = G / (1 + np.exp(-G)) * U
    ref = X + A @ wd[0].astype(np.float64).T
    np.testing.assert_allclose(r["w"], 1.0, rtol=0, atol=0)
    np.testing.assert_allclose(r["y"], ref, rtol=1e-12, atol=1e-12)


def test_layer_matches_per_token_library_evaluation():
    """Each token: y_t = x_t + sum_j w_tj * FFN_{S_tj}(x_t), evaluated with numpy matmuls."""
    x, wr, wg, wu, wd = _layer(T=64, H=64, E=8, k=2, h=128, seed=3)
    r = oracle.moe_layer(x, wr, wg, wu, wd, 2)
    X = x.astype(np.float64)
    ref = X.copy()
    for t in range(X.shape[0]):
        for j in range(2):
            e = r["ids"][t, j]
            g_, u_ = wg[e].astype(np.float64) @ X[t], wu[e].astype(np.float64) @ X[t]
            ref[t] += r["w"][t, j] * (wd[e].astype(np.float64) @ (g_ / (1 + np.exp(-g_)) * u_))
    np.testing.assert_allclose(r["y"], ref, rtol=1e-12, atol=1e-12)


def test_identity_experts_reproduce_weighted_input_sum():
    """Plumbing pin (north_star): identity experts give y = sum_j w_tj x_t = x_t."""
    x, wr, *_ = _layer(T=100, H=64, E=8, k=2)
    r = oracle.moe_layer(x, wr, 128, None, None, 2, residual=False, identity_experts=True)
    np.testing.assert_allclose(r["y"], x.astype(np.float64), rtol=1e-14, atol=1e-14)
    r2 = oracle.moe_layer(x, wr, 128, None, None, 2, residual=True, identity_experts=True)
    np.testing.assert_allclose(r2["y"], 2 * x.astype(np.float64), rtol=1e-14, atol=1e-14)


def test_expert_index_permutation_invariance():
    """Relabelling experts by pi (router rows and expert weights) leaves y unchanged (to
    fp64 rounding: the full-E softmax denominator is summed in expert-id order, R1);
    ids map through pi; counts permute by pi (north_star pin)."""
    x, wr, wg, wu, wd = _layer(T=96, H=64, E=8, k=2, seed=7)
    pi = np.random.default_rng(1).permutation(8)  # new id of old expert e is inv[e]
    inv = np.argsort(pi)
    a = oracle.moe_layer(x, wr, wg, wu, wd, 2)
    b = oracle.moe_layer(x, wr[pi], wg[pi], wu[pi], wd[pi], 2)
    near = a["gap"] < 1e-12
    assert not near.any()
    np.testing.assert_allclose(a["y"], b["y"], rtol=1e-13, atol=1e-13)
    assert np.array_equal(inv[a["ids"]], b["ids"])
    ca = np.bincount(a["ids"].ravel(), minlength=8)
    cb = np.bincount(b["ids"].ravel(), minlength=8)
    assert np.array_equal(ca, cb[inv])


def test_sharded_then_gathered_weights_equal_unsharded():
    """rank r holds experts [r*E/N,(r+1)*E/N); concatenating the shards
    rank-major restores the layer, and the layer output is unchanged."""
    x, wr, wg, wu, wd = _layer(T=64, H=64, E=8, k=2, seed=9)
    ref = oracle.moe_layer(x, wr, wg, wu, wd, 2)["y"]
    for N in (1, 2, 4, 8):
        per = 8 // N
        shards = [(wg[r * per:(r + 1) * per], wu[r * per:(r + 1) * per], wd[r * per:(r + 1) * per]) for r in range(N)]
        g2 = np.concatenate([s[0] for s in shards])
        u2 = np.concatenate([s[1] for s in shards])
        d2 = np.concatenate([s[2] for s in shards])
        assert g2.tobytes() == wg.tobytes() and u2.tobytes() == wu.tobytes() and d2.tobytes() == wd.tobytes()
        assert np.array_equal(oracle.moe_layer(x, wr, g2, u2, d2, 2)["y"], ref)


def test_empty_batch_is_noop():
    x, wr, wg, wu, wd = _layer(T=1, H=64, E=8, k=2)
    r = oracle.moe_layer(x[:0], wr, wg, wu, wd, 2)
    assert r["y"].shape == (0, 64)


def test_silu_special_values():
    """silu(0) = 0 and silu(z) -> z for large z (R4), through a 1-expert layer."""
    H, h = 2, 1
    x = np.array([[1.0, 0.0]], np.float32)
    wr = np.zeros((1, H), np.float32)
    for gval, expect in ((0.0, 0.0), (40.0, 40.0)):
        wg = np.array([[[gval, 0.0]]], np.float32)
        wu = np.array([[[1.0, 0.0]]], np.float32)
        wd = np.array([[[1.0], [0.0]]], np.float32)
        y = oracle.moe_layer(x, wr, wg, wu, wd, 1, residual=False)["y"]
        assert abs(y[0, 0] - expect) <= 1e-15 * max(1.0, expect)


# ------------------------------------------------------------------ FP8 (R6)

def test_e4m3_decode_known_codes():
    cases = {0x00: 0.0, 0x38: 1.0, 0xB8: -1.0, 0x7E: 448.0, 0x01: 2.0 ** -9, 0x08: 2.0 ** -6,
             0x07: 7 * 2.0 ** -9, 0x3C: 1.5, 0x40: 2.0}
    for c, v in cases.items():
        assert oracle.e4m3_decode_one(c) == v
    assert math.isnan(oracle.e4m3_decode_one(0x7F))
    # monotone over the non-negative finite codes
    vals = [oracle.e4m3_decode_one(c) for c in range(0x7F)]
    assert all(a < b for a, b in zip(vals, vals[1:]))


def test_e4m3_encode_rne_and_saturation():
    assert oracle.e4m3_encode_one(1.0) == 0x38
    assert oracle.e4m3_encode_one(1.0625) == 0x38   # tie between 1.0 (even) and 1.125
    assert oracle.e4m3_encode_one(1.1875) == 0x3A   # tie between 1.125 and 1.25 (even 0x3A)
    assert oracle.e4m3_encode_one(500.0) == 0x7E    # satfinite
    assert oracle.e4m3_encode_one(-1e9) == 0xFE
    for c in range(0x7F):
        assert oracle.e4m3_encode_one(oracle.e4m3_decode_one(c)) == c


# ------------------------------------------------------------------ Eq. 1

def test_threshold_spec_examples():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    e = g["eq1"]
    assert oracle.eq1_threshold(e["t_ep"], e["f_gpu"], e["gamma"]) == pytest.approx(e["T_flops"], rel=1e-12)
    assert oracle.eq1_threshold(0.0, 1e15, 1.2) == 0.0
    c = g["calibrated"]
    assert oracle.calibrated_T(c["gamma"], c["ratio"], 1.0, c["c_dummy"]) == pytest.approx(c["T"], rel=1e-12)
    assert oracle.calibrated_T(1.2, 0.5, 1.0, 7.0) == pytest.approx(1.2 * 7.0, rel=1e-15)  # collapses
    cf = g["closed_form_T_tok"]
    t_tok, t_fl = oracle.saturation_T(cf["E"], cf["k"], 4096, 1536, cf["b"], cf["N"], cf["gamma"], cf["F"], cf["BW"])
    assert t_tok == pytest.approx(cf["T_tok"], rel=1e-12)
    assert t_fl == pytest.approx(cf["T_tok"] * 6 * 8 * 4096 * 1536, rel=1e-12)
    # gather time of the SPEC example: 2,113,929,216 B at 450 GB/s ~= 4.70e-3 s
    t = g["transfer_time"]
    _, tfl = oracle.saturation_T(128, 8, 4096, 1536, 1, 8, 1.0, 1.0, t["bw"])
    assert tfl == pytest.approx(t["bytes"] / t["bw"], rel=1e-12)
    assert tfl == pytest.approx(t["seconds_approx"], rel=1e-3)


def test_threshold_invariants():
    base = dict(E=128, k=8, H=4096, h=1536, bytes_per_elem=2, N=8, gamma=1.2,
                flops_per_s=1.4e15, ag_bytes_per_s=7.5e11)
    T0, _ = oracle.saturation_T(**base)
    assert oracle.saturation_T(**{**base, "N": 1})[0] == 0.0
    assert oracle.saturation_T(**{**base, "H": 2048, "h": 768})[0] == pytest.approx(T0, rel=1e-12)
    assert oracle.saturation_T(**{**base, "gamma": 2.4})[0] == pytest.approx(2 * T0, rel=1e-12)
    fp8 = oracle.saturation_T(**{**base, "bytes_per_elem": 1, "flops_per_s": 2.8e15})[0]
    assert fp8 == pytest.approx(T0, rel=1e-12)
    with pytest.raises(ValueError):
        oracle.saturation_T(**{**base, "gamma": 0.5})


def test_e4m3_fast_encoder_matches_brute_force_definition():
    """The arithmetic encoder used by the emulation mode equals the nearest-code search."""
    rng = np.random.default_rng(0)
    vals = [0.0, -0.0, 448.0, 449.0, 464.0, 480.0, 1e9, -1e9, 2.0 ** -9, 2.0 ** -10, 3 * 2.0 ** -11,
            2.0 ** -6, 2.0 ** -6 * (1 + 1 / 16), 7.5 * 2.0 ** -9]
    codes = [oracle.e4m3_decode_one(c) for c in range(0x7F)]
    for a, b in zip(codes, codes[1:]):  # every midpoint (ties) and its neighbours
        m = (a + b) / 2
        vals += [m, -m, np.nextafter(m, 0), np.nextafter(m, 1e9)]
    vals += list(rng.standard_normal(3000) * 50) + list(rng.standard_normal(2000) * 0.01)
    for v in vals:
        assert oracle.e4m3_encode_fast_one(v) == oracle.e4m3_encode_one(v), v


def test_act_quant_emulation_of_the_input_row():
    """Identity experts + act_quant: y_t = (sum_j w_tj) * Q(x_t), Q = the R6 per-token rule
    evaluated here with the brute-force encoder and numpy fp32 arithmetic."""
    x, wr, *_ = _layer(T=20, H=64, E=8, k=2)
    r = oracle.moe_layer(x, wr, 128, None, None, 2, residual=False, identity_experts=True, act_quant=True)
    for t in range(x.shape[0]):
        row = x[t].astype(np.float32)
        amax = np.float32(np.abs(row).max())
        inv = np.float32(448.0) / amax
        sc = amax / np.float32(448.0)
        q = np.array([oracle.e4m3_decode_one(oracle.e4m3_encode_one(float(np.float32(v * inv)))) for v in row])
        np.testing.assert_allclose(r["y"][t], q * float(sc) * r["w"][t].sum(), rtol=1e-14, atol=0)
    # quantisation error is bounded by half an e4m3 ulp (2^-4 relative) of each element
    assert np.all(np.abs(r["y"] - x) <= np.abs(x) * 2.0 ** -4 + 2.0 ** -9 * np.abs(x).max(1, keepdims=True))


# ------------------------------------------------------------------ FP8 emulation branch (R5, R6)

def _bf16_nearest(v64: float) -> float:
    """bf16 RNE of fp32(v) by choosing between the two neighbouring bf16 values (no bit trick):
    the candidates are fp32(v) truncated to 16 bits and the next bf16 away from zero; the nearer
    wins, an exact tie goes to the one with an even last mantissa bit."""
    f = np.float32(v64)
    if not np.isfinite(f):
        return float(f)
    b = np.array([f], np.float32).view(np.uint32)[0]
    lo_bits = np.uint32(b & np.uint32(0xFFFF0000))
    hi_bits = np.uint32(lo_bits + np.uint32(0x10000))
    lo = np.array([lo_bits], np.uint32).view(np.float32)[0]
    hi = np.array([hi_bits], np.uint32).view(np.float32)[0]
    dlo = abs(float(f) - float(lo))
    dhi = abs(float(hi) - float(f)) if np.isfinite(hi) else abs((2.0 ** 128) * math.copysign(1, f) - float(f))
    if dlo < dhi:
        return float(lo)
    if dhi < dlo:
        return float(hi)
    return float(lo) if ((int(lo_bits) >> 16) & 1) == 0 else float(hi)


def test_to_bf16_rounding_points():
    """The intermediate's bf16 rounding (R5): RNE at ties, sign of zero, inf/NaN pass through,
    overflow past the largest bf16 goes to inf; random values against the nearest-neighbour rule."""
    ulp = 2.0 ** -7
    cases = {1.0 + ulp / 2: 1.0,                      # tie -> even (mantissa 0)
             1.0 + 3 * ulp / 2: 1.0 + 2 * ulp,        # tie -> even (up)
             1.0 + ulp / 2 + 2.0 ** -20: 1.0 + ulp,   # just above the tie -> up
             -(1.0 + ulp / 2): -1.0, 0.0: 0.0, 2.0 ** -133: 2.0 ** -133}
    for v, want in cases.items():
        assert float(oracle.to_bf16([v])[0]) == want, v
    z = oracle.to_bf16([0.0, -0.0])
    assert not np.signbit(z[0]) and np.signbit(z[1])
    sp = oracle.to_bf16([np.inf, -np.inf, np.nan, 3.4e38, -3.4e38])
    assert sp[0] == np.inf and sp[1] == -np.inf and np.isnan(sp[2])
    assert sp[3] == np.inf and sp[4] == -np.inf             # 3.4e38 rounds past 0x7F7F -> inf
    assert float(oracle.to_bf16([3.389e38])[0]) == float(np.array([0x7F7F0000], np.uint32).view(np.float32)[0])
    rng = np.random.default_rng(5)
    v = np.concatenate([rng.standard_normal(4000) * 10.0 ** rng.integers(-30, 30, 4000), rng.standard_normal(500)])
    got = oracle.to_bf16(v)
    want = np.array([_bf16_nearest(a) for a in v], np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def _q_row(v32):
    """R6 per-row e4m3 quantisation with the brute-force nearest-code encoder, numpy fp32."""
    v32 = np.asarray(v32, np.float32)
    amax = np.float32(np.abs(v32).max())
    if amax == 0:
        return np.zeros(v32.shape)
    inv = np.float32(448.0) / amax
    sc = amax / np.float32(448.0)
    return np.array([oracle.e4m3_decode_one(oracle.e4m3_encode_one(float(np.float32(a * inv)))) for a in v32]) * float(sc)


@pytest.mark.parametrize("E,k", [(1, 1), (4, 2)])
def test_act_quant_full_expert_path(E, k):
    """act_quant with real experts (the branch identity experts never reach): per token,
    x -> per-token e4m3, g/u by numpy matmul, silu(g)*u, -> fp32 -> bf16 (nearest-neighbour rule),
    -> per-row e4m3, W_down, weighted sum with the oracle's routing weights.  E=1, k=1 reduces to
    one dense FP8-emulated SwiGLU FFN (weight 1)."""
    T, H, h = 24, 64, 96
    x, wr, wg, wu, wd = _layer(T=T, H=H, E=E, k=k, h=h, seed=7)
    r = oracle.moe_layer(x, wr, wg, wu, wd, k, residual=False, act_quant=True)
    if E == 1:
        assert np.all(r["w"] == 1.0)
    for t in range(T):
        xq = _q_row(x[t])
        y = np.zeros(H)
        for j in range(k):
            e = int(r["ids"][t, j])
            g = wg[e].astype(np.float64) @ xq
            u = wu[e].astype(np.float64) @ xq
            a = g / (1.0 + np.exp(-g)) * u
            ab = np.array([_bf16_nearest(v) for v in a], np.float32)
            y += r["w"][t, j] * (wd[e].astype(np.float64) @ _q_row(ab))
        np.testing.assert_allclose(r["y"][t], y, rtol=1e-12, atol=1e-12 * np.abs(y).max())
    # the order matters: quantising before the bf16 rounding (or skipping it) gives another answer
    plain = oracle.moe_layer(x, wr, wg, wu, wd, k, residual=False, act_quant=False)["y"]
    assert np.abs(plain - r["y"]).max() > 1e-4 * np.abs(plain).max()


# ------------------------------------------------------------------ MX intermediate (R6b)

def _mx_block_brute(v32):
    """R6b by brute force: e = the smallest integer in [-127, 127] with amax <= 448 * 2^e found by
    scanning every candidate, each element encoded by the nearest-code search, decoded, rescaled."""
    v = [float(a) for a in np.asarray(v32, np.float32)]
    amax = max(abs(a) for a in v)
    e = next((c for c in range(-127, 128) if amax <= math.ldexp(448.0, c)), 127)
    return np.array([math.ldexp(oracle.e4m3_decode_one(oracle.e4m3_encode_one(math.ldexp(a, -e))), e) for a in v]), e


def _q_mx(row):
    row = np.asarray(row, np.float32)
    return np.concatenate([_mx_block_brute(row[b:b + 32])[0] for b in range(0, row.size, 32)])


def test_mx_block_rule_against_brute_force():
    """The MX rule (R6b, S3) against the brute-force scale search and nearest-code encoder,
    on blocks spanning 60 decades, all-zero blocks, blocks whose amax sits exactly on 448 * 2^j
    (scale 2^j) or one bf16 ulp above it (2^(j+1)), mixed tiny/large blocks and the clamp at 2^-127."""
    rng = np.random.default_rng(21)
    blocks = []
    for d in range(-30, 31, 3):
        blocks.append(_rand((32,), 10.0 ** d, 100 + d))
    blocks.append(np.zeros(32, np.float32))
    for j in (-20, -3, 0, 5, 30):
        b = _rand((32,), 1.0, 200 + j) * np.float32(2.0 ** j)
        b[7] = np.float32(448.0 * 2.0 ** j)
        blocks.append(b)
        c = b.copy()
        c[7:8] = (c[7:8].view(np.uint32) + np.uint32(0x10000)).view(np.float32)  # next bf16 above
        blocks.append(c)
    mix = _rand((32,), 1e-6, 300)
    mix[0] = np.float32(1000.0)
    blocks.append(mix)
    blocks.append(np.full(32, np.float32(2.0 ** -133)))  # below 448 * 2^-127 / 2^... -> e clamps at -127
    row = np.concatenate(blocks).astype(np.float32)
    got = oracle.quant_row_mx(row)
    want = np.concatenate([_mx_block_brute(row[b:b + 32])[0] for b in range(0, row.size, 32)])
    assert np.array_equal(got, want)
    # the scale each block took: exactly 2^j on the boundary, 2^(j+1) one ulp above it
    for j in (-20, -3, 0, 5, 30):
        b = _rand((32,), 1.0, 200 + j) * np.float32(2.0 ** j)
        b[7] = np.float32(448.0 * 2.0 ** j)
        assert _mx_block_brute(b)[1] == j
        assert oracle.quant_row_mx(b)[7] == 448.0 * 2.0 ** j   # the amax element is exact
        b[7:8] = (b[7:8].view(np.uint32) + np.uint32(0x10000)).view(np.float32)
        assert _mx_block_brute(b)[1] == j + 1
    assert _mx_block_brute(np.full(32, np.float32(2.0 ** -133)))[1] == -127
    # invariants: no element saturates; every block's largest code lies in (224, 448] * 2^e
    for b0 in range(0, row.size, 32):
        q, e = _mx_block_brute(row[b0:b0 + 32])
        if np.abs(row[b0:b0 + 32]).max() > math.ldexp(448.0, -127):
            assert 224.0 * 2.0 ** e <= np.abs(q).max() <= 448.0 * 2.0 ** e
    # e4m3-representable values times a power of two come back exactly
    codes = np.array([oracle.e4m3_decode_one(c) for c in range(0, 0x7F)], np.float64)
    exact = (rng.choice(codes, 64) * rng.choice([-1, 1], 64) * 2.0 ** 7).astype(np.float32)
    exact[3] = 448.0 * 2.0 ** 7
    exact[40] = -448.0 * 2.0 ** 7
    assert np.array_equal(oracle.quant_row_mx(exact), exact.astype(np.float64))


@pytest.mark.parametrize("E,k", [(1, 1), (4, 2)])
def test_act_quant_mx_full_expert_path(E, k):
    """act_quant="mx" with real experts: per token, x -> per-token e4m3 (R6), g/u by numpy matmul,
    silu(g)*u -> bf16 (nearest-neighbour rule) -> MX blocks of 32 (brute force), W_down, weighted sum
    with the oracle's routing weights.  E=1, k=1 is one dense FP8-emulated SwiGLU FFN."""
    T, H, h = 16, 64, 96
    x, wr, wg, wu, wd = _layer(T=T, H=H, E=E, k=k, h=h, seed=9)
    r = oracle.moe_layer(x, wr, wg, wu, wd, k, residual=False, act_quant="mx")
    for t in range(T):
        xq = _q_row(x[t])
        y = np.zeros(H)
        for j in range(k):
            e = int(r["ids"][t, j])
            g = wg[e].astype(np.float64) @ xq
            u = wu[e].astype(np.float64) @ xq
            a = g / (1.0 + np.exp(-g)) * u
            ab = np.array([_bf16_nearest(v) for v in a], np.float32)
            y += r["w"][t, j] * (wd[e].astype(np.float64) @ _q_mx(ab))
        np.testing.assert_allclose(r["y"][t], y, rtol=1e-12, atol=1e-12 * np.abs(y).max())
    # a different rule from the per-row one (R6), and both close to the unquantised intermediate
    row = oracle.moe_layer(x, wr, wg, wu, wd, k, residual=False, act_quant=True)["y"]
    assert np.abs(row - r["y"]).max() > 1e-6 * np.abs(row).max()
    assert np.abs(row - r["y"]).max() < 0.1 * np.abs(row).max()
