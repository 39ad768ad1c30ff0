"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no routing, no MLP, no combine):
it only draws the random tensors a run consumes, with the shapes and value laws of
SURVEY.md S8(d) / DESIGN.md S4 ("input recipe").

Generator: a counter-based hash (Wellons' "lowbias32", 32-bit) evaluated with plain
torch integer ops, so the SAME call produces bit-identical tensors on CPU (for the
oracle) and on CUDA (for the device path, e.g. the 38.7 GB weight stack that would be
far too slow to draw on the host and copy):

    key      = H(H(seed) ^ H(tensor_id))
    h_a, h_b = H(key ^ H(2i)), H(key ^ H(2i+1))            for element i
    s        = lo16(h_a) + hi16(h_a) + lo16(h_b) + hi16(h_b) - 131070   (integer, exact)
    value    = bf16_rne( fp32(s) * fp32(std / sigma_IH) )   sigma_IH = sqrt((2^32-1)/3)

s is an Irwin-Hall(4) sum of 16-bit uniforms: mean 0, unit variance after scaling,
support +-3.46 sigma (a bounded stand-in for N(0, std^2)).  Every step is exact
integer arithmetic followed by one correctly rounded fp32 multiply and one RNE cast,
so CPU and GPU agree bit for bit.
"""
from __future__ import annotations

import math

import torch

M32 = 0xFFFFFFFF
_SIGMA_IH = math.sqrt((2.0 ** 32 - 1.0) / 3.0)  # std of the sum of four U{0..65535}
_CHUNK = 1 << 25

# tensor-id namespaces
KIND_X, KIND_WR, KIND_WG, KIND_WU, KIND_WD, KIND_PERM = 1, 2, 3, 4, 5, 6


def _h32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32 on int64 tensors holding values in [0, 2^32)."""
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & M32
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & M32
    x = x ^ (x >> 16)
    return x


def _h32_int(v: int) -> int:
    v &= M32
    v ^= v >> 16
    v = (v * 0x7FEB352D) & M32
    v ^= v >> 15
    v = (v * 0x846CA68B) & M32
    v ^= v >> 16
    return v


def tensor_id(kind: int, layer: int = 0, expert: int = 0) -> int:
    return ((kind & 0xFF) << 24) | ((layer & 0xFF) << 16) | (expert & 0xFFFF)


def fill_normal_(out: torch.Tensor, seed: int, tid: int, std: float) -> torch.Tensor:
    """Fill ``out`` (any float dtype, contiguous, any device) in place."""
    assert out.is_contiguous()
    key = _h32_int(_h32_int(seed) ^ _h32_int(tid))
    flat = out.view(-1)
    n = flat.numel()
    scale = torch.tensor(std / _SIGMA_IH, dtype=torch.float32, device=out.device)
    for s0 in range(0, n, _CHUNK):
        m = min(_CHUNK, n - s0)
        i2 = torch.arange(2 * s0, 2 * (s0 + m), 2, dtype=torch.int64, device=out.device)
        ha = _h32(_h32(i2) ^ key)
        hb = _h32(_h32(i2 + 1) ^ key)
        s = (ha & 0xFFFF) + (ha >> 16) + (hb & 0xFFFF) + (hb >> 16) - 131070
        v = s.to(torch.float32) * scale
        flat[s0:s0 + m].copy_(v.to(flat.dtype) if flat.dtype != torch.float32 else v)
        del i2, ha, hb, s, v
    return out


def normal(shape, seed: int, tid: int, std: float = 1.0, device="cpu",
           dtype=torch.bfloat16) -> torch.Tensor:
    """bf16 (default) tensor of Irwin-Hall(4) 'normal' values; see module doc."""
    return fill_normal_(torch.empty(shape, dtype=dtype, device=device), seed, tid, std)


def expert_rank_perm(E: int, seed: int, tid_extra: int = 0) -> torch.Tensor:
    """Seeded permutation of range(E) (CPU), by sorting hash keys (ties impossible)."""
    key = _h32_int(_h32_int(seed) ^ _h32_int(tensor_id(KIND_PERM, 0, tid_extra)))
    idx = torch.arange(E, dtype=torch.int64)
    keys = _h32(_h32(idx) ^ key) * E + idx  # unique
    return torch.argsort(keys)


# ----------------------------------------------------------------------------------
# Workload recipe (S4 / SURVEY.md S8(d)): x ~ N(0,1); Wr ~ N(0,1/H);
# Wg, Wu ~ N(0,1/H); Wd ~ N(0,1/h); all bf16.  Zipf skew (R14): x[:,0] = 1 and
# Wr[e,0] = -s * ln(rank_e) with rank a seeded permutation of 1..E.
# ----------------------------------------------------------------------------------

def tokens(T: int, H: int, seed: int, layer: int = 0, device="cpu", zipf_s: float = 0.0):
    x = normal((T, H), seed, tensor_id(KIND_X, layer), 1.0, device)
    if zipf_s:
        x[:, 0] = 1.0
    return x


def router_weight(E: int, H: int, seed: int, layer: int, device="cpu", zipf_s: float = 0.0):
    wr = normal((E, H), seed, tensor_id(KIND_WR, layer), 1.0 / math.sqrt(H), device)
    if zipf_s:
        rank = expert_rank_perm(E, seed, layer).to(torch.float64) + 1.0  # rank_e in 1..E
        col = (-zipf_s * torch.log(rank)).to(torch.bfloat16)
        wr[:, 0] = col.to(wr.device)
    return wr


def expert_weights(E: int, H: int, h: int, seed: int, layer: int, device="cpu",
                   experts: range | None = None):
    """Natural-layout expert weights for experts in ``experts`` (default all):
    (gate [n,h,H], up [n,h,H], down [n,H,h]) bf16.  Expert e's tensors depend only on
    (seed, layer, e), so any subset can be regenerated independently."""
    ex = range(E) if experts is None else experts
    n = len(ex)
    g = torch.empty((n, h, H), dtype=torch.bfloat16, device=device)
    u = torch.empty((n, h, H), dtype=torch.bfloat16, device=device)
    d = torch.empty((n, H, h), dtype=torch.bfloat16, device=device)
    for i, e in enumerate(ex):
        fill_normal_(g[i], seed, tensor_id(KIND_WG, layer, e), 1.0 / math.sqrt(H))
        fill_normal_(u[i], seed, tensor_id(KIND_WU, layer, e), 1.0 / math.sqrt(H))
        fill_normal_(d[i], seed, tensor_id(KIND_WD, layer, e), 1.0 / math.sqrt(h))
    return g, u, d


def expert_weights_fp8(E: int, H: int, h: int, seed: int, layer: int, device="cpu",
                       experts: range | None = None):
    """FP8 experts (reading R6: the model's expert weights ARE e4m3 + per-row scales):
    the bf16 master weights of ``expert_weights`` quantised per output row,
        s = amax_row / 448 (fp32);  code = e4m3_rne( w * (448 / amax_row) ).
    Returns (gate, up, down codes as uint8, gate_scale [n,h], up_scale [n,h], down_scale [n,H]).
    Every step is an IEEE fp32 op or the RNE fp32 -> e4m3 cast, so CPU and GPU agree."""
    g, u, d = expert_weights(E, H, h, seed, layer, device=device, experts=experts)
    out = []
    scales = []
    for w in (g, u, d):
        wf = w.float()
        amax = wf.abs().amax(dim=-1, keepdim=True)
        inv = torch.where(amax > 0, torch.full_like(amax, 448.0) / amax, torch.zeros_like(amax))
        codes = (wf * inv).to(torch.float8_e4m3fn).view(torch.uint8)
        out.append(codes.contiguous())
        # tensor / tensor (IEEE division on both devices; a python-scalar divisor becomes a
        # reciprocal multiply on CUDA)
        scales.append((amax / torch.full_like(amax, 448.0)).squeeze(-1).contiguous())
        del wf
    return out[0], out[1], out[2], scales[0], scales[1], scales[2]


# ----------------------------------------------------------------------------------
# NEXT-3 attention layer recipe (S4, reading R19; Qwen3-235B-A22B attention:
# H=4096, Hq=64, Hkv=4, d=128): W_qkv ~ N(0, 1/H) [(Hq+2Hkv)d, H]; W_o ~ N(0, 1/(Hq d))
# [H, Hq d]; RMSNorm weights 1 + N(0, 0.1^2) (w_ln1 [H], w_qn [d], w_kn [d], w_ln2 [H]).
# Prompt mix: packed prompts of the lengths prompt_lengths() draws.
# ----------------------------------------------------------------------------------
KIND_WQKV, KIND_WO, KIND_LN1, KIND_QN, KIND_KN, KIND_LN2 = 7, 8, 9, 10, 11, 12


def _norm_weight(n: int, seed: int, tid: int, device) -> torch.Tensor:
    # 1 + 0.1 z, rounded once to bf16 (fp32 add of a bf16 value and 1.0 is exact)
    return (normal((n,), seed, tid, 0.1, device).float() + 1.0).to(torch.bfloat16)


def attn_weights(H: int, Hq: int, Hkv: int, d: int, seed: int, layer: int, device="cpu"):
    """(w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2), bf16."""
    w_qkv = normal(((Hq + 2 * Hkv) * d, H), seed, tensor_id(KIND_WQKV, layer), 1.0 / math.sqrt(H), device)
    w_o = normal((H, Hq * d), seed, tensor_id(KIND_WO, layer), 1.0 / math.sqrt(Hq * d), device)
    return (_norm_weight(H, seed, tensor_id(KIND_LN1, layer), device), w_qkv,
            _norm_weight(d, seed, tensor_id(KIND_QN, layer), device),
            _norm_weight(d, seed, tensor_id(KIND_KN, layer), device), w_o,
            _norm_weight(H, seed, tensor_id(KIND_LN2, layer), device))


def prompt_lengths(total: int, mean: int, seed: int, spread: float = 0.5) -> list:
    """Seeded prompt lengths summing to ``total``: uniform in [mean(1-spread), mean(1+spread)]
    (spread 0: all equal to mean), the last prompt takes the remainder."""
    out, left, i = [], total, 0
    while left > 0:
        u = _h32_int(_h32_int(seed) ^ _h32_int(0x5EED0000 + i)) / float(M32)
        n = max(1, int(round(mean * (1.0 - spread + 2.0 * spread * u))))
        n = min(n, left)
        out.append(n)
        left -= n
        i += 1
    return out
