"""CPU oracle for the AsyncEP MoE hot path -- TEST INFRASTRUCTURE ONLY.

Plain fp64 C implementation (``oracle/moe_oracle.c``) of what the path computes, by
definition (S2.2; Eq. 1 at PAPER.md:315-319).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package.  It shares no code with ``paper_2605_02960_b200`` and
never imports it.

Every function here only marshals numpy arrays into the C library.
Parity pins for each function live in ``tests/test_oracle_*.py``; S3 lists
the readings (R1..R15) of points the paper leaves open.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "moe_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "attn_oracle.c")]
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# -ffp-contract=off: no fused multiply-add, every product and sum is one IEEE fp64 op.
CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            I64, I32, D = ctypes.c_int64, ctypes.c_int, ctypes.c_double
            lib.oracle_router.argtypes = [P, P, I64, I32, I32, I32, I32, P, P, P, P, P, P]
            lib.oracle_router.restype = I32
            lib.oracle_moe_layer.argtypes = [P, P, P, P, P, I64, I32, I32, I32, I32, I32, I32, I32, I32,
                                             P, P, P, P, P, P]
            lib.oracle_moe_layer.restype = I32
            lib.oracle_e4m3_decode.argtypes = [ctypes.c_uint8]
            lib.oracle_e4m3_decode.restype = D
            lib.oracle_e4m3_encode.argtypes = [D]
            lib.oracle_e4m3_encode.restype = ctypes.c_uint8
            lib.oracle_e4m3_encode_fast.argtypes = [D]
            lib.oracle_e4m3_encode_fast.restype = ctypes.c_uint8
            lib.oracle_e4m3_decode_array.argtypes = [P, I64, P]
            lib.oracle_e4m3_decode_array.restype = None
            lib.oracle_to_bf16_array.argtypes = [P, I64, P]
            lib.oracle_to_bf16_array.restype = None
            lib.oracle_quant_row_mx.argtypes = [P, I32, P]
            lib.oracle_quant_row_mx.restype = None
            lib.oracle_eq1_threshold.argtypes = [D, D, D]
            lib.oracle_eq1_threshold.restype = D
            lib.oracle_saturation_T.argtypes = [I32, I32, I32, I32, D, I32, D, D, D, P, P]
            lib.oracle_saturation_T.restype = I32
            lib.oracle_calibrated_T.argtypes = [D, D, D, D]
            lib.oracle_calibrated_T.restype = D
            lib.oracle_rmsnorm.argtypes = [P, P, I64, I32, D, P]
            lib.oracle_rmsnorm.restype = I32
            lib.oracle_rope.argtypes = [P, P, I64, I32, I32, D]
            lib.oracle_rope.restype = I32
            lib.oracle_attention.argtypes = [P, P, P, P, I32, I32, I32, I32, I32, D, P, I64, P]
            lib.oracle_attention.restype = I32
            lib.oracle_attn_layer.argtypes = [P, I64, I32, P, I32, I32, I32, I32, P, P, P, P, P, P, D, D, P, I64,
                                              P, P]
            lib.oracle_attn_layer.restype = I32
            lib.oracle_num_threads.argtypes = []
            lib.oracle_num_threads.restype = I32
            lib.oracle_set_num_threads.argtypes = [I32]
            lib.oracle_set_num_threads.restype = None
            _lib = lib
    return _lib


def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))


def router(x, wr, k: int, norm_topk: bool = True, ids_in=None):
    """Router of T tokens (readings R1-R3, R15).

    x [T,H], wr [E,H] -> dict(logits [T,E] f64, ids [T,k] i32, w [T,k] f64,
    counts [E] i64, gap [T] f64 = logit_(k) - logit_(k+1)).
    """
    x, wr = _f32(x), _f32(wr)
    T, H = x.shape
    E = wr.shape[0]
    assert wr.shape[1] == H
    logits = np.empty((T, E), np.float64)
    ids = np.empty((T, k), np.int32)
    w = np.empty((T, k), np.float64)
    counts = np.empty((E,), np.int64)
    gap = np.empty((T,), np.float64)
    if ids_in is not None:
        ids_in = np.ascontiguousarray(ids_in, dtype=np.int32)
    rc = _load().oracle_router(_ptr(x), _ptr(wr), T, H, E, k, int(norm_topk), _ptr(ids_in),
                               _ptr(logits), _ptr(ids), _ptr(w), _ptr(counts), _ptr(gap))
    if rc:
        raise ValueError(f"oracle_router rc={rc}")
    return dict(logits=logits, ids=ids, w=w, counts=counts, gap=gap)


def moe_layer(x, wr, wg, wu, wd, k: int, norm_topk: bool = True, residual: bool = True,
              identity_experts: bool = False, ids_in=None, act_quant=False):
    """One MoE FFN layer by definition (R1-R5, R9, R15).

    x [T,H]; wr [E,H]; wg, wu [E,h,H]; wd [E,H,h] (natural layout, fp32 holding exact
    bf16/e4m3-dequantised values).  act_quant emulates the FP8 path's activation
    quantisation (R6: per-token e4m3 x, bf16 then per-row e4m3 intermediate); act_quant="mx"
    the MX variant (R6b: per-token e4m3 x, bf16 then 1x32 blocks with E8M0 scales).
    Returns dict(y [T,H] f64, ids, w, logits, gap).
    """
    x, wr = _f32(x), _f32(wr)
    T, H = x.shape
    E = wr.shape[0]
    if identity_experts:
        h = int(wg) if isinstance(wg, int) else 64
        wg_p = wu_p = wd_p = None
    else:
        wg, wu, wd = _f32(wg), _f32(wu), _f32(wd)
        h = wg.shape[1]
        assert wg.shape == (E, h, H) and wu.shape == (E, h, H) and wd.shape == (E, H, h)
        wg_p, wu_p, wd_p = _ptr(wg), _ptr(wu), _ptr(wd)
    y = np.empty((T, H), np.float64)
    ids = np.empty((T, k), np.int32)
    w = np.empty((T, k), np.float64)
    logits = np.empty((T, E), np.float64)
    gap = np.empty((T,), np.float64)
    if ids_in is not None:
        ids_in = np.ascontiguousarray(ids_in, dtype=np.int32)
    rc = _load().oracle_moe_layer(_ptr(x), _ptr(wr), wg_p, wu_p, wd_p, T, H, E, k, h,
                                  int(norm_topk), int(residual), int(identity_experts),
                                  2 if act_quant == "mx" else int(bool(act_quant)), _ptr(ids_in), _ptr(y), _ptr(ids), _ptr(w), _ptr(logits), _ptr(gap))
    if rc:
        raise ValueError(f"oracle_moe_layer rc={rc}")
    return dict(y=y, ids=ids, w=w, logits=logits, gap=gap)


def e4m3_decode(q) -> np.ndarray:
    """OCP E4M3 bytes -> float32 values (exact)."""
    q = np.ascontiguousarray(q, dtype=np.uint8)
    out = np.empty(q.shape, np.float32)
    _load().oracle_e4m3_decode_array(_ptr(q), q.size, _ptr(out))
    return out


def to_bf16(v) -> np.ndarray:
    """fp64 values -> fp32 -> bf16 round-to-nearest-even (as float32 arrays): the rounding the
    act_quant emulation applies to the intermediate (R5)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty(v.shape, np.float32)
    _load().oracle_to_bf16_array(_ptr(v), v.size, _ptr(out))
    return out


def quant_row_mx(v) -> np.ndarray:
    """The MX intermediate rule (R6b) over one row (length a multiple of 32), fp64 result."""
    v = _f32(v).ravel()
    assert v.size % 32 == 0
    out = np.empty(v.shape, np.float64)
    _load().oracle_quant_row_mx(_ptr(v), v.size, _ptr(out))
    return out


def e4m3_decode_one(b: int) -> float:
    return _load().oracle_e4m3_decode(b)


def e4m3_encode_one(v: float) -> int:
    """RNE satfinite encode by brute-force nearest search (R6)."""
    return int(_load().oracle_e4m3_encode(float(v)))


def e4m3_encode_fast_one(v: float) -> int:
    """The arithmetic RNE satfinite encoder the emulation mode uses."""
    return int(_load().oracle_e4m3_encode_fast(float(v)))


def eq1_threshold(t_ep: float, f_gpu: float, gamma: float) -> float:
    """Eq. 1: T = t_EP * F_GPU * gamma [FLOPs]."""
    return _load().oracle_eq1_threshold(t_ep, f_gpu, gamma)


def saturation_T(E, k, H, h, bytes_per_elem, N, gamma, flops_per_s, ag_bytes_per_s):
    """Per-layer Eq. 1 in tokens/GPU (readings R11, R12) -> (T_tok, T_flops)."""
    t_tok = ctypes.c_double()
    t_fl = ctypes.c_double()
    rc = _load().oracle_saturation_T(E, k, H, h, float(bytes_per_elem), N, float(gamma),
                                     float(flops_per_s), float(ag_bytes_per_s),
                                     ctypes.byref(t_tok), ctypes.byref(t_fl))
    if rc:
        raise ValueError(f"oracle_saturation_T rc={rc}")
    return t_tok.value, t_fl.value


def calibrated_T(gamma: float, t_e: float, t_c: float, c_dummy: float) -> float:
    """App. B.4 Eq. 3: T = gamma * (t_e/t_c) * C_dummy."""
    return _load().oracle_calibrated_T(gamma, t_e, t_c, c_dummy)


# ------------------------------------------------------------------ NEXT-3: DP attention layer
# (oracle/attn_oracle.c; reading R19)

def rmsnorm(x, w=None, eps: float = 1e-6) -> np.ndarray:
    """Row-wise RMSNorm x / sqrt(mean(x^2) + eps) * w, fp64."""
    x = _f32(x)
    n = x.shape[-1]
    out = np.empty(x.shape, np.float64)
    rc = _load().oracle_rmsnorm(_ptr(x), _ptr(None if w is None else _f32(w)), x.size // n, n, float(eps),
                                _ptr(out))
    if rc:
        raise ValueError(f"oracle_rmsnorm rc={rc}")
    return out


def rope(x, pos, theta: float = 1e6) -> np.ndarray:
    """Rotate-half rotary embedding of x [T, nh, d] at positions pos [T], fp64."""
    out = np.array(x, dtype=np.float64, copy=True, order="C")
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    T, nh, d = out.shape
    rc = _load().oracle_rope(_ptr(out), _ptr(pos), T, nh, d, float(theta))
    if rc:
        raise ValueError(f"oracle_rope rc={rc}")
    return out


def attention(q, k, v, cu_seqlens, causal: bool = True, scale=None, rows=None) -> np.ndarray:
    """GQA softmax attention over packed prompts; q [n, Hq, d] (one row per entry of rows,
    or [T, Hq, d] when rows is None), k / v [T, Hkv, d]; returns [n, Hq, d] fp64."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    cu = np.ascontiguousarray(cu_seqlens, dtype=np.int32)
    Hq, d = q.shape[1], q.shape[2]
    Hkv = k.shape[1]
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    n = q.shape[0]
    out = np.empty((n, Hq, d), np.float64)
    sc = float(1.0 / np.sqrt(d)) if scale is None else float(scale)
    rc = _load().oracle_attention(_ptr(q), _ptr(k), _ptr(v), _ptr(cu), len(cu) - 1, Hq, Hkv, d, int(causal), sc,
                                  _ptr(r), 0 if r is None else len(r), _ptr(out))
    if rc:
        raise ValueError(f"oracle_attention rc={rc}")
    return out


def attn_layer(x, cu_seqlens, Hq: int, Hkv: int, d: int, w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2,
               eps: float = 1e-6, theta: float = 1e6, rows=None):
    """One DP attention layer (R19) for the tokens in rows (None = all):
    returns (x' = x + attn, RMSNorm(x'; w_ln2)) as fp32 arrays [n, H]."""
    x = _f32(x)
    T, H = x.shape
    cu = np.ascontiguousarray(cu_seqlens, dtype=np.int32)
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    n = T if r is None else len(r)
    xo = np.empty((n, H), np.float32)
    xn2 = np.empty((n, H), np.float32)
    ws = [_f32(a) for a in (w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2)]
    rc = _load().oracle_attn_layer(_ptr(x), T, H, _ptr(cu), len(cu) - 1, Hq, Hkv, d, *[_ptr(a) for a in ws],
                                   float(eps), float(theta), _ptr(r), 0 if r is None else len(r), _ptr(xo), _ptr(xn2))
    if rc:
        raise ValueError(f"oracle_attn_layer rc={rc}")
    return xo, xn2
