"""Thin Python binding of the C ABI in ``include/asyncep.h`` (libasyncep.so).

Argument marshalling only: every step of the hot path runs in the library's CUDA
kernels.  The functions carry the C names.  There is no CPU fallback: if the
extension is missing the import of this module fails loudly.

PyTorch supplies device memory (tensors), streams (``torch.cuda.Stream``) and the NCCL
communicator (``ProcessGroupNCCL._comm_ptr()``); the library borrows all of them.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# ASYNCEP_LIB: an in-tree variant build (build.py -D ... --out ...) for same-box A/B runs
LIB_PATH = os.environ.get("ASYNCEP_LIB") or os.path.join(_HERE, "libasyncep.so")

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_CUDA, ERR_NCCL, ERR_NOT_PREFETCHED, ERR_WORKSPACE = range(7)
BF16, FP8_E4M3 = 0, 1
FLAG_IDENTITY_EXPERTS = 0x1
FLAG_SIMT_GEMM = 0x2
FLAG_STAGE_TIMING = 0x4
FLAG_SIMT_ROUTER = 0x8
FLAG_XPERM = 0x10
FLAG_OFFLOAD = 0x20
FLAG_NO_SWAP_TAILS = 0x40
FLAG_SWAP_TAILS = 0x80
FLAG_MX_ACT = 0x100
FLAG_FUSED_DISPATCH = 0x200
STAGES = ("router", "permute", "gather_wait", "gemm1_gateup_swiglu", "gemm2_down", "combine")


class AsyncEPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"asyncep status {status}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_experts", ctypes.c_int32),
                ("top_k", ctypes.c_int32), ("hidden", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("expert_dtype", ctypes.c_int32), ("world_size", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("replicate_layer0", ctypes.c_int32),
                ("norm_topk", ctypes.c_int32), ("max_tokens", ctypes.c_int64),
                ("gamma", ctypes.c_float), ("flags", ctypes.c_int32)]


def make_config(num_layers, num_experts, top_k, hidden, ffn, *, expert_dtype=BF16, world_size=1,
                rank=0, replicate_layer0=1, norm_topk=1, max_tokens=1, gamma=1.2, flags=0) -> Config:
    return Config(num_layers, num_experts, top_k, hidden, ffn, expert_dtype, world_size, rank,
                  replicate_layer0, norm_topk, max_tokens, gamma, flags)


class AttnConfig(ctypes.Structure):
    """asyncep_attn_config (NEXT-3 attention layer, reading R19)."""
    _fields_ = [("hidden", ctypes.c_int32), ("q_heads", ctypes.c_int32), ("kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("max_tokens", ctypes.c_int64), ("max_prompts", ctypes.c_int64),
                ("eps", ctypes.c_double), ("rope_theta", ctypes.c_double)]


def make_attn_config(hidden, q_heads, kv_heads, head_dim=128, *, max_tokens=1, max_prompts=0, eps=1e-6,
                     rope_theta=1e6) -> AttnConfig:
    return AttnConfig(hidden, q_heads, kv_heads, head_dim, max_tokens, max_prompts, eps, rope_theta)


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, D, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
        CP = ctypes.POINTER(Config)
        sig = {
            "asyncep_abi_version": ([], I32),
            "asyncep_last_error": ([], ctypes.c_char_p),
            "asyncep_expert_bytes": ([CP], SZ),
            "asyncep_slot_bytes": ([CP], SZ),
            "asyncep_shard_bytes": ([CP], SZ),
            "asyncep_workspace_size": ([CP], SZ),
            "asyncep_pack_experts": ([CP, I32, P, P, P, P, P, P, P, P], I32),
            "asyncep_init": ([CP, P, P, P, P, P, P, P, P, ctypes.POINTER(P)], I32),
            "asyncep_prefetch_layer": ([P, I32], I32),
            "asyncep_prefetch_layer_local": ([P, I32, P], I32),
            "asyncep_set_gather_transport": ([P, I32, I32], I32),
            "asyncep_set_gather_copy_ctas": ([P, I32], I32),
            "asyncep_set_gather_comm": ([P, P], I32),
            "asyncep_timeline_begin": ([P], I32),
            "asyncep_timeline_read": ([P, P, I32, ctypes.POINTER(I32)], I32),
            "asyncep_probe_gather": ([P, I32, P, ctypes.POINTER(D), ctypes.POINTER(D)], I32),
            "asyncep_moe_forward": ([P, I32, P, I64, P, P, P, P, P], I32),
            "asyncep_saturation_T": ([CP, D, D, ctypes.POINTER(D), ctypes.POINTER(D)], I32),
            "asyncep_stage_times": ([P, ctypes.POINTER(D), I32, ctypes.POINTER(I64)], I32),
            "asyncep_reset_stage_times": ([P], I32),
            "asyncep_kernel_launches": ([P], I64),
            "asyncep_forward_times": ([P, ctypes.POINTER(D), ctypes.POINTER(I32), I32, ctypes.POINTER(I32)], I32),
            "asyncep_calibrated_T": ([D, D, D, D, ctypes.POINTER(D)], I32),
            "asyncep_calibrate_T": ([P, D, I64, ctypes.POINTER(D), ctypes.POINTER(D), ctypes.POINTER(D),
                                     ctypes.POINTER(D)], I32),
            "asyncep_set_link_emulation": ([P, D], I32),
            "asyncep_set_gather_gate": ([P, I32], I32),
            "asyncep_set_peer_shards": ([P, P], I32),
            "asyncep_gather_copy": ([P, P, SZ, P], I32),
            "asyncep_enable_offload": ([P, P, P, I32, P], I32),
            "asyncep_stage_layer": ([P, I32], I32),
            "asyncep_cost_delta": ([P, I64, I64, I64], D),
            "asyncep_router_create": ([P, ctypes.POINTER(P)], I32),
            "asyncep_router_destroy": ([P], I32),
            "asyncep_router_set_T": ([P, D], I32),
            "asyncep_router_loads": ([P, P], I32),
            "asyncep_router_schedule_round": ([P, I32, I64, P, P, P, P, P, P, ctypes.POINTER(I64)], I32),
            "asyncep_router_blocks_stored": ([P, I32, P, I64], I32),
            "asyncep_router_progress": ([P, I32, I64], I32),
            "asyncep_ep_plan": ([CP, P, P, P, P, P, P, P, ctypes.POINTER(I64)], I32),
            "asyncep_ep_workspace_size": ([CP, I64], SZ),
            "asyncep_ep_forward": ([P, I32, P, I64, P, P, P, I64], I32),
            "asyncep_attn_workspace_size": ([ctypes.POINTER(AttnConfig)], SZ),
            "asyncep_attention": ([ctypes.POINTER(AttnConfig), P, P, P, I64, P, P, I32, I64, P, P, P], I32),
            "asyncep_attn_layer": ([ctypes.POINTER(AttnConfig), P, I64, P, I32, P, P, P, P, P, P, P, P, P, SZ, P],
                                   I32),
            "asyncep_destroy": ([P], I32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != OK:
        raise AsyncEPError(status, lib().asyncep_last_error().decode(errors="replace"))


def _p(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(s) -> int | None:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ------------------------------------------------------------------------------ sizes
def asyncep_expert_bytes(cfg: Config) -> int:
    return lib().asyncep_expert_bytes(ctypes.byref(cfg))


def asyncep_slot_bytes(cfg: Config) -> int:
    return lib().asyncep_slot_bytes(ctypes.byref(cfg))


def asyncep_shard_bytes(cfg: Config) -> int:
    return lib().asyncep_shard_bytes(ctypes.byref(cfg))


def asyncep_workspace_size(cfg: Config) -> int:
    n = lib().asyncep_workspace_size(ctypes.byref(cfg))
    if n == 0:
        _check(ERR_INVALID_ARG)
    return n


def asyncep_pack_experts(cfg: Config, gate, up, down, out, stream=None, gate_scale=None,
                         up_scale=None, down_scale=None) -> None:
    _check(lib().asyncep_pack_experts(ctypes.byref(cfg), gate.shape[0], _p(gate), _p(up), _p(down),
                                      _p(gate_scale), _p(up_scale), _p(down_scale), _p(out),
                                      _stream(stream)))


# ------------------------------------------------------------------------------ context
@dataclass
class Context:
    handle: ctypes.c_void_p
    cfg: Config
    keep: list = field(default_factory=list)  # tensors that must outlive the context

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.asyncep_destroy(self.handle)
            self.handle = None


def asyncep_init(cfg: Config, nccl_comm, compute_stream, comm_stream, router_w, expert_shard,
                 slot0, slot1, workspace) -> Context:
    L = cfg.num_layers
    assert len(router_w) == L and len(expert_shard) == L
    rw = (ctypes.c_void_p * L)(*[_p(t) for t in router_w])
    sh = (ctypes.c_void_p * L)(*[_p(t) for t in expert_shard])
    h = ctypes.c_void_p()
    _check(lib().asyncep_init(ctypes.byref(cfg), nccl_comm, _stream(compute_stream), _stream(comm_stream),
                              rw, sh, _p(slot0), _p(slot1), _p(workspace), ctypes.byref(h)))
    return Context(h, cfg, [list(router_w), list(expert_shard), slot0, slot1, workspace,
                            compute_stream, comm_stream])


def asyncep_prefetch_layer(ctx: Context, layer: int) -> None:
    _check(lib().asyncep_prefetch_layer(ctx.handle, layer))


def asyncep_prefetch_layer_local(ctx: Context, layer: int, shards) -> None:
    arr = (ctypes.c_void_p * len(shards))(*[_p(t) for t in shards])
    _check(lib().asyncep_prefetch_layer_local(ctx.handle, layer, arr))


def asyncep_ep_plan(cfg: Config, send_counts, recv_counts):
    """Host-side row plan of the DP x EP exchange (see asyncep.h).  Counts: int32 numpy [E]."""
    import numpy as np
    N, E = cfg.world_size, cfg.num_experts
    sc = np.ascontiguousarray(send_counts, dtype=np.int32)
    rc = np.ascontiguousarray(recv_counts, dtype=np.int32)
    out = {k: np.zeros(n, np.int64) for k, n in (("send_off", N), ("send_rows", N), ("recv_off", N),
                                                    ("recv_rows", N), ("group_off", E + 1))}
    tot = ctypes.c_int64()
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(lib().asyncep_ep_plan(ctypes.byref(cfg), vp(sc), vp(rc), vp(out["send_off"]), vp(out["send_rows"]),
                                 vp(out["recv_off"]), vp(out["recv_rows"]), vp(out["group_off"]),
                                 ctypes.byref(tot)))
    out["recv_total"] = tot.value
    return out


def asyncep_ep_workspace_size(cfg: Config, max_recv_rows: int) -> int:
    n = lib().asyncep_ep_workspace_size(ctypes.byref(cfg), max_recv_rows)
    if n == 0:
        _check(ERR_INVALID_ARG)
    return n


def asyncep_ep_forward(ctx: Context, layer: int, x, ep_workspace, max_recv_rows: int, residual=None, y=None):
    if y is None:
        y = torch.empty_like(x)
    _check(lib().asyncep_ep_forward(ctx.handle, layer, _p(x), x.shape[0], _p(residual), _p(y), _p(ep_workspace),
                                    max_recv_rows))
    return y


def asyncep_enable_offload(ctx: Context, host_shards, window, w: int, h2d_stream) -> None:
    L = ctx.cfg.num_layers
    hs = (ctypes.c_void_p * L)(*[_p(t) for t in host_shards])
    wb = (ctypes.c_void_p * w)(*[_p(t) for t in window])
    _check(lib().asyncep_enable_offload(ctx.handle, hs, wb, w, _stream(h2d_stream)))
    ctx.keep += [list(host_shards), list(window), h2d_stream]


def asyncep_stage_layer(ctx: Context, layer: int) -> None:
    _check(lib().asyncep_stage_layer(ctx.handle, layer))


def asyncep_set_peer_shards(ctx: Context, shards) -> None:
    """shards: [layer][rank] tensors (peer ones CUDA-IPC-mapped) or None to revert to NCCL."""
    if shards is None:
        _check(lib().asyncep_set_peer_shards(ctx.handle, None))
        return
    L, N = ctx.cfg.num_layers, ctx.cfg.world_size
    flat = [(_p(shards[l][r]) if shards[l] is not None and shards[l][r] is not None else None)
            for l in range(L) for r in range(N)]
    arr = (ctypes.c_void_p * (L * N))(*flat)
    _check(lib().asyncep_set_peer_shards(ctx.handle, arr))
    ctx.keep.append(shards)


GATHER_COPY_KERNEL, GATHER_COPY_ENGINE, GATHER_NCCL = 0, 1, 2
GATHER_NAMES = {GATHER_COPY_KERNEL: "copy_kernel", GATHER_COPY_ENGINE: "copy_engine", GATHER_NCCL: "nccl"}


def asyncep_set_gather_transport(ctx: Context, transport: int, reserve_sms: int = 0) -> None:
    _check(lib().asyncep_set_gather_transport(ctx.handle, int(transport), int(reserve_sms)))


def asyncep_set_gather_comm(ctx: Context, nccl_comm) -> None:
    """ncclComm_t (int) for the NCCL gather, or None for the context's communicator."""
    _check(lib().asyncep_set_gather_comm(ctx.handle, nccl_comm))


def nccl_gather_group(max_ctas: int):
    """A dedicated NCCL process group over all ranks for the weight gather, its kernels capped at
    max_ctas CTAs (the SMs the grouped GEMMs leave free); eagerly initialised.  -> (group, comm)."""
    import torch.distributed as dist
    opts = dist.ProcessGroupNCCL.Options()
    opts.config.max_ctas = int(max_ctas)
    opts.config.min_ctas = 1
    g = dist.new_group(ranks=list(range(dist.get_world_size())), backend="nccl", pg_options=opts)
    dist.all_reduce(torch.ones(1, device="cuda"), group=g)
    return g, nccl_comm_ptr(g)


def asyncep_set_gather_copy_ctas(ctx: Context, ctas: int) -> None:
    _check(lib().asyncep_set_gather_copy_ctas(ctx.handle, int(ctas)))


def asyncep_probe_gather(ctx: Context, layer: int, shards=None):
    """One timed gather of `layer` (startup probe, R12) -> (ms, bytes received per rank)."""
    arr = None
    if shards is not None:
        arr = (ctypes.c_void_p * len(shards))(*[_p(t) for t in shards])
    ms, nb = ctypes.c_double(), ctypes.c_double()
    _check(lib().asyncep_probe_gather(ctx.handle, int(layer), arr, ctypes.byref(ms), ctypes.byref(nb)))
    return ms.value, nb.value


def asyncep_gather_copy(dst, src, nbytes: int, stream=None) -> None:
    _check(lib().asyncep_gather_copy(_p(dst), _p(src), nbytes, _stream(stream or torch.cuda.current_stream())))


def asyncep_set_link_emulation(ctx: Context, bytes_per_s: float) -> None:
    _check(lib().asyncep_set_link_emulation(ctx.handle, float(bytes_per_s)))


def asyncep_set_gather_gate(ctx: Context, on: bool) -> None:
    """Copy-kernel gathers move bytes only while a forward's grouped GEMMs run (asyncep.h)."""
    _check(lib().asyncep_set_gather_gate(ctx.handle, int(bool(on))))


def asyncep_moe_forward(ctx: Context, layer: int, x: torch.Tensor, residual=None, y=None,
                        topk_ids_out=None, topk_w_out=None, expert_counts_out=None) -> torch.Tensor:
    T = x.shape[0]
    if y is None:
        y = torch.empty_like(x)
    _check(lib().asyncep_moe_forward(ctx.handle, layer, _p(x), T, _p(residual), _p(y),
                                     _p(topk_ids_out), _p(topk_w_out), _p(expert_counts_out)))
    return y


def asyncep_saturation_T(cfg: Config, flops_per_s: float, ag_bytes_per_s: float):
    t = ctypes.c_double()
    f = ctypes.c_double()
    _check(lib().asyncep_saturation_T(ctypes.byref(cfg), flops_per_s, ag_bytes_per_s, ctypes.byref(t),
                                      ctypes.byref(f)))
    return t.value, f.value


def asyncep_stage_times(ctx: Context):
    ms = (ctypes.c_double * len(STAGES))()
    n = ctypes.c_int64()
    _check(lib().asyncep_stage_times(ctx.handle, ms, len(STAGES), ctypes.byref(n)))
    return dict(zip(STAGES, list(ms))), n.value


def asyncep_forward_times(ctx: Context, n: int = 4096):
    """[(layer, ms)] of the last recorded forwards (ASYNCEP_FLAG_STAGE_TIMING), oldest first."""
    ms = (ctypes.c_double * n)()
    ly = (ctypes.c_int32 * n)()
    m = ctypes.c_int32()
    _check(lib().asyncep_forward_times(ctx.handle, ms, ly, n, ctypes.byref(m)))
    return [(ly[i], ms[i]) for i in range(m.value)]


def asyncep_calibrated_T(gamma: float, t_e: float, t_c: float, c_dummy: float) -> float:
    """App. B.4 Eq. 3: T = gamma * (t_e / t_c) * C_dummy [FLOPs]."""
    out = ctypes.c_double()
    _check(lib().asyncep_calibrated_T(gamma, t_e, t_c, c_dummy, ctypes.byref(out)))
    return out.value


def asyncep_calibrate_T(ctx: Context, gamma: float, n_ref: int):
    """NEXT-1 (App. B.4) from the last profile pass: -> dict(T_flops, T_tokens, t_c_ms, t_e_ms)."""
    out = [ctypes.c_double() for _ in range(4)]
    _check(lib().asyncep_calibrate_T(ctx.handle, float(gamma), int(n_ref), *[ctypes.byref(o) for o in out]))
    return dict(zip(("T_flops", "T_tokens", "t_c_ms", "t_e_ms"), (o.value for o in out)))


class TimelineRec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("layer", ctypes.c_int32), ("t0", ctypes.c_float),
                ("t1", ctypes.c_float), ("t2", ctypes.c_float), ("t3", ctypes.c_float)]


def asyncep_timeline_begin(ctx: Context) -> None:
    _check(lib().asyncep_timeline_begin(ctx.handle))


def asyncep_timeline_read(ctx: Context, n: int = 4096):
    """-> [(kind 'forward'|'gather', layer, t0, t1, t2, t3)] in ms since asyncep_timeline_begin:
    forward = (start, dispatch done, GEMM1 start, end), gather = (start, end, end, end)."""
    buf = (TimelineRec * n)()
    m = ctypes.c_int32()
    _check(lib().asyncep_timeline_read(ctx.handle, buf, n, ctypes.byref(m)))
    return [("forward" if r.kind == 0 else "gather", r.layer, r.t0, r.t1, r.t2, r.t3)
            for r in buf[:min(n, m.value)]]


def asyncep_reset_stage_times(ctx: Context) -> None:
    _check(lib().asyncep_reset_stage_times(ctx.handle))


def asyncep_kernel_launches(ctx: Context) -> int:
    return lib().asyncep_kernel_launches(ctx.handle)


def asyncep_destroy(ctx: Context) -> None:
    if ctx.handle:
        _check(lib().asyncep_destroy(ctx.handle))
        ctx.handle = None


def asyncep_abi_version() -> int:
    return lib().asyncep_abi_version()


def nccl_comm_ptr(pg=None) -> int:
    """The ncclComm_t of torch's NCCL process group (must be eagerly initialised)."""
    import torch.distributed as dist
    pg = pg or dist.group.WORLD
    return pg._get_backend(torch.device("cuda"))._comm_ptr()


# ------------------------------------------------------------------------------ NEXT-3 attention
def asyncep_attn_workspace_size(cfg: AttnConfig) -> int:
    n = lib().asyncep_attn_workspace_size(ctypes.byref(cfg))
    if n == 0:
        _check(ERR_INVALID_ARG)
    return n


def asyncep_attention(cfg: AttnConfig, q, k, vt, ldv: int, vt_cu, cu_seqlens, o, stream=None, sched=None) -> None:
    """Causal GQA attention core: q [T,Hq,d], k [T,Hkv,d], vt [Hkv,d,ldv] with prompt b at columns
    vt_cu[b] (multiples of 8), cu_seqlens int32 [B+1]; sched: int32 device counter (one per call)."""
    T = q.shape[0]
    st = stream or torch.cuda.current_stream()
    if sched is None:  # allocated in the launching stream's pool: a concurrent call never gets the same int
        with torch.cuda.stream(st):
            sched = torch.empty(1, dtype=torch.int32, device=q.device)
    _check(lib().asyncep_attention(ctypes.byref(cfg), _p(q), _p(k), _p(vt), ldv, _p(vt_cu), _p(cu_seqlens),
                                   cu_seqlens.shape[0] - 1, T, _p(o), _p(sched), _stream(st)))


def asyncep_attn_layer(cfg: AttnConfig, x, cu_seqlens, weights, x_out, xn2_out, workspace, stream=None) -> None:
    """One DP attention layer; weights = (w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2)."""
    _check(lib().asyncep_attn_layer(ctypes.byref(cfg), _p(x), x.shape[0], _p(cu_seqlens), cu_seqlens.shape[0] - 1,
                                    *[_p(w) for w in weights], _p(x_out), _p(xn2_out), _p(workspace),
                                    workspace.numel() * workspace.element_size(),
                                    _stream(stream or torch.cuda.current_stream())))


# ------------------------------------------------------------------------------ NEXT-4 admission
class RouterConfig(ctypes.Structure):
    _fields_ = [("num_gpus", ctypes.c_int32), ("block_size", ctypes.c_int32), ("f_tok", ctypes.c_double),
                ("attn_hl", ctypes.c_double), ("T_flops", ctypes.c_double)]


def asyncep_cost_delta(rcfg: RouterConfig, P: int, M: int, S: int) -> float:
    return lib().asyncep_cost_delta(ctypes.byref(rcfg), P, M, S)


class Router:
    """Saturation-bounded admission (Algorithm 1) -- thin wrapper."""

    def __init__(self, num_gpus, block_size, f_tok, attn_hl, T_flops):
        self.cfg = RouterConfig(num_gpus, block_size, f_tok, attn_hl, T_flops)
        self.h = ctypes.c_void_p()
        _check(lib().asyncep_router_create(ctypes.byref(self.cfg), ctypes.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.asyncep_router_destroy(self.h)
            self.h = None

    def schedule_round(self, chains, prefix_len, suffix_len, reset_loads=True):
        import numpy as np
        n = len(chains)
        off = np.zeros(n + 1, np.int64)
        off[1:] = np.cumsum([len(c) for c in chains])
        hashes = np.ascontiguousarray(np.concatenate([np.asarray(c, np.uint64) for c in chains])
                                      if n else np.zeros(0, np.uint64), dtype=np.uint64)
        pl = np.ascontiguousarray(prefix_len, np.int64)
        sl = np.ascontiguousarray(suffix_len, np.int64)
        gpu = np.empty(n, np.int32)
        delta = np.empty(n, np.float64)
        adm = ctypes.c_int64()
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        _check(lib().asyncep_router_schedule_round(self.h, int(reset_loads), n, vp(off), vp(hashes), vp(pl), vp(sl),
                                                   vp(gpu), vp(delta), ctypes.byref(adm)))
        return gpu, delta

    def loads(self):
        import numpy as np
        out = np.empty(self.cfg.num_gpus, np.float64)
        _check(lib().asyncep_router_loads(self.h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def blocks_stored(self, gpu, hashes):
        import numpy as np
        a = np.ascontiguousarray(hashes, np.uint64)
        _check(lib().asyncep_router_blocks_stored(self.h, gpu, a.ctypes.data_as(ctypes.c_void_p), a.size))

    def progress(self, gpu, tokens):
        _check(lib().asyncep_router_progress(self.h, gpu, tokens))

    def set_T(self, T_flops):
        _check(lib().asyncep_router_set_T(self.h, T_flops))
