"""Host-side driver for an L-layer AsyncEP MoE stack on one GPU (one rank).

Allocates (with torch) the replicated router weights, this rank's packed expert shards
(layer 0 fully replicated), the two gather slots and the workspace, creates
the library context, and runs the per-layer schedule of the "MoE gatherer"
(PAPER.md:630): issue the AllGather of layer l+1, then compute layer l.

Weights are supplied by callables so this module holds no generator:
  router_fn(l)             -> [E, H] bf16 tensor
  expert_fn(l, experts)    -> (gate [n,h,H], up [n,h,H], down [n,H,h]) bf16 tensors, or for
                              FP8 experts (codes uint8 x3, gate_scale [n,h], up_scale [n,h],
                              down_scale [n,H] fp32)
"""
from __future__ import annotations

import torch

from . import asyncep as A
from .schedule import layer_resident, shard_range, stack_schedule, staged_layers


class MoEStack:
    def __init__(self, L, E, k, H, h, max_tokens, router_fn, expert_fn, *, world_size=1, rank=0,
                 replicate_layer0=True, norm_topk=True, flags=0, gamma=1.2, device="cuda",
                 nccl_comm=None, compute_stream=None, comm_stream=None, pack_chunk=8, fp8=False,
                 offload_window=0):
        self.device = torch.device(device)
        flags |= A.FLAG_OFFLOAD if offload_window else 0
        self.offload_w = offload_window
        self.cfg = A.make_config(L, E, k, H, h, world_size=world_size, rank=rank,
                                 replicate_layer0=int(replicate_layer0), norm_topk=int(norm_topk),
                                 max_tokens=max_tokens, gamma=gamma, flags=flags,
                                 expert_dtype=A.FP8_E4M3 if fp8 else A.BF16)
        self.L, self.E, self.k, self.H, self.h = L, E, k, H, h
        self.N, self.rank = world_size, rank
        self.compute_stream = compute_stream or torch.cuda.current_stream(self.device)
        self.comm_stream = comm_stream if comm_stream is not None else (
            torch.cuda.Stream(self.device) if world_size > 1 else None)
        ebytes = A.asyncep_expert_bytes(self.cfg)
        self.expert_bytes = ebytes
        self.router_w = [router_fn(l).to(self.device, torch.bfloat16).contiguous() for l in range(L)]
        self.fp8, self.expert_fn, self.pack_chunk = fp8, expert_fn, pack_chunk
        self.shards = []
        self.host_shards = [None] * L
        staged = set(staged_layers(L, world_size, replicate_layer0)) if offload_window else set()
        for l in range(L):
            full = layer_resident(l, world_size, replicate_layer0)
            buf = self.pack(l, range(E) if full else shard_range(E, world_size, rank))
            if l in staged:  # NEXT-2: the backing store is pinned host memory
                self.host_shards[l] = buf.cpu().pin_memory()
                del buf
                buf = None
            self.shards.append(buf)
        if world_size > 1:
            sb = A.asyncep_slot_bytes(self.cfg)
            self.slots = [torch.empty(sb, dtype=torch.uint8, device=self.device) for _ in range(2)]
        else:
            self.slots = [None, None]
        self.workspace = torch.empty(A.asyncep_workspace_size(self.cfg), dtype=torch.uint8, device=self.device)
        torch.cuda.synchronize(self.device)
        self.ctx = A.asyncep_init(self.cfg, nccl_comm, self.compute_stream, self.comm_stream, self.router_w,
                                  self.shards, self.slots[0], self.slots[1], self.workspace)
        self._bufs = None
        self.attn_w = None
        if offload_window:
            nb = A.asyncep_slot_bytes(self.cfg) if world_size == 1 else A.asyncep_shard_bytes(self.cfg)
            self.window = [torch.empty(nb, dtype=torch.uint8, device=self.device) for _ in range(offload_window)]
            self.h2d_stream = torch.cuda.Stream(self.device)
            A.asyncep_enable_offload(self.ctx, self.host_shards, self.window, offload_window, self.h2d_stream)

    def enable_attention(self, attn_fn, q_heads: int, kv_heads: int, head_dim: int = 128, max_prompts: int = 0,
                         eps: float = 1e-6, rope_theta: float = 1e6) -> None:
        """NEXT-3: run each layer as a decoder layer, DP attention (KV-cache-free) then MoE:
        x' = x + Attn_l(x);  x_{l+1} = x' + MoE_l(RMSNorm(x'))  (reading R19).
        attn_fn(l) -> (w_ln1, w_qkv, w_qn, w_kn, w_o, w_ln2) bf16 tensors (replicated on
        every rank).  The gather of layer l+1 then overlaps attention and MoE."""
        self.attn_cfg = A.make_attn_config(self.H, q_heads, kv_heads, head_dim, max_tokens=self.cfg.max_tokens,
                                           max_prompts=max_prompts, eps=eps, rope_theta=rope_theta)
        self.attn_w = [tuple(t.to(self.device, torch.bfloat16).contiguous() for t in attn_fn(l))
                       for l in range(self.L)]
        self.attn_ws = torch.empty(A.asyncep_attn_workspace_size(self.attn_cfg), dtype=torch.uint8,
                                   device=self.device)
        self._abufs = [torch.empty((self.cfg.max_tokens, self.H), dtype=torch.bfloat16, device=self.device)
                       for _ in range(2)]

    def attention(self, l, x, cu_seqlens):
        """Attention half of decoder layer l: returns (x', RMSNorm(x'; w_ln2)) views."""
        T = x.shape[0]
        xa, xn = self._abufs[0][:T], self._abufs[1][:T]
        A.asyncep_attn_layer(self.attn_cfg, x, cu_seqlens, self.attn_w[l], xa, xn, self.attn_ws,
                             stream=self.compute_stream)
        return xa, xn

    def pack(self, l: int, experts: range) -> torch.Tensor:
        """Packed blobs of ``experts`` of layer l (the shard format of asyncep.h)."""
        ebytes = self.expert_bytes
        buf = torch.empty(len(experts) * ebytes, dtype=torch.uint8, device=self.device)
        st = torch.cuda.current_stream(self.device)
        for c0 in range(0, len(experts), self.pack_chunk):
            sub = experts[c0:c0 + self.pack_chunk]
            dst = buf[c0 * ebytes:(c0 + len(sub)) * ebytes]
            if self.fp8:
                g, u, d, gs, us, ds = (t.to(self.device).contiguous() for t in self.expert_fn(l, sub))
                A.asyncep_pack_experts(self.cfg, g, u, d, dst, stream=st, gate_scale=gs, up_scale=us,
                                       down_scale=ds)
                del gs, us, ds
            else:
                g, u, d = (t.to(self.device, torch.bfloat16).contiguous() for t in self.expert_fn(l, sub))
                A.asyncep_pack_experts(self.cfg, g, u, d, dst, stream=st)
            del g, u, d
        return buf

    def peer_shards(self):
        """Single-GPU emulation of the other ranks (tests / --emulate-gather): the shards of
        ranks != self.rank for every gathered layer, so asyncep_prefetch_layer_local can
        assemble the slot with device-to-device copies.  Returns local_shards(l)."""
        table = {}
        for l in range(self.L):
            if self.layer_resident(l):
                continue
            own = self.shards[l] if self.shards[l] is not None else self.window[0]  # offload: C reads the window
            table[l] = [own if r == self.rank else self.pack(l, shard_range(self.E, self.N, r))
                        for r in range(self.N)]
        return lambda l: table[l]

    def enable_p2p_gather(self, pg=None) -> None:
        """Copy-engine gather across real ranks (asyncep_set_peer_shards): every rank shares its
        shard buffers through CUDA IPC (torch's tensor IPC, exchanged with all_gather_object) and
        maps the peers'; asyncep_prefetch_layer then copies them over NVLink with copy engines,
        leaving every SM to the persistent GEMMs.  Collective over the process group."""
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        mine = [None if self.layer_resident(l) else reduce_tensor(self.shards[l]) for l in range(self.L)]
        allh = [None] * self.N
        dist.all_gather_object(allh, mine, group=pg)
        table = [None] * self.L
        for l in range(self.L):
            if self.layer_resident(l):
                continue
            row = []
            for r in range(self.N):
                if r == self.rank:
                    row.append(self.shards[l])
                else:
                    fn, args = allh[r][l]
                    row.append(fn(*args))  # peer memory mapped into this process
            table[l] = row
        self._peer_table = table
        A.asyncep_set_peer_shards(self.ctx, table)
        dist.barrier(group=pg)

    def set_peer_table(self, table) -> None:
        """Install a [layer][rank] shard table for the copy-engine gather (1-GPU emulation in
        tests: local tensors stand in for the IPC-mapped peers)."""
        self._peer_table = table
        A.asyncep_set_peer_shards(self.ctx, table)

    def layer_resident(self, l: int) -> bool:
        return layer_resident(l, self.N, bool(self.cfg.replicate_layer0))

    def prefetch(self, l: int, local_shards=None) -> None:
        if local_shards is not None:
            if not self.layer_resident(l):
                A.asyncep_prefetch_layer_local(self.ctx, l, local_shards(l))
        else:
            A.asyncep_prefetch_layer(self.ctx, l)

    def forward(self, l, x, residual=None, y=None, ids=None, w=None, counts=None):
        return A.asyncep_moe_forward(self.ctx, l, x, residual=residual, y=y, topk_ids_out=ids,
                                     topk_w_out=w, expert_counts_out=counts)

    def run(self, x, residual=True, out=None, local_shards=None, record=None, cu_seqlens=None):
        """One pass of the whole stack: x_{l+1} = x_l + MoE_l(x_l) (reading R9), or with
        attention enabled the decoder layer x' = x + Attn_l(x), x_{l+1} = x' + MoE_l(RMSNorm(x'))
        over the packed prompts cu_seqlens (int32 device [B+1]).
        Returns the final activations (a ping-pong buffer unless ``out`` is given; it may be
        passed back in as ``x``, but the next call reuses it).
        ``record(l, x_l)`` (optional) sees each layer's input before it runs."""
        T = x.shape[0]
        if self._bufs is None or self._bufs[0].shape[0] < T:
            self._bufs = [torch.empty((self.cfg.max_tokens, self.H), dtype=torch.bfloat16, device=self.device)
                          for _ in range(2)]
        # ping-pong parity chosen so that no layer's destination is its own input, even when x is
        # a buffer this stack returned earlier
        par = 1 if self._bufs[0].data_ptr() == x.data_ptr() else 0
        cur = x
        for op, l, _slot in stack_schedule(self.L, self.N, bool(self.cfg.replicate_layer0), self.offload_w):
            if op == "stage":
                A.asyncep_stage_layer(self.ctx, l)  # PCIe channel, up to w layers ahead
                continue
            if op == "prefetch":
                self.prefetch(l, local_shards)  # gather of layer l overlaps layer l-1
                continue
            if record is not None:
                record(l, cur)
            dst = out if (out is not None and l == self.L - 1) else self._bufs[(l + par) % 2][:T]
            if self.attn_w is not None:
                xa, xn = self.attention(l, cur, cu_seqlens)
                self.forward(l, xn, residual=xa, y=dst)
            else:
                self.forward(l, cur, residual=cur if residual else None, y=dst)
            cur = dst
        return cur

    def run_ep(self, x, residual=True, out=None, recv_factor: float = 2.0):
        """Contrast baseline: the same stack as synchronous DP x EP: each
        layer dispatches its permuted rows to the owners of their experts and returns the
        outputs with two on-path AllToAlls (asyncep_ep_forward).  recv_factor sizes the
        receive buffer in units of this rank's own rows (dropless within it)."""
        T = x.shape[0]
        cap = int(recv_factor * self.cfg.max_tokens * self.k) + self.E * 256
        if getattr(self, "_ep_ws", None) is None or self._ep_cap < cap:
            self._ep_ws = torch.empty(A.asyncep_ep_workspace_size(self.cfg, cap), dtype=torch.uint8,
                                      device=self.device)
            self._ep_cap = cap
        if self._bufs is None or self._bufs[0].shape[0] < T:
            self._bufs = [torch.empty((self.cfg.max_tokens, self.H), dtype=torch.bfloat16, device=self.device)
                          for _ in range(2)]
        par = 1 if self._bufs[0].data_ptr() == x.data_ptr() else 0
        cur = x
        for l in range(self.L):
            dst = out if (out is not None and l == self.L - 1) else self._bufs[(l + par) % 2][:T]
            A.asyncep_ep_forward(self.ctx, l, cur, self._ep_ws, self._ep_cap, residual=cur if residual else None,
                                 y=dst)
            cur = dst
        return cur

    def calibrate_T(self, x, gamma: float | None = None, local_shards=None):
        """NEXT-1, App. B.4: one profile pass of the stack at
        n_ref = len(x) tokens with per-forward CUDA-event timing; t_c = wall time of the
        resident layer 0 (pure compute), t_e = max wall time of the layers >= 1 (each the
        envelope max(compute, transfer)); C_dummy = f_tok * n_ref with f_tok the per-token
        FLOPs of one MoE layer (2HE + 6kHh); returns T = gamma * (t_e/t_c) * C_dummy in FLOPs
        and in tokens per GPU (T / f_tok), plus the measured (t_c, t_e)."""
        gamma = float(self.cfg.gamma) if gamma is None else gamma
        A.asyncep_reset_stage_times(self.ctx)
        self.run(x, local_shards=local_shards)
        r = A.asyncep_calibrate_T(self.ctx, gamma, x.shape[0])
        r["n_ref"] = x.shape[0]
        return r
