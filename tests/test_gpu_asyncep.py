"""AsyncEP weight streaming on one GPU (Tier 1 at PAPER.md:544).

N ranks are emulated in one process: every "rank" r holds only experts [rE/N,(r+1)E/N) of
layers >= 1 (layer 0 replicated); rank 0 runs the stack with the double-buffered slot and
the same event ordering as the NCCL path, filling the slot by device-to-device copies of
the N shards (asyncep_prefetch_layer_local).  The output must be BITWISE equal to the
resident 1-GPU stack (the gather is a memcpy and the kernels are deterministic)."""
import pytest
import torch

import synth
from gpu_helpers import Workload
from paper_2605_02960_b200 import asyncep as A

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.contiguous().view(torch.int16)


@pytest.mark.parametrize("N,fp8", [(2, False), (4, False), (8, False), (8, True)])
def test_sharded_stack_bitwise_equals_resident(N, fp8):
    wl = Workload(L=5, E=16, k=4, H=256, h=256, seed=11, fp8=fp8)
    T = 1500
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T).run(x).clone()
    ranks = [wl.stack(max_tokens=T, world_size=N, rank=r) for r in range(N)]
    s0 = ranks[0]

    def shards(l):
        return [ranks[r].shards[l] for r in range(N)]

    out = s0.run(x, local_shards=shards).clone()
    torch.cuda.synchronize()
    assert torch.equal(_bits(out), _bits(ref))
    # a second pass reuses both slots (WAR ordering through slot_free events)
    out2 = s0.run(x, local_shards=shards).clone()
    torch.cuda.synchronize()
    assert torch.equal(_bits(out2), _bits(ref))


def test_slot_holds_the_unsharded_layer_bytes():
    wl = Workload(L=3, E=8, k=2, H=64, h=128, seed=12)
    full = wl.stack(max_tokens=64)
    N = 4
    ranks = [wl.stack(max_tokens=64, world_size=N, rank=r) for r in range(N)]
    s0 = ranks[0]
    from paper_2605_02960_b200 import asyncep as A
    A.asyncep_prefetch_layer_local(s0.ctx, 1, [ranks[r].shards[1] for r in range(N)])
    torch.cuda.synchronize()
    # rank-major slot = the unsharded layer, except rank 0's own region: the copy transport does
    # not copy the own shard (the GEMMs read it in place from the rank's resident shard)
    sb = s0.slots[1].numel() // N
    assert torch.equal(s0.slots[1][sb:], full.shards[1][sb:])
    assert torch.equal(ranks[0].shards[1], full.shards[1][:sb])
    # with the SIMT debug GEMM (which reads the whole slot) the own shard is copied too
    s1 = wl.stack(max_tokens=64, world_size=N, rank=0, flags=A.FLAG_SIMT_GEMM)
    A.asyncep_prefetch_layer_local(s1.ctx, 1, [ranks[r].shards[1] for r in range(N)])
    torch.cuda.synchronize()
    assert torch.equal(s1.slots[1], full.shards[1])


def test_prefetch_ordering_errors():
    from paper_2605_02960_b200 import asyncep as A
    wl = Workload(L=4, E=8, k=2, H=64, h=128, seed=13)
    N = 2
    ranks = [wl.stack(max_tokens=64, world_size=N, rank=r) for r in range(N)]
    s0 = ranks[0]
    sh = lambda l: [ranks[r].shards[l] for r in range(N)]
    x = wl.tokens(64)
    y = torch.empty_like(x)
    s0.forward(0, x, y=y)  # layer 0 is replicated: no prefetch needed
    with pytest.raises(A.AsyncEPError) as ei:
        s0.forward(1, x, y=y)
    assert ei.value.status == A.ERR_NOT_PREFETCHED
    A.asyncep_prefetch_layer_local(s0.ctx, 1, sh(1))
    with pytest.raises(A.AsyncEPError) as ei:   # layer 3 would overwrite slot 1 before forward(1)
        A.asyncep_prefetch_layer_local(s0.ctx, 3, sh(3))
    assert ei.value.status == A.ERR_INVALID_ARG
    s0.forward(1, x, y=y)
    A.asyncep_prefetch_layer_local(s0.ctx, 3, sh(3))   # now legal
    with pytest.raises(A.AsyncEPError):
        A.asyncep_prefetch_layer(s0.ctx, 2)  # no NCCL communicator given
    torch.cuda.synchronize()


def test_delayed_gather_only_slows_down():
    """Fault injection: a long spin kernel on the comm stream before the
    gather must not change the output (catches a missing ag_done wait)."""
    wl = Workload(L=3, E=16, k=4, H=256, h=256, seed=14)
    T = 512
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T).run(x).clone()
    N = 2
    ranks = [wl.stack(max_tokens=T, world_size=N, rank=r) for r in range(N)]
    s0 = ranks[0]
    sh = lambda l: [ranks[r].shards[l] for r in range(N)]
    with torch.cuda.stream(s0.comm_stream):
        torch.cuda._sleep(200_000_000)  # ~0.1 s of spinning on the comm stream
    out = s0.run(x, local_shards=sh).clone()
    torch.cuda.synchronize()
    assert torch.equal(_bits(out), _bits(ref))


def test_poisoned_slot_after_use_is_never_read():
    """Poison a slot right after its layer's GEMMs (ordered after slot_free on the comm
    stream); a later layer reading it too early would produce NaN (catches WAR bugs)."""
    from paper_2605_02960_b200 import asyncep as A
    wl = Workload(L=4, E=8, k=2, H=64, h=128, seed=15)
    T = 256
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T).run(x).clone()
    N = 2
    ranks = [wl.stack(max_tokens=T, world_size=N, rank=r) for r in range(N)]
    s0 = ranks[0]
    sh = lambda l: [ranks[r].shards[l] for r in range(N)]
    bufs = [torch.empty_like(x) for _ in range(2)]
    cur = x
    A.asyncep_prefetch_layer_local(s0.ctx, 1, sh(1))
    for l in range(4):
        if l + 1 < 4:
            A.asyncep_prefetch_layer_local(s0.ctx, l + 1, sh(l + 1))
        dst = bufs[l % 2]
        s0.forward(l, cur, residual=cur, y=dst)
        if l >= 1:
            # poison on the comm stream after the event that frees the slot: the next
            # prefetch into this slot is ordered after the poison, so results stay exact
            ev = torch.cuda.Event()
            ev.record(s0.compute_stream)
            s0.comm_stream.wait_event(ev)
            with torch.cuda.stream(s0.comm_stream):
                s0.slots[l % 2].view(torch.int16).fill_(0x7FC0)  # bf16 NaN pattern
        cur = dst
    torch.cuda.synchronize()
    assert torch.equal(_bits(cur), _bits(ref))


def test_peer_shards_and_calibrated_T():
    """MoEStack.peer_shards (1-GPU rank emulation) gives the resident output bitwise, and
    the App. B.4 profile pass returns T = gamma * (t_e / t_c) * C_dummy with the measured
    per-layer wall times."""
    from paper_2605_02960_b200 import asyncep as A
    wl = Workload(L=4, E=16, k=4, H=256, h=256, seed=16)
    T = 1024
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T).run(x).clone()
    st = wl.stack(max_tokens=T, world_size=4, flags=A.FLAG_STAGE_TIMING)
    sh = st.peer_shards()
    out = st.run(x, local_shards=sh).clone()
    torch.cuda.synchronize()
    assert torch.equal(_bits(out), _bits(ref))
    cal = st.calibrate_T(x, local_shards=sh)
    assert cal["t_c_ms"] > 0 and cal["t_e_ms"] > 0
    f_tok = 2 * 256 * 16 + 6 * 4 * 256 * 256
    ratio = max(1.0, cal["t_e_ms"] / cal["t_c_ms"])
    assert cal["T_flops"] == pytest.approx(1.2 * ratio * f_tok * T, rel=1e-6)
    assert cal["T_tokens"] == pytest.approx(1.2 * ratio * T, rel=1e-6)
    times = A.asyncep_forward_times(st.ctx)
    assert [l for l, _ in times][-4:] == [0, 1, 2, 3]


def test_nccl_allgather_path_with_borrowed_torch_comm():
    """The real NCCL path on one GPU: borrow the communicator of a 1-rank torch NCCL process
    group (ProcessGroupNCCL._comm_ptr) in a context configured as rank 0 of 2.  ncclAllGather
    over that 1-rank communicator then writes this rank's shard into the first half of the
    slot (rank-major placement), on the comm stream, ordered by the ag_done event before
    GEMM1.  Checks the comm borrowing, the in-process NCCL symbol resolution, the stream and
    event plumbing end to end."""
    import os
    import socket

    import torch.distributed as dist
    from paper_2605_02960_b200 import asyncep as A

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        dist.all_reduce(torch.ones(1, device="cuda"))
        comm = A.nccl_comm_ptr()
        assert comm
        wl = Workload(L=3, E=8, k=2, H=64, h=128, seed=17)
        full = wl.stack(max_tokens=64)
        st = wl.stack(max_tokens=64, world_size=2, rank=0, nccl_comm=comm)
        st.slots[1].fill_(0xAB)
        A.asyncep_prefetch_layer(st.ctx, 1)
        x = wl.tokens(64)
        st.forward(0, x, y=torch.empty_like(x))
        st.forward(1, x, y=torch.empty_like(x))   # waits on the NCCL gather's event
        torch.cuda.synchronize()
        half = st.shards[1].numel()
        assert torch.equal(st.slots[1][:half], st.shards[1])
        assert torch.equal(st.slots[1][:half], full.shards[1][:half])
        assert torch.all(st.slots[1][half:] == 0xAB)  # the absent rank's half is untouched
        # the explicit NCCL transport with SMs reserved for NCCL's kernels, on a dedicated gather
        # communicator whose NCCL config caps its kernels at those SMs, and the startup probe
        _g, gcomm = A.nccl_gather_group(16)
        assert gcomm and gcomm != comm
        A.asyncep_set_gather_comm(st.ctx, gcomm)
        A.asyncep_set_gather_transport(st.ctx, A.GATHER_NCCL, 16)
        st.slots[0].fill_(0xCD)
        ms, nbytes = A.asyncep_probe_gather(st.ctx, 2)
        torch.cuda.synchronize()
        assert ms > 0 and nbytes == half  # (N - 1) x shard bytes
        assert torch.equal(st.slots[0][:half], st.shards[2])
        A.asyncep_prefetch_layer(st.ctx, 2)     # the probe handed the slot back
        st.forward(2, x, y=torch.empty_like(x))
        torch.cuda.synchronize()
        with pytest.raises(A.AsyncEPError):
            A.asyncep_set_gather_transport(st.ctx, A.GATHER_COPY_KERNEL, 0)
            A.asyncep_prefetch_layer(st.ctx, 1)  # copy transport without peer shards
    finally:
        dist.destroy_process_group()


def test_ep_contrast_layer_matches_asyncep_forward():
    """The synchronous DP x EP contrast layer (world_size 1: local exchange) computes the
    same layer bit for bit as the AsyncEP forward (same tiles, same K order)."""
    wl = Workload(L=2, E=16, k=4, H=256, h=256, seed=18)
    T = 777
    x = wl.tokens(T)
    st = wl.stack(max_tokens=T)
    ref = st.run(x).clone()
    out = st.run_ep(x).clone()
    torch.cuda.synchronize()
    assert torch.equal(_bits(out), _bits(ref))


@pytest.mark.parametrize("N,w,fp8", [(1, 1, False), (1, 2, False), (2, 2, False), (4, 3, False), (1, 2, True),
                                     (4, 3, True)])
def test_offload_window_bitwise_equals_resident(N, w, fp8):
    """NEXT-2 hybrid offload: shards in pinned host memory, a w-deep device
    window filled over PCIe on a third stream, then gathered (N > 1, emulated locally) or
    computed directly (N == 1).  Two passes reuse every window buffer; the output must equal
    the resident stack bit for bit (FP8 blobs too: codes and scales travel as bytes)."""
    wl = Workload(L=5, E=16, k=4, H=256, h=256, seed=19, fp8=fp8)
    T = 640
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T).run(x).clone()
    st = wl.stack(max_tokens=T, world_size=N, offload_window=w)
    assert all(st.shards[l] is None for l in range(1, 5))  # no device copy of offloaded layers
    sh = st.peer_shards() if N > 1 else None
    for _ in range(2):
        out = st.run(x, local_shards=sh).clone()
        torch.cuda.synchronize()
        assert torch.equal(_bits(out), _bits(ref))


@pytest.mark.parametrize("N", [2, 4])
def test_copy_engine_gather_bitwise_equals_resident(N):
    """asyncep_set_peer_shards (the copy-engine gather used across real ranks with IPC-mapped
    peer shards) through the plain asyncep_prefetch_layer: bitwise = resident, two passes."""
    wl = Workload(L=4, E=16, k=4, H=256, h=256, seed=31)
    T = 1200
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T).run(x).clone()
    st = wl.stack(max_tokens=T, world_size=N, rank=N - 1)
    sh = st.peer_shards()
    st.set_peer_table([None if st.layer_resident(l) else sh(l) for l in range(wl.L)])
    for _ in range(2):
        out = st.run(x).clone()
        torch.cuda.synchronize()
        assert torch.equal(_bits(out), _bits(ref))
    with pytest.raises(A.AsyncEPError):  # a gathered layer without a peer entry is rejected
        bad = [None] * wl.L
        A.asyncep_set_peer_shards(st.ctx, bad)


def test_gather_copy_transport():
    """asyncep_gather_copy: the co-resident copy kernel for 16-B aligned sizes, cudaMemcpyAsync
    otherwise -- both byte-exact; zero bytes is a no-op."""
    src = torch.randint(0, 256, (3 * (1 << 20) + 48,), dtype=torch.uint8, device="cuda")
    for off, n in ((0, src.numel()), (16, 1 << 20), (1, 12345), (0, 0)):
        dst = torch.zeros_like(src)
        A.asyncep_gather_copy(dst[off:], src[off:], n)
        torch.cuda.synchronize()
        assert torch.equal(dst[off:off + n], src[off:off + n])
        assert int(dst[:off].sum()) == 0 and int(dst[off + n:].sum()) == 0


def test_attention_abi_errors():
    cfg = A.make_attn_config(256, 8, 2, 128, max_tokens=64)
    q = torch.zeros((64, 8, 128), dtype=torch.bfloat16, device="cuda")
    k = torch.zeros((64, 2, 128), dtype=torch.bfloat16, device="cuda")
    vt = torch.zeros((2, 128, 64), dtype=torch.bfloat16, device="cuda")
    cu = torch.tensor([0, 64], dtype=torch.int32, device="cuda")
    o = torch.empty_like(q)
    with pytest.raises(A.AsyncEPError):  # ldv not a multiple of 8
        A.asyncep_attention(cfg, q, k, vt, 63, cu, cu, o)
    with pytest.raises(A.AsyncEPError):  # head_dim must be 128
        A.asyncep_attention(A.make_attn_config(256, 8, 2, 64, max_tokens=64), q, k, vt, 64, cu, cu, o)
    with pytest.raises(A.AsyncEPError):  # q_heads not a multiple of kv_heads
        A.asyncep_attention(A.make_attn_config(256, 6, 4, 128, max_tokens=64), q, k, vt, 64, cu, cu, o)
    A.asyncep_attention(cfg, q, k, vt, 64, cu, cu, o)  # all-zero inputs: uniform attention over v = 0
    torch.cuda.synchronize()
    assert int(torch.count_nonzero(o)) == 0


@pytest.mark.parametrize("L", [2, 3])
def test_stack_output_fed_back_as_input(L):
    """MoEStack.run's returned ping-pong buffer may be passed back in as x: the
    second pass equals running the stack on a private copy, for odd and even L."""
    wl = Workload(L=L, E=16, k=4, H=256, h=256, seed=21)
    T = 700
    st = wl.stack(max_tokens=T)
    y1 = st.run(wl.tokens(T))
    y1_copy = y1.clone()
    y2 = st.run(y1).clone()
    ref = wl.stack(max_tokens=T).run(y1_copy).clone()
    torch.cuda.synchronize()
    assert torch.equal(_bits(y2), _bits(ref))


def test_timeline_orders_gather_before_its_gemms():
    """asyncep_timeline: every gathered layer's GEMM1 starts after its gather ended (the event order
    the slot's ag_done wait enforces), the resident layer 0 has no gather, and forwards follow each
    other on the compute stream."""
    wl = Workload(L=4, E=16, k=4, H=256, h=256, seed=19)
    T = 1024
    x = wl.tokens(T)
    st = wl.stack(max_tokens=T, world_size=4, flags=A.FLAG_STAGE_TIMING)
    sh = st.peer_shards()
    st.run(x, local_shards=sh)
    A.asyncep_timeline_begin(st.ctx)
    st.run(x, local_shards=sh)
    torch.cuda.synchronize()
    recs = A.asyncep_timeline_read(st.ctx)
    fwd = {l: (a, b, c, d) for k, l, a, b, c, d in recs if k == "forward"}
    gat = {l: (a, b) for k, l, a, b, _, _ in recs if k == "gather"}
    assert sorted(fwd) == [0, 1, 2, 3] and sorted(gat) == [1, 2, 3]
    for l in (1, 2, 3):
        assert gat[l][0] <= gat[l][1] <= fwd[l][2] + 1e-3   # GEMM1 waits for the slot
    for l in range(4):
        assert fwd[l][0] <= fwd[l][1] <= fwd[l][2] <= fwd[l][3]
        if l:
            assert fwd[l - 1][3] <= fwd[l][0] + 1e-3
    with pytest.raises(A.AsyncEPError):
        A.asyncep_timeline_read(st.ctx)   # the capture ended


@pytest.mark.parametrize("fp8", [False, True], ids=["bf16", "fp8"])
def test_sharded_stack_with_swap_tails_bitwise(fp8):
    """Swap-AB tail tiles on gathered layers: this rank's own experts come through the second weight
    map (own shard in place), the others through the slot -- both in the swapped orientation; the
    4-rank emulated stack stays bitwise equal to the resident one (both with FLAG_SWAP_TAILS)."""
    wl = Workload(L=3, E=16, k=4, H=512, h=256, seed=29, fp8=fp8)
    T = 700  # ~175-row tails per expert: every expert's last tile is a swap tile
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T, flags=A.FLAG_SWAP_TAILS).run(x).clone()
    for rank in (0, 3):
        st = wl.stack(max_tokens=T, world_size=4, rank=rank, flags=A.FLAG_SWAP_TAILS)
        out = st.run(x, local_shards=st.peer_shards()).clone()
        torch.cuda.synchronize()
        assert torch.equal(_bits(out), _bits(ref)), rank


@pytest.mark.parametrize("fp8", [False, True], ids=["bf16", "fp8"])
def test_stack_step_replays_as_cuda_graph(fp8):
    """A resident stack step (N = 1, no stage timing) captures into one CUDA graph on the stack's
    compute stream: every library call is stream-ordered and host-sync free, and the tensor maps /
    tile tables are rebuilt from the same buffers.  Replays equal eager runs bitwise, also after new
    tokens are copied into the captured input buffer."""
    wl = Workload(L=3, E=16, k=4, H=512, h=256, seed=37, fp8=fp8)
    T = 900
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        st = wl.stack(max_tokens=T, compute_stream=cs)
        x_in = wl.tokens(T).clone()
        out = torch.empty_like(x_in)
        st.run(x_in, out=out)          # warm-up: one-time attributes, lazily built state
        cs.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            st.run(x_in, out=out)
        for seed in (1, 2):
            x_new = synth.tokens(T, 512, 100 + seed, device="cuda")
            x_in.copy_(x_new)
            g.replay()
            cs.synchronize()
            got = out.clone()
            ref = wl.stack(max_tokens=T, compute_stream=cs).run(x_new).clone()
            cs.synchronize()
            assert torch.equal(_bits(got), _bits(ref)), seed


@pytest.mark.parametrize("fp8", [False, True], ids=["bf16", "fp8"])
def test_gated_gather_bitwise_and_no_hang(fp8):
    """asyncep_set_gather_gate: a prefetched layer's gather starts only when the next forward has
    finished its dispatch (the comm stream waits on a device word the compute stream writes); the
    4-rank emulated stack still equals the resident one bitwise over repeated steps, and a prefetch
    with no forward coming is released by turning the gate off."""
    wl = Workload(L=3, E=16, k=4, H=512, h=256, seed=31, fp8=fp8)
    T = 600
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T).run(x).clone()
    st = wl.stack(max_tokens=T, world_size=4, rank=1)
    A.asyncep_set_link_emulation(st.ctx, 770e9)
    A.asyncep_set_gather_gate(st.ctx, True)
    sh = st.peer_shards()
    for _ in range(3):
        out = st.run(x, local_shards=sh).clone()
        torch.cuda.synchronize()
        assert torch.equal(_bits(out), _bits(ref))
    st.prefetch(1, sh)                       # no forward follows
    A.asyncep_set_gather_gate(st.ctx, False)  # releases the waiting gather
    torch.cuda.synchronize()
    st.forward(1, x, y=torch.empty_like(x))  # the slot holds layer 1
    A.asyncep_set_gather_gate(st.ctx, True)  # a new epoch works again
    out = st.run(x, local_shards=sh).clone()
    torch.cuda.synchronize()
    assert torch.equal(_bits(out), _bits(ref))


@pytest.mark.parametrize("gate", [False, True], ids=["ungated", "gated"])
def test_empty_batch_keeps_the_gather_schedule(gate):
    """A DP rank with no tokens this step still takes part in every gather (the other ranks' NCCL
    AllGathers need it): asyncep_moe_forward with num_tokens == 0 computes nothing but releases the
    layer's slot in stream order (and starts a held, gated gather), so the next prefetch into that
    slot proceeds.  Steps with 0 tokens between real steps leave the real steps bitwise equal to the
    resident stack."""
    wl = Workload(L=4, E=16, k=4, H=256, h=256, seed=33)
    T = 300
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T).run(x).clone()
    st = wl.stack(max_tokens=T, world_size=2, rank=0)
    if gate:
        A.asyncep_set_gather_gate(st.ctx, True)
    sh = st.peer_shards()
    empty = x[:0]
    for _ in range(2):
        e = st.run(empty, local_shards=sh)
        assert e.shape == (0, wl.H)
        out = st.run(x, local_shards=sh).clone()
        torch.cuda.synchronize()
        assert torch.equal(_bits(out), _bits(ref))
    # the empty forward still enforces the schedule: a gathered layer that was not prefetched
    with pytest.raises(A.AsyncEPError):
        st.forward(3, empty, y=empty)
