"""The multi-process peer-copy gather (MoEStack.enable_p2p_gather -> asyncep_set_peer_shards) with
two real processes sharing one B200: every rank exports its shard buffers through CUDA IPC
(torch tensor IPC handles over a gloo all_gather_object), maps the other rank's, and runs the
AsyncEP stack with asyncep_prefetch_layer copying the peer shard through the mapping.  Each
rank's output must be BITWISE equal to the single-process resident stack on the same tokens.
(NCCL refuses two ranks on one GPU; the IPC transport does not.)"""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

L, E, K, H, h, T = 4, 16, 4, 256, 256, 900


def _rank(rank, world, port, q, transport="kernel"):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    nccl = transport == "nccl"
    dev = rank if nccl else 0
    torch.cuda.set_device(dev)
    if nccl:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from gpu_helpers import Workload
        from paper_2605_02960_b200 import asyncep as A
        wl = Workload(L=L, E=E, k=K, H=H, h=h, seed=41)
        x = wl.tokens(T)
        comm = None
        if nccl:
            dist.all_reduce(torch.ones(1, device="cuda"))
            comm = A.nccl_comm_ptr()
        st = wl.stack(max_tokens=T, world_size=world, rank=rank, nccl_comm=comm)
        if nccl:
            A.asyncep_set_gather_transport(st.ctx, A.GATHER_NCCL, 16)
        else:
            st.enable_p2p_gather()
            A.asyncep_set_gather_transport(st.ctx, A.GATHER_COPY_ENGINE if transport == "ce" else
                                           A.GATHER_COPY_KERNEL, 0)
        ms, nbytes = A.asyncep_probe_gather(st.ctx, 1)  # startup bandwidth probe (collective)
        assert ms > 0 and nbytes == (world - 1) * st.shards[1].numel()
        outs = []
        for _ in range(2):  # the second pass reuses both slots
            outs.append(st.run(x).clone())
        torch.cuda.synchronize()
        if nccl:  # the gathered slot holds the unsharded layer, byte for byte
            full = wl.stack(max_tokens=T).shards[L - 1]
            assert torch.equal(st.slots[(L - 1) % 2], full)
        ref = wl.stack(max_tokens=T).run(x).clone()
        torch.cuda.synchronize()
        ok = all(torch.equal(o.view(torch.int16), ref.view(torch.int16)) for o in outs)
        if nccl:
            # rank 1 has an empty batch: it still joins every AllGather (and both AllToAlls of the
            # EP contrast layer, computing rank 0's rows for its experts); rank 0's output is unchanged
            xin = x if rank == 0 else x[:0]
            o2 = st.run(xin).clone()
            ep_ref = wl.stack(max_tokens=T).run_ep(x).clone()  # N = 1: equals the AsyncEP stack
            o3 = st.run_ep(xin).clone()
            torch.cuda.synchronize()
            if rank == 0:
                ok = ok and torch.equal(o2.view(torch.int16), ref.view(torch.int16))
                ok = ok and torch.equal(o3.view(torch.int16), ep_ref.view(torch.int16))
            else:
                ok = ok and o2.shape[0] == 0 and o3.shape[0] == 0
        dist.barrier()  # keep this rank's shards mapped until the peer is done
        q.put((rank, ok, ""))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, False, f"{type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("transport", ["kernel", "ce"])
def test_two_process_ipc_gather_bitwise_equals_resident(transport):
    """Both peer-copy transports: the co-resident copy kernel and the copy-engine memcpy."""
    _spawn(2, transport)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (NCCL refuses two ranks on one GPU)")
def test_two_gpu_nccl_allgather_bitwise_equals_resident():
    """The north_star path across two real GPUs: ncclAllGather of layer l+1 on the side stream
    (GEMMs leave 16 SMs), slot = the unsharded layer bytes, output = the resident stack."""
    _spawn(2, "nccl")


def _spawn(world, transport):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q, transport)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, ok, err in sorted(res):
        assert ok, f"rank {rank}: {err or 'output differs from the resident stack'}"
