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


def _rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from gpu_helpers import Workload
        wl = Workload(L=L, E=E, k=K, H=H, h=h, seed=41)
        x = wl.tokens(T)
        st = wl.stack(max_tokens=T, world_size=world, rank=rank)
        st.enable_p2p_gather()
        outs = []
        for _ in range(2):  # the second pass reuses both slots
            outs.append(st.run(x).clone())
        torch.cuda.synchronize()
        ref = wl.stack(max_tokens=T).run(x).clone()
        torch.cuda.synchronize()
        ok = all(torch.equal(o.view(torch.int16), ref.view(torch.int16)) for o in outs)
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


def test_two_process_ipc_gather_bitwise_equals_resident():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for rank, ok, err in sorted(res):
        assert ok, f"rank {rank}: {err or 'output differs from the resident stack'}"
