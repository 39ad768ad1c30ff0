"""The N > 1 host path on CPU: world_size-2 (and 4) gloo process groups.

Each rank holds, for layers >= 1, only its shard of experts [rE/N, (r+1)E/N) and the full
layer 0; it walks the product's schedule (paper_2605_02960_b200.schedule:
prefetch of layer l+1 before forward of layer l, two slots), performs the gather as a real
collective (dist.all_gather over gloo, rank-major), and computes each layer on its OWN
data-parallel tokens with the CPU oracle.  Checks: every gathered slot equals the unsharded
layer bit for bit; each rank's output equals a single-process resident run bit for bit;
the schedule obeys the double-buffer invariants.  No data-path collective is used."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2605_02960_b200.schedule import (check_schedule, layer_resident, shard_range, stack_schedule,
                                            staged_layers)

L, E, K, H, h, T = 4, 8, 2, 64, 128, 40


def _natural(l, experts):
    g, u, d = synth.expert_weights(E, H, h, 0, l, device="cpu", experts=experts)
    return g.float().numpy(), u.float().numpy(), d.float().numpy()


def _router(l):
    return synth.router_weight(E, H, 0, l, device="cpu").float().numpy()


def _flat(g, u, d):
    return np.concatenate([g.ravel(), u.ravel(), d.ravel()]).astype(np.float32)


def _unflat(buf, n):
    a, b = n * h * H, 2 * n * h * H
    return buf[:a].reshape(n, h, H), buf[a:b].reshape(n, h, H), buf[b:].reshape(n, H, h)


def _run_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        per = E // world
        # this rank's resident weights: full layer 0, shards of layers >= 1 (expert-major, per-expert blobs)
        mine = {}
        for l in range(L):
            ex = range(E) if layer_resident(l, world) else shard_range(E, world, rank)
            mine[l] = np.concatenate([_flat(*_natural(l, range(e, e + 1))) for e in ex])
        slots = [None, None]
        x = synth.tokens(T, H, 100 + rank).float().numpy()    # DP: each rank its own tokens
        cur = x
        ops = stack_schedule(L, world)
        check_schedule(ops, L)
        slot_ok = True
        for op, l, s in ops:
            if op == "prefetch":
                parts = [torch.empty(mine[l].shape[0], dtype=torch.float32) for _ in range(world)]
                dist.all_gather(parts, torch.from_numpy(mine[l]))          # rank-major
                slots[s] = torch.cat(parts).numpy()
                full = np.concatenate([_flat(*_natural(l, range(e, e + 1))) for e in range(E)])
                slot_ok &= slots[s].tobytes() == full.tobytes()
                continue
            blob = mine[l] if s < 0 else slots[s]
            per_e = [_unflat(b, 1) for b in np.split(blob, E)]
            g = np.concatenate([p[0] for p in per_e])
            u = np.concatenate([p[1] for p in per_e])
            d = np.concatenate([p[2] for p in per_e])
            cur = oracle.moe_layer(cur, _router(l), g, u, d, K)["y"].astype(np.float32)
        q.put((rank, slot_ok, cur.tobytes()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_asyncep_gather_schedule_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, slot_ok, out in sorted(res):
        assert slot_ok, f"rank {rank}: gathered slot != unsharded layer"
        # single-process resident reference on the same tokens
        cur = synth.tokens(T, H, 100 + rank).float().numpy()
        for l in range(L):
            g, u, d = _natural(l, range(E))
            cur = oracle.moe_layer(cur, _router(l), g, u, d, K)["y"].astype(np.float32)
        assert out == cur.tobytes(), f"rank {rank}: N={world} output != resident output"


def test_schedule_invariants():
    for N in (1, 2, 8):
        for rep in (True, False):
            for Lx in (1, 2, 5, 8):
                ops = stack_schedule(Lx, N, rep)
                check_schedule(ops, Lx)
                n_pref = sum(1 for o in ops if o[0] == "prefetch")
                assert n_pref == sum(1 for l in range(Lx) if not layer_resident(l, N, rep))
    # NEXT-2 offload windows
    for N in (1, 2, 8):
        for w in (1, 2, 3):
            for Lx in (2, 5, 8):
                ops = stack_schedule(Lx, N, True, w)
                check_schedule(ops, Lx, N, w)
                assert sum(1 for o in ops if o[0] == "stage") == len(staged_layers(Lx, N))
    with pytest.raises(AssertionError):  # computing an unstaged layer
        check_schedule([("forward", 0, -1), ("forward", 1, -1)], 2, 1, 1)
    with pytest.raises(AssertionError):  # re-staging a window before its layer was read
        check_schedule([("stage", 1, 0), ("stage", 2, 0)], 3, 1, 1)
    # a broken order is rejected: two gathers into the same slot before its forward
    with pytest.raises(AssertionError):
        check_schedule([("prefetch", 1, 1), ("prefetch", 3, 1), ("forward", 0, -1)], 4)
    with pytest.raises(AssertionError):
        check_schedule([("forward", 0, -1), ("forward", 1, 1)], 2)
    assert list(shard_range(128, 8, 3)) == list(range(48, 64))
    with pytest.raises(ValueError):
        shard_range(100, 8, 0)


def _ep_rank(rank, world, port, q, empty=False):
    """Each rank routes its own tokens (oracle router), exchanges per-expert counts with a
    real gloo all_to_all, and plans the DP x EP exchange with the library's asyncep_ep_plan.
    The plans must agree pairwise: what r sends to d is what d expects from r.  empty: the last
    rank has no tokens this step (it sends nothing but still receives rows for its experts)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_02960_b200 import asyncep as A
        E_ = 16
        per = E_ // world
        x = synth.tokens(300, 64, 50 + rank).float().numpy()
        wr = synth.router_weight(E_, 64, 0, 0, zipf_s=1.0).float().numpy()
        ids = oracle.router(x, wr, 4)["ids"]
        counts = np.bincount(ids.ravel(), minlength=E_).astype(np.int32)
        if empty and rank == world - 1:
            counts[:] = 0
        recv = torch.empty(E_, dtype=torch.int32)
        dist.all_to_all_single(recv, torch.from_numpy(counts), [per] * world, [per] * world)
        cfg = A.make_config(1, E_, 4, 64, 128, world_size=world, rank=rank, max_tokens=300)
        plan = A.asyncep_ep_plan(cfg, counts, recv.numpy())
        sr = torch.from_numpy(plan["send_rows"])
        rr = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(rr, sr, [1] * world, [1] * world)  # what each source plans to send me
        ok = bool(np.array_equal(rr.numpy(), plan["recv_rows"]))
        if empty and rank == world - 1:
            ok = ok and int(plan["send_rows"].sum()) == 0 and int(plan["recv_total"]) > 0
        q.put((rank, ok, int(counts.sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,empty", [(2, False), (4, False), (2, True), (4, True)],
                         ids=["w2", "w4", "w2_empty_rank", "w4_empty_rank"])
def test_ep_exchange_plan_over_gloo(world, empty):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_rank, args=(r, world, port, q, empty)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, n in res:
        assert ok, f"rank {rank}: receive plan disagrees with the senders' plans"
        assert n == (0 if empty and rank == world - 1 else 300 * 4)
