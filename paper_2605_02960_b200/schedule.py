"""Host-side AsyncEP plan: expert shard layout and the per-layer issue order.

PAPER.md:311 (S6.2 "Weight layout and execution"): every GPU holds 1/N of each MoE
layer's experts "partitioned by expert index", and all GPUs "additionally replicat[e] the
complete expert set for the first MoE layer".  PAPER.md:630 (App. B.1, "MoE gatherer"):
the AllGather of layer i+1 is issued as soon as layer i starts, with one wait before
layer i+1 computes.  With two slots, slot l % 2 holds layer l; the gather of layer l+2
into the same slot may only start after layer l's GEMMs (event slot_free[l % 2]).

Pure Python, no device work: used by ``stack.MoEStack.run`` and tested on CPU over a
real gloo process group (tests/test_multirank_gloo.py).
"""
from __future__ import annotations


def shard_range(E: int, N: int, r: int) -> range:
    """Experts owned by rank r: [r*E/N, (r+1)*E/N) (requires E % N == 0)."""
    if N <= 0 or E % N or not 0 <= r < N:
        raise ValueError(f"bad shard spec E={E} N={N} r={r}")
    per = E // N
    return range(r * per, (r + 1) * per)


def layer_resident(l: int, N: int, replicate_layer0: bool = True) -> bool:
    """Resident layers need no gather: all of them at N == 1, layer 0 when replicated."""
    return N == 1 or (l == 0 and replicate_layer0)


def staged_layers(L: int, N: int, replicate_layer0: bool = True):
    """NEXT-2 offload: layers whose shard comes from the host window:
    every layer >= 1 at N == 1, every gathered layer at N > 1."""
    return [l for l in range(L) if (l > 0 if N == 1 else not layer_resident(l, N, replicate_layer0))]


def stack_schedule(L: int, N: int, replicate_layer0: bool = True, offload_w: int = 0):
    """Issue order of one pass over an L-layer stack: a list of ("prefetch", l, slot) and
    ("forward", l, slot) with slot = l % 2 for gathered layers, -1 for resident ones; with a
    host-offload window of offload_w shards also ("stage", l, l % offload_w): the PCIe
    channel runs up to offload_w layers ahead of the layer being gathered (or, at N == 1,
    computed), and a window buffer is re-staged right after its layer has been read."""
    ops = []
    slot = lambda l: -1 if layer_resident(l, N, replicate_layer0) else l % 2
    todo = staged_layers(L, N, replicate_layer0) if offload_w else []
    nxt = 0

    def stage_next():
        nonlocal nxt
        if nxt < len(todo):
            ops.append(("stage", todo[nxt], todo[nxt] % offload_w))
            nxt += 1

    for _ in range(min(offload_w, len(todo))):
        stage_next()
    if not layer_resident(0, N, replicate_layer0):
        ops.append(("prefetch", 0, 0))
        if 0 in todo:
            stage_next()
    for l in range(L):
        if l + 1 < L and not layer_resident(l + 1, N, replicate_layer0):
            ops.append(("prefetch", l + 1, slot(l + 1)))   # overlaps forward(l)
            if N > 1 and (l + 1) in todo:
                stage_next()                                  # its window buffer was read
        ops.append(("forward", l, slot(l)))
        if N == 1 and l in todo:
            stage_next()                                      # forward(l) read its window buffer
    return ops


def check_schedule(ops, L: int, N: int = 2, offload_w: int = 0) -> None:
    """Invariants of the double buffer: every gathered forward(l) reads a slot that holds
    layer l; a slot is re-filled only after the forward of its previous layer; at most two
    gathered layers are in flight.  With an offload window: a layer is staged before it is
    gathered (N > 1) or computed (N == 1), and a window buffer is re-staged only after its
    previous layer was read.  Raises AssertionError on violation."""
    held = {0: None, 1: None}          # slot -> layer gathered into it
    consumed = {0: True, 1: True}      # its forward has been issued
    whold = {}                         # window buffer -> staged layer
    wcons = {}                         # ... has been read
    staged = set()
    done = set()
    for op, l, s in ops:
        if op == "stage":
            assert s == l % offload_w, (op, l, s)
            assert wcons.get(s, True), f"stage({l}) overwrites window {s} before layer {whold.get(s)} was read"
            whold[s], wcons[s] = l, False
            staged.add(l)
            continue
        if offload_w and ((op == "prefetch") or (op == "forward" and N == 1 and l > 0)):
            assert l in staged and whold.get(l % offload_w) == l and not wcons[l % offload_w], \
                f"{op}({l}) before its layer was staged"
            wcons[l % offload_w] = True
        if op == "prefetch":
            assert s == l % 2, (op, l, s)
            assert consumed[s], f"prefetch({l}) would overwrite slot {s} before forward({held[s]})"
            held[s], consumed[s] = l, False
        elif op == "forward":
            if s >= 0:
                assert held[s] == l and not consumed[s], f"forward({l}) without its gather"
                consumed[s] = True
            assert all(p in done for p in range(l)), "layers out of order"
            done.add(l)
        else:
            raise AssertionError(op)
        assert sum(1 for x in (0, 1) if not consumed[x]) <= 2
    assert done == set(range(L))
