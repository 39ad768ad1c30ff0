"""FP8 experts with the MX intermediate (ASYNCEP_FLAG_MX_ACT, reading R6b): the gate/up GEMM's
epilogue quantises the bf16 intermediate to e4m3 with one E8M0 scale per 32 columns and the down
GEMM runs tcgen05 kind::mxf8f6f4.block_scale MMAs over alternating 256/224-wide N tiles.
Acceptance as for FP8 (north_star): within 6e-2 of the plain oracle; secondary bound 1e-2 against
the oracle that emulates the MX rule (act_quant="mx")."""
import numpy as np
import pytest
import torch

from gpu_helpers import Workload, f32
from parity import check_layer
from test_gpu_fp8 import run_layer

pytestmark = pytest.mark.gpu

MX = 0x100


@pytest.mark.parametrize("flags", [MX | 0x200, MX], ids=["fused_dispatch", "xperm_default"])
@pytest.mark.parametrize("T", [300, 2048])
def test_mx_layer_parity(T, flags):
    """H = 512: one 256-wide, one 224-wide and one clipped 32-wide N tile per row tile."""
    wl = Workload(L=2, E=16, k=4, H=512, h=256, seed=21, fp8=True)
    st = wl.stack(max_tokens=2048, flags=flags)
    x = wl.tokens(T)
    for l in range(2):
        y, ids, w, counts = run_layer(wl, st, l, x, residual=False)
        wr, g, u, d = wl.host_layer(l)
        plain = check_layer(f32(x), wr, g, u, d, wl.k, y, ids, w, counts, residual=False, tol=6e-2)
        emul = check_layer(f32(x), wr, g, u, d, wl.k, y, ids, w, None, residual=False, tol=1e-2, act_quant="mx")
        print(l, "plain", plain, "mx-emulated", emul)
        x = torch.from_numpy(y).to("cuda", torch.bfloat16) + x


@pytest.mark.parametrize("H,h", [(256, 128), (1024, 384), (2048, 768)])
def test_mx_tile_widths(H, h):
    """N-tile coverage of the down GEMM for other widths: H = 256 (one 256 tile), 1024 (256 / 224 /
    256 / 224 / 64), 2048 (... / 128), with h = 128 / 384 / 768 (1, 3, 6 k-blocks of scales)."""
    wl = Workload(L=1, E=8, k=2, H=H, h=h, seed=4, fp8=True)
    st = wl.stack(max_tokens=1024, flags=MX)
    x = wl.tokens(1000)
    y, ids, w, counts = run_layer(wl, st, 0, x, residual=True)
    wr, g, u, d = wl.host_layer(0)
    check_layer(f32(x), wr, g, u, d, wl.k, y, ids, w, counts, residual=True, tol=6e-2)
    check_layer(f32(x), wr, g, u, d, wl.k, y, ids, w, None, residual=True, tol=1e-2, act_quant="mx")


@pytest.mark.parametrize("T", [1, 777, 4096])
def test_mx_fused_dispatch_bitwise(T):
    """The gathered-A GEMM1 (default) and the materialised X_perm path give the same bits with MX."""
    wl = Workload(L=1, E=64, k=6, H=1024, h=512, seed=5, fp8=True)
    x = wl.tokens(T)
    outs = []
    for flags in (MX | 0x200, MX):
        st = wl.stack(max_tokens=4096, flags=flags)
        outs.append(run_layer(wl, st, 0, x)[0])
        del st
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))


@pytest.mark.parametrize("shape,T,zipf", [((128, 8, 4096, 1536), 32768, 0.0), ((128, 8, 2048, 768), 16384, 0.0),
                                          ((128, 8, 4096, 1536), 32768, 0.35)],
                         ids=["qwen3_235b", "qwen3_30b_16k", "qwen3_235b_zipf"])
def test_mx_baseline_configs_sampled(shape, T, zipf):
    """The BASELINE layer shapes with MX: 48 sampled tokens against both oracles, counts against the
    histogram of the GPU ids."""
    E, k, H, h = shape
    wl = Workload(L=1, E=E, k=k, H=H, h=h, seed=3, fp8=True, zipf_s=zipf)
    st = wl.stack(max_tokens=T, flags=MX)
    x = wl.tokens(T)
    y, ids, w, counts = run_layer(wl, st, 0, x, residual=False)
    assert np.array_equal(counts, np.bincount(ids.ravel(), minlength=E)) and counts.sum() == T * k
    del st
    torch.cuda.empty_cache()
    idx = np.unique(np.concatenate([[0, T - 1], np.random.default_rng(4).choice(T, 46, replace=False)]))
    wr, g, u, d = wl.host_layer_subset(0, ids[idx].ravel())
    xs = f32(x)[idx]
    print("plain", check_layer(xs, wr, g, u, d, k, y[idx], ids[idx], w[idx], None, residual=False, tol=6e-2))
    print("mx", check_layer(xs, wr, g, u, d, k, y[idx], ids[idx], w[idx], None, residual=False, tol=1e-2,
                            act_quant="mx"))


@pytest.mark.parametrize("rank", [0, 3])
def test_mx_sharded_stack_bitwise(rank):
    """MX on gathered layers: this rank's experts through its own shard's weight map, the others
    through the slot; the 4-rank emulated stack equals the resident MX stack bitwise."""
    from test_gpu_asyncep import _bits
    wl = Workload(L=3, E=16, k=4, H=512, h=256, seed=29, fp8=True)
    T = 700
    x = wl.tokens(T)
    ref = wl.stack(max_tokens=T, flags=MX).run(x).clone()
    st = wl.stack(max_tokens=T, world_size=4, rank=rank, flags=MX)
    out = st.run(x, local_shards=st.peer_shards()).clone()
    torch.cuda.synchronize()
    assert torch.equal(_bits(out), _bits(ref))


def test_mx_deterministic_and_empty():
    """Two runs give the same bits (no atomics on outputs, dynamic tile order notwithstanding); a
    zero-token forward is a no-op."""
    wl = Workload(L=2, E=32, k=8, H=1024, h=384, seed=13, fp8=True)
    st = wl.stack(max_tokens=3000, flags=MX)
    x = wl.tokens(2999)
    a = st.run(x).clone()
    b = st.run(x).clone()
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    y0 = st.forward(0, x[:0], y=torch.empty_like(x[:0]))  # empty batch is a no-op
    assert y0.shape[0] == 0
