"""FP8 experts (BASELINE config 4 shape; reading R6): e4m3 weights with per-row scales,
per-token e4m3 activations, kind::f8f6f4 tcgen05 GEMMs.  Acceptance (north_star): FP8
outputs within 6e-2 (R7 metric) of the plain oracle evaluated with the dequantised FP8
weights; secondary bound 1e-2 against the oracle that emulates the activation
quantisation rule; ids / counts as in the BF16 path (the router is BF16)."""
import numpy as np
import pytest
import torch

import synth
from gpu_helpers import Workload, f32
from parity import check_layer

pytestmark = pytest.mark.gpu


def run_layer(wl, st, l, x, residual=True):
    T = x.shape[0]
    ids = torch.empty((T, wl.k), dtype=torch.int32, device="cuda")
    w = torch.empty((T, wl.k), dtype=torch.float32, device="cuda")
    counts = torch.empty((wl.E,), dtype=torch.int32, device="cuda")
    y = torch.empty_like(x)
    st.forward(l, x, residual=x if residual else None, y=y, ids=ids, w=w, counts=counts)
    torch.cuda.synchronize()
    return f32(y), ids.cpu().numpy(), w.cpu().numpy(), counts.cpu().numpy()


def test_fp8_weights_bit_identical_cpu_gpu():
    a = synth.expert_weights_fp8(4, 256, 128, 3, 1, device="cpu")
    b = synth.expert_weights_fp8(4, 256, 128, 3, 1, device="cuda")
    for ta, tb in zip(a, b):
        assert torch.equal(ta.view(torch.uint8) if ta.dtype == torch.uint8 else ta.view(torch.int32),
                           tb.cpu().view(torch.uint8) if tb.dtype == torch.uint8 else tb.cpu().view(torch.int32))


@pytest.mark.parametrize("flags", [0x200, 0], ids=["fused_dispatch", "xperm_default"])
@pytest.mark.parametrize("T", [300, 2048])
def test_fp8_layer_parity(T, flags):
    wl = Workload(L=2, E=16, k=4, H=512, h=256, seed=21, fp8=True)
    st = wl.stack(max_tokens=2048, flags=flags)
    x = wl.tokens(T)
    for l in range(2):
        y, ids, w, counts = run_layer(wl, st, l, x, residual=False)
        wr, g, u, d = wl.host_layer(l)
        plain = check_layer(f32(x), wr, g, u, d, wl.k, y, ids, w, counts, residual=False, tol=6e-2)
        emul = check_layer(f32(x), wr, g, u, d, wl.k, y, ids, w, None, residual=False, tol=1e-2,
                           act_quant=True)
        print(l, "plain", plain, "emulated", emul)
        x = torch.from_numpy(y).to("cuda", torch.bfloat16) + x


def test_fp8_qwen3_235b_shape_sampled():
    """Config 4 layer shape at 32,768 tokens/GPU; 64 sampled tokens against both oracles."""
    T = 32768
    wl = Workload(L=1, E=128, k=8, H=4096, h=1536, seed=0, fp8=True)
    st = wl.stack(max_tokens=T)
    x = wl.tokens(T)
    y, ids, w, counts = run_layer(wl, st, 0, x, residual=False)
    assert np.array_equal(counts, np.bincount(ids.ravel(), minlength=wl.E))
    del st
    torch.cuda.empty_cache()
    idx = np.unique(np.concatenate([[0, T - 1], np.random.default_rng(2).choice(T, 62, replace=False)]))
    wr, g, u, d = wl.host_layer(0)
    xs = f32(x)[idx]
    print("plain", check_layer(xs, wr, g, u, d, 8, y[idx], ids[idx], w[idx], None, residual=False, tol=6e-2))
    print("emul", check_layer(xs, wr, g, u, d, 8, y[idx], ids[idx], w[idx], None, residual=False, tol=1e-2,
                              act_quant=True))


@pytest.mark.parametrize("H", [1024, 2048])
@pytest.mark.parametrize("T", [1, 777, 4096])
def test_fp8_fused_dispatch_bitwise(T, H):
    """GEMM1 gathering e4m3 token rows itself (FLAG_FUSED_DISPATCH: token-major x_q + per-token
    scale) computes exactly what the materialised X_perm path (the FP8 default) computes; H = 2048
    runs the register-resident quantisation kernel."""
    wl = Workload(L=1, E=64, k=6, H=H, h=512, seed=5, fp8=True)
    x = wl.tokens(T)
    outs = []
    for flags in (0x200, 0):
        st = wl.stack(max_tokens=4096, flags=flags)
        outs.append(run_layer(wl, st, 0, x)[0])
        del st
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))


@pytest.mark.parametrize("shape,T,zipf", [((128, 8, 2048, 768), 16384, 0.0), ((128, 8, 4096, 1536), 32768, 0.35)],
                         ids=["qwen3_30b_16k", "qwen3_235b_zipf"])
def test_fp8_other_configs_sampled(shape, T, zipf):
    """FP8 experts on the other BASELINE workloads: the Qwen3-30B layer shape (config 2) and the
    Zipf-skewed routing of config 5 (s = 0.35, reading R14) -- 48 sampled tokens against both oracles,
    the counts against the histogram of the GPU ids over all tokens."""
    E, k, H, h = shape
    wl = Workload(L=1, E=E, k=k, H=H, h=h, seed=3, fp8=True, zipf_s=zipf)
    st = wl.stack(max_tokens=T)
    x = wl.tokens(T)
    y, ids, w, counts = run_layer(wl, st, 0, x, residual=False)
    assert np.array_equal(counts, np.bincount(ids.ravel(), minlength=E)) and counts.sum() == T * k
    if zipf:
        assert counts.max() / max(counts.min(), 1) >= 8
    del st
    torch.cuda.empty_cache()
    idx = np.unique(np.concatenate([[0, T - 1], np.random.default_rng(4).choice(T, 46, replace=False)]))
    wr, g, u, d = wl.host_layer_subset(0, ids[idx].ravel())
    xs = f32(x)[idx]
    check_layer(xs, wr, g, u, d, k, y[idx], ids[idx], w[idx], None, residual=False, tol=6e-2)
    check_layer(xs, wr, g, u, d, k, y[idx], ids[idx], w[idx], None, residual=False, tol=1e-2, act_quant=True)
