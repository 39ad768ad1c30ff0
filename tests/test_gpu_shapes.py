"""Seeded random-shape sweep against the oracle (SURVEY S8(c) acceptance, tests/parity.py): shapes the
fixed-shape tests do not reach -- odd expert counts (the router pads E to a multiple of 16 and masks
the padding experts out of the top-k; 1-CTA or CTA-pair router tiles), top-k up to 16, hidden sizes
that are not powers of two, ragged token counts -- each run through one forward of the product path
(tcgen05 router and grouped GEMMs, swap-AB tails where they apply) and checked element by element
against the fp64 oracle; FP8 experts also against the oracle's emulation of the intermediate's
quantisation (reading R6)."""
import numpy as np
import pytest
import torch

from gpu_helpers import Workload, f32
from parity import check_layer

pytestmark = pytest.mark.gpu


def _shape(i):
    rng = np.random.default_rng(1000 + i)
    E = int(rng.choice([3, 8, 23, 37, 64, 80, 96, 120, 128, 144, 200, 256]))
    k = int(rng.integers(1, min(E, 16) + 1))
    H = int(rng.choice([256, 512, 768, 1024, 1280]))
    h = int(rng.choice([128, 256, 384, 512]))
    T = int(rng.integers(1, 700))
    return E, k, H, h, T


CASES = [(_shape(i), False) for i in range(10)] + [(_shape(100 + i), True) for i in range(5)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "{}-E{}k{}H{}h{}T{}".format("fp8" if c[1] else "bf16", *c[0]))
def test_random_shape_layer_parity(case):
    (E, k, H, h, T), fp8 = case
    wl = Workload(L=1, E=E, k=k, H=H, h=h, seed=E + H + T, fp8=fp8)
    st = wl.stack(max_tokens=T)
    x = wl.tokens(T)
    ids = torch.empty((T, k), dtype=torch.int32, device="cuda")
    w = torch.empty((T, k), dtype=torch.float32, device="cuda")
    counts = torch.empty((E,), dtype=torch.int32, device="cuda")
    y = torch.empty_like(x)
    st.forward(0, x, residual=x, y=y, ids=ids, w=w, counts=counts)
    torch.cuda.synchronize()
    ids_h, counts_h = ids.cpu().numpy(), counts.cpu().numpy()
    assert ids_h.min() >= 0 and ids_h.max() < E, "a padding expert was selected"
    assert counts_h.sum() == T * k
    wr, g, u, d = wl.host_layer(0)
    if fp8:
        print(check_layer(f32(x), wr, g, u, d, k, f32(y), ids_h, w.cpu().numpy(), counts_h, tol=6e-2))
        print(check_layer(f32(x), wr, g, u, d, k, f32(y), ids_h, w.cpu().numpy(), None, tol=1e-2,
                          act_quant=True))
    else:
        print(check_layer(f32(x), wr, g, u, d, k, f32(y), ids_h, w.cpu().numpy(), counts_h))
