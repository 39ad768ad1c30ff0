"""Acceptance procedure of the CUDA path against the oracle (S5).

Per layer, on the same seeded inputs:
  1. K = tokens whose oracle gap logit_(k) - logit_(k+1) >= 1e-4 (north_star).
  2. On K: sorted GPU ids == sorted oracle ids exactly; |w_gpu - w_oracle| <= 1e-5.
  3. Counts over K from the GPU ids == oracle counts over K; the GPU-emitted counts equal
     the histogram of the GPU ids over all tokens.
  4. Output: err = max|y - y*| / max|y*| (reading R7) <= tol (2e-2 BF16), where y* is the
     oracle evaluated with the GPU's routing for tokens outside K (reading R15: both
     routings are correct for a near tie; elsewhere the ids are equal by step 2).
"""
from __future__ import annotations

import numpy as np

import oracle

GAP = 1e-4


def bf16_to_f32(t) -> np.ndarray:
    import torch
    return t.detach().to("cpu", torch.float32).numpy()


def check_router(ids_gpu, w_gpu, counts_gpu, orc, E):
    """Steps 1-3.  Returns (mask K, report dict)."""
    K = orc["gap"] >= GAP
    ids_s = np.sort(ids_gpu, axis=1)
    oid_s = np.sort(orc["ids"], axis=1)
    bad = K & ~np.all(ids_s == oid_s, axis=1)
    assert not bad.any(), f"{bad.sum()} non-near-tie tokens route differently (first {np.nonzero(bad)[0][:5]})"
    # weights compared per expert id
    og = np.argsort(orc["ids"], axis=1)
    gg = np.argsort(ids_gpu, axis=1)
    w_o = np.take_along_axis(orc["w"], og, 1)
    w_g = np.take_along_axis(w_gpu.astype(np.float64), gg, 1)
    werr = np.abs(w_o - w_g)[K].max(initial=0.0)
    assert werr <= 1e-5, f"routing weight error {werr}"
    if counts_gpu is not None:
        assert np.array_equal(counts_gpu, np.bincount(ids_gpu.ravel(), minlength=E)), "counts != histogram(ids)"
    cK_g = np.bincount(ids_gpu[K].ravel(), minlength=E)
    cK_o = np.bincount(orc["ids"][K].ravel(), minlength=E)
    assert np.array_equal(cK_g, cK_o), "counts over K differ"
    return K, dict(K_frac=float(K.mean()), w_err=float(werr), n_subst=int((~K).sum()))


def output_error(y_gpu: np.ndarray, y_ref: np.ndarray) -> dict:
    d = np.abs(y_gpu.astype(np.float64) - y_ref)
    scale = np.abs(y_ref).max()
    return dict(err=float(d.max() / scale) if scale > 0 else float(d.max()),
                rel_l2=float(np.linalg.norm(y_gpu - y_ref) / max(np.linalg.norm(y_ref), 1e-300)),
                tok_inf=float((d.max(1) / np.maximum(np.abs(y_ref).max(1), 1e-300)).max()))


def check_layer(x, wr, wg, wu, wd, k, y_gpu, ids_gpu, w_gpu, counts_gpu, residual=True, tol=2e-2,
                norm_topk=True, act_quant=False):
    """Full acceptance for one layer on tokens x (numpy fp32, bf16-valued).  ``counts_gpu``
    must be None when x is a sample of the tokens the GPU counted."""
    E = wr.shape[0]
    orc = oracle.router(x, wr, k, norm_topk=norm_topk)
    K, rep = check_router(ids_gpu, w_gpu, counts_gpu, orc, E)
    ref = oracle.moe_layer(x, wr, wg, wu, wd, k, norm_topk=norm_topk, residual=residual, ids_in=ids_gpu,
                           act_quant=act_quant)
    rep.update(output_error(y_gpu, ref["y"]))
    assert rep["err"] <= tol, f"output error {rep['err']} > {tol} ({rep})"
    return rep
