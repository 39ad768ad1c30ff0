"""Shared builders for the GPU tests: seeded synthetic stacks (synth) run through the
library (paper_2605_02960_b200), plus host copies of the same weights for the oracle."""
from __future__ import annotations

import numpy as np
import torch

import synth


def f32(t) -> np.ndarray:
    return t.detach().to("cpu", torch.float32).numpy()


class Workload:
    """Natural-layout weights of an L-layer stack, generated on demand on any device."""

    def __init__(self, L, E, k, H, h, seed=0, zipf_s=0.0, fp8=False, draw=None):
        self.L, self.E, self.k, self.H, self.h, self.seed, self.zipf_s = L, E, k, H, h, seed, zipf_s
        self.fp8 = fp8
        # draw="cpu": generate on the host and copy (synth is bit-identical on both), so a tiny
        # run launches no torch kernels besides copies (smoke(): the driver's launch capture)
        self.draw = draw

    def _on(self, device, fn):
        if self.draw is None:
            return fn(device)
        out = fn(self.draw)
        return tuple(t.to(device) for t in out) if isinstance(out, tuple) else out.to(device)

    def router(self, l, device="cuda"):
        return self._on(device, lambda d: synth.router_weight(self.E, self.H, self.seed, l, device=d,
                                                              zipf_s=self.zipf_s))

    def experts(self, l, experts=None, device="cuda"):
        if self.fp8:
            return self._on(device, lambda d: synth.expert_weights_fp8(self.E, self.H, self.h, self.seed, l,
                                                                       device=d, experts=experts))
        return self._on(device, lambda d: synth.expert_weights(self.E, self.H, self.h, self.seed, l, device=d,
                                                               experts=experts))

    def tokens(self, T, device="cuda"):
        return self._on(device, lambda d: synth.tokens(T, self.H, self.seed, device=d, zipf_s=self.zipf_s))

    def host_layer(self, l):
        """fp32 numpy copies for the oracle (drawn on the GPU: synth is bit-identical).
        FP8 experts are dequantised code * row scale (exact up to one fp32 rounding)."""
        wr = f32(self.router(l))
        if self.fp8:
            import oracle
            g, u, d, gs, us, ds = self.experts(l)
            deq = lambda c, s: oracle.e4m3_decode(c.cpu().numpy()) * s.cpu().numpy()[..., None]
            return wr, deq(g, gs), deq(u, us), deq(d, ds)
        g, u, d = self.experts(l)
        return wr, f32(g), f32(u), f32(d)

    def stack(self, max_tokens, **kw):
        from paper_2605_02960_b200.stack import MoEStack
        return MoEStack(self.L, self.E, self.k, self.H, self.h, max_tokens,
                        lambda l: self.router(l), lambda l, ex: self.experts(l, ex), fp8=self.fp8, **kw)

    def host_layer_subset(self, l, experts):
        """Like host_layer, but only the listed experts' weights are filled (the others stay zero
        pages of np.zeros, never touched by an oracle call whose routing avoids them).  FP8 codes are
        decoded on the device through the oracle's own 256-entry decode table (oracle.e4m3_decode of
        every byte), then scaled by the row scale -- the same values host_layer produces."""
        E, H, h = self.E, self.H, self.h
        wr = f32(self.router(l))
        g = np.zeros((E, h, H), np.float32)
        u = np.zeros((E, h, H), np.float32)
        d = np.zeros((E, H, h), np.float32)
        table = None
        if self.fp8:
            import oracle
            table = torch.from_numpy(oracle.e4m3_decode(np.arange(256, dtype=np.uint8))).cuda()
        for e in sorted(set(int(v) for v in experts)):
            if self.fp8:
                gc, uc, dc, gs, us, ds = self.experts(l, range(e, e + 1))
                deq = lambda c, sc: (table[c.long()] * sc[..., None]).cpu().numpy()[0]
                g[e], u[e], d[e] = deq(gc, gs), deq(uc, us), deq(dc, ds)
            else:
                ge, ue, de = self.experts(l, range(e, e + 1))
                g[e], u[e], d[e] = f32(ge)[0], f32(ue)[0], f32(de)[0]
        return wr, g, u, d
