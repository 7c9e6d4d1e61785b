"""Shared parity harness: seeded inputs (synth) -> the CUDA layer (libsmile via its
binding) and the CPU oracle, side by side.  Test infrastructure only."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth


class Case:
    def __init__(self, n, m, e, T, d, d_ff, cf, dtype="fp32", mode="bilevel", dist="balanced", seed=0,
                 fused=False, alpha=None, beta=0.005, ffn_impl="auto", bias=True):
        self.n, self.m, self.e, self.T, self.d, self.d_ff, self.cf = n, m, e, T, d, d_ff, cf
        self.dtype, self.mode, self.dist, self.seed, self.fused = dtype, mode, dist, seed, fused
        self.flat = mode == "flat"
        self.alpha = alpha if alpha is not None else (0.01 if self.flat else 0.005)
        self.beta = beta
        self.ffn_impl = ffn_impl
        self.cfg = oracle.Config(n, m, e, T, cf, flat=self.flat, alpha=self.alpha, beta=beta)
        self.G = n * m
        KW = self.cfg.logit_width
        self.x = synth.tokens(self.G, T, d, seed=seed, dtype=dtype)
        if fused:
            self.w_router = synth.router_weights(KW, d, seed=seed)
            self.logits = None
        else:
            self.w_router = None
            self.logits = synth.supplied_logits(self.G, T, KW, seed=seed, dist=dist, K1=n if not self.flat else None)
        self.W1, self.b1, self.W2, self.b2 = synth.expert_weights(self.G * e, d, d_ff, seed=seed, dtype=dtype,
                                                                  bias=bias)

    # ---- GPU side ------------------------------------------------------------------
    def gpu_tensors(self, dev="cuda"):
        tdt = torch.bfloat16 if self.dtype == "bf16" else torch.float32
        t = lambda a, dt=tdt: torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dt).contiguous()
        g = dict(x=t(self.x),
                 W1t=t(self.W1.transpose(0, 2, 1)), W2t=t(self.W2.transpose(0, 2, 1)),
                 b1=t(self.b1, torch.float32), b2=t(self.b2, torch.float32))
        g["logits"] = None if self.logits is None else t(self.logits, torch.float32)
        g["w_router"] = None if self.w_router is None else t(self.w_router, torch.float32)
        return g

    def run_gpu(self, layer=None, g=None):
        from paper_2212_05191_b200 import SmileLayer
        if layer is None:
            layer = SmileLayer(self.n, self.m, self.e, self.d, self.d_ff, self.T, self.cf, self.dtype, self.mode,
                               ffn_impl=self.ffn_impl)
        g = g or self.gpu_tensors()
        out = torch.empty_like(g["x"])
        loss = torch.empty(layer.V, dtype=torch.float64, device=g["x"].device)
        layer.forward(g["x"], g["W1t"], g["b1"], g["W2t"], g["b2"], out, loss, logits=g["logits"],
                      w_router=g["w_router"], alpha=self.alpha, beta=self.beta)
        torch.cuda.synchronize()
        err = layer.get_error()
        return layer, out, loss, err

    # ---- oracle side ---------------------------------------------------------------
    def oracle_route(self, logits=None):
        lg = self.logits if logits is None else logits
        if lg is None:
            lg = oracle.logits(self.x.reshape(-1, self.d), self.w_router).reshape(self.G, self.T, -1)
        return oracle.route(self.cfg, lg)

    def oracle_out(self, r, rows=None):
        return oracle.out_rows(self.cfg, r, self.x, self.W1, self.b1, self.W2, self.b2, rows=rows)


def assert_close_scaled(got, ref, rtol, what=""):
    """allclose with atol = rtol * max|ref| (SURVEY §8(c) tolerance convention)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    atol = rtol * max(np.abs(ref).max(), 1e-30)
    err = np.abs(got - ref) - (atol + rtol * np.abs(ref))
    if (err > 0).any():
        idx = np.unravel_index(np.argmax(err), err.shape)
        raise AssertionError(f"{what}: {int((err > 0).sum())} mismatches; worst at {idx}: got {got[idx]} "
                             f"ref {ref[idx]} (rtol {rtol}, atol {atol:.3e})")


def dense_rows(case, r, stride=32):
    """Global token rows g = rank*T + t for full-size output parity:
    at least one row of every `stride`-row strip of every expert segment (the tcgen05 FFN
    works in 32-row strips, so stride 32 touches every strip and hence every M tile), the
    first and last row of every segment, and every dropped token.  Pure index bookkeeping
    on the oracle's route (no arithmetic of the method)."""
    G, T, m, e = case.G, case.T, case.m, case.e
    g = np.arange(G * T)
    rr = g // T
    d1 = r.dest1.reshape(-1).astype(np.int64)
    s1 = r.slot1.reshape(-1).astype(np.int64)
    keep = r.keep.reshape(-1).astype(bool)
    if case.flat:
        key = ((d1 // e) * G + rr) * e + d1 % e          # (expert rank, source rank, local expert)
        pos = s1
        cnt = r.counts1[rr, d1]
    else:
        K2, C1 = r.K2, r.C1
        d2 = r.dest2.reshape(-1).astype(np.int64)
        s, l = rr // m, rr % m
        u = d1 * m + l
        keep1 = r.keep1.reshape(-1).astype(bool)
        pos = np.full(G * T, -1, np.int64)
        pos[keep1] = r.slot2[u[keep1], s[keep1] * C1 + s1[keep1]]
        key = ((d1 * m + d2 // e) * m + l) * e + d2 % e  # (expert rank, source intermediate, local expert)
        cnt = r.counts2[u, d2]
    sel = keep & ((pos % stride == 0) | (pos == cnt - 1))
    rows = np.flatnonzero(sel | ~keep)
    # every segment that holds rows contributes its first and last row
    ks = key[keep]
    assert np.unique(ks[(pos[keep] == 0)]).size == np.unique(ks).size
    return rows
