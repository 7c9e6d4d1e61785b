"""Pins of the oracle's full-size helpers (oracle_logits_mt, oracle_out_rows_mt,
oracle_backward_sampled; SURVEY §8(d) "OpenMP over tokens"): each must return exactly --
bit for bit -- what the serial, already-pinned function returns for the same entries
(tests/test_oracle_routing.py, test_oracle_ffn_loss.py, test_oracle_backward.py pin those
to closed forms, brute force and finite differences).  CPU only."""
import numpy as np
import pytest

import oracle
import synth


def _case(n, m, e, T, d, d_ff, cf, flat, seed, fused):
    cfg = oracle.Config(n, m, e, T, cf, flat=flat, alpha=0.01 if flat else 0.005)
    G, KW = n * m, cfg.logit_width
    x = synth.tokens(G, T, d, seed=seed, dtype="bf16")
    W = synth.router_weights(KW, d, seed=seed) if fused else None
    lg = oracle.logits(x.reshape(-1, d), W).reshape(G, T, KW) if fused else \
        synth.supplied_logits(G, T, KW, seed=seed, dist="skewed", K1=None if flat else n)
    W1, b1, W2, b2 = synth.expert_weights(G * e, d, d_ff, seed=seed, dtype="bf16")
    return cfg, x, W, lg, W1, b1, W2, b2


def test_logits_mt_bit_identical():
    x = synth.tokens(3, 101, 96, seed=1)
    W = synth.router_weights(7, 96, seed=1)
    a = oracle.logits(x.reshape(-1, 96), W)
    b = oracle.logits(x.reshape(-1, 96), W, threads=True)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("flat", [False, True])
def test_out_rows_mt_bit_identical(flat):
    cfg, x, W, lg, W1, b1, W2, b2 = _case(2, 2, 2, 150, 32, 64, 1.0, flat, 3, False)
    r = oracle.route(cfg, lg)
    rows = np.arange(cfg.G * cfg.T)[::3]
    a = oracle.out_rows(cfg, r, x, W1, b1, W2, b2, rows=rows)
    b = oracle.out_rows(cfg, r, x, W1, b1, W2, b2, rows=rows, threads=True)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert (r.keep.reshape(-1)[rows] == 0).any()          # dropped rows included (zeros)


@pytest.mark.parametrize("n,m,e,flat,fused", [(2, 2, 1, False, True), (2, 2, 2, False, False),
                                              (2, 1, 2, True, True), (1, 2, 2, False, True)])
def test_backward_sampled_bit_identical(n, m, e, flat, fused):
    """Every entry oracle_backward_sampled returns equals oracle_backward's (same loops, same
    order; only the evaluated subset differs)."""
    T, d, d_ff = 40, 16, 24
    cfg, x, W, lg, W1, b1, W2, b2 = _case(n, m, e, T, d, d_ff, 0.75, flat, 5, fused)
    r = oracle.route(cfg, lg)
    assert (r.keep == 0).any()
    gout = synth.round_bf16(np.random.default_rng(9).normal(size=x.shape).astype(np.float32))
    full = oracle.backward(cfg, r, x, W1, b1, W2, b2, gout, lam=2.0, W=W, logits=None if fused else lg)
    toks = np.array([0, 3, 7, T + 1, cfg.G * T - 1] + list(np.flatnonzero(r.keep.reshape(-1) == 0)[:3]))
    cols = np.array([0, 5, d_ff - 1], np.int32)
    s = oracle.backward_sampled(cfg, r, x, W1, b1, W2, b2, gout, toks, cols, lam=2.0, W=W,
                                logits=None if fused else lg)
    G, KW = cfg.G, cfg.logit_width
    eq = lambda u, v: np.array_equal(np.asarray(u).view(np.uint64), np.ascontiguousarray(v).view(np.uint64))
    assert eq(s["dlogits"], full["dlogits"].reshape(G * T, KW)[toks])
    assert eq(s["dx"], full["dx"].reshape(G * T, d)[toks])
    assert eq(s["dW1c"], full["dW1"][:, :, cols])
    assert eq(s["db1c"], full["db1"][:, cols])
    assert eq(s["dW2r"], full["dW2"][:, cols, :])
    assert eq(s["db2"], full["db2"])
