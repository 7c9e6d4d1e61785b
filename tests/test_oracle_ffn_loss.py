"""Pins for the oracle's expert FFN (oracle_ffn_row), layer output (oracle_out_rows),
logits (oracle_logits) and Eq. (4) aux loss: textbook numpy/scipy evaluations, hand
cases, the identity expert, location transparency, and the paper's closed forms.
"""
import math

import numpy as np
import pytest
from scipy.special import erf

import oracle
import synth


def textbook_ffn(x, W1, b1, W2, b2):
    """W2^T GELU(W1^T x + b1) + b2, exact erf GELU, numpy fp64."""
    a = x.astype(np.float64) @ W1.astype(np.float64) + b1
    h = 0.5 * a * (1.0 + erf(a / math.sqrt(2.0)))
    return h @ W2.astype(np.float64) + b2


def test_ffn_zero_weights_and_gelu_fixed_point():
    d, f = 5, 7
    x = np.arange(d, dtype=np.float32)
    z = lambda *s: np.zeros(s, np.float32)
    assert (oracle.ffn_row(x, z(d, f), z(f), z(f, d), z(d)) == 0).all()
    b2 = np.linspace(-1, 1, d).astype(np.float32)
    W1 = np.ones((d, f), np.float32)
    W2 = np.ones((f, d), np.float32)
    np.testing.assert_array_equal(oracle.ffn_row(z(d), W1, z(f), W2, b2), b2)


def test_ffn_hand_case_d2():
    # d = d_ff = 2, hand-evaluated: x = (1, -1), W1 = [[1, 2], [0, 1]],
    # b1 = (0, 1): a = (1, 2 - 1 + 1) = (1, 2);  GELU(1) = Phi(1) = 0.841344746...,
    # GELU(2) = 2 Phi(2) = 1.954499736...; W2 = [[1, 0], [1, -1]], b2 = (0.5, 0):
    # y = (0.841344746 + 1.954499736 + 0.5, -1.954499736)
    x = np.array([1, -1], np.float32)
    W1 = np.array([[1, 2], [0, 1]], np.float32)
    W2 = np.array([[1, 0], [1, -1]], np.float32)
    y = oracle.ffn_row(x, W1, np.array([0, 1], np.float32), W2, np.array([0.5, 0], np.float32))
    phi1, phi2 = 0.8413447460685429, 0.9772498680518208
    np.testing.assert_allclose(y, [phi1 + 2 * phi2 + 0.5, -2 * phi2], rtol=0, atol=1e-14)


def test_ffn_textbook_random():
    rs = np.random.default_rng(1)
    d, f = 48, 80
    for _ in range(5):
        x, W1, b1 = rs.normal(size=d), rs.normal(size=(d, f)) / 7, rs.normal(size=f)
        W2, b2 = rs.normal(size=(f, d)) / 9, rs.normal(size=d)
        args = [a.astype(np.float32) for a in (x, W1, b1, W2, b2)]
        np.testing.assert_allclose(oracle.ffn_row(*args), textbook_ffn(*args), rtol=1e-12, atol=1e-12)


def test_logits_match_numpy_fp64():
    rs = np.random.default_rng(2)
    x = rs.normal(size=(37, 96)).astype(np.float32)
    W = rs.uniform(-0.1, 0.1, size=(6, 96)).astype(np.float32)
    ref = (x.astype(np.float64) @ W.astype(np.float64).T)
    got = oracle.logits(x, W)
    np.testing.assert_allclose(got, ref, rtol=1.2e-7, atol=1e-9)   # <= 1 fp32 ulp of rounding


@pytest.mark.parametrize("flat", [False, True])
def test_identity_expert_gives_gate_times_x(flat):
    cfg = oracle.Config(2, 2, 2, T=40, cf=1.0, flat=flat)
    lg = synth.supplied_logits(cfg.G, cfg.T, cfg.logit_width, seed=4, dist="skewed", K1=cfg.n)
    x = synth.tokens(cfg.G, cfg.T, 8, seed=4)
    r = oracle.route(cfg, lg)
    out = oracle.out_rows(cfg, r, x, identity=True).reshape(cfg.G, cfg.T, 8)
    assert (r.keep == 0).any() and (r.keep == 1).any()          # both branches exercised
    exp = np.where(r.keep[..., None].astype(bool), r.gate[..., None].astype(np.float64) * x, 0.0)
    np.testing.assert_array_equal(out, exp)


def test_location_transparency_eq3():
    """No drops (cf large): each output equals Eq. (3) evaluated in place,
    p_i(x) q_j(x) E_{i,j}(x), with the experts indexed i*K2 + j."""
    n, m, e, T, d, f = 2, 2, 2, 16, 12, 20
    cfg = oracle.Config(n, m, e, T=T, cf=64.0)
    x = synth.tokens(cfg.G, T, d, seed=2)
    W = synth.router_weights(n + m * e, d, seed=2)
    lg = oracle.logits(x.reshape(-1, d), W).reshape(cfg.G, T, -1)
    W1, b1, W2, b2 = synth.expert_weights(cfg.G * e, d, f, seed=2)
    r = oracle.route(cfg, lg)
    assert r.keep.all()
    out = oracle.out_rows(cfg, r, x, W1, b1, W2, b2).reshape(cfg.G, T, d)
    for rk in range(cfg.G):
        for t in range(T):
            z = lg[rk, t].astype(np.float64)
            p = np.exp(z[:n] - z[:n].max()); p /= p.sum()
            q = np.exp(z[n:] - z[n:].max()); q /= q.sum()
            i, j = int(np.argmax(p)), int(np.argmax(q))
            g = i * m * e + j
            ref = p[i] * q[j] * textbook_ffn(x[rk, t], W1[g], b1[g], W2[g], b2[g])
            np.testing.assert_allclose(out[rk, t], ref, rtol=1e-6, atol=1e-7)


# ---- Eq. (4) aux loss -------------------------------------------

def test_lb_uniform_is_alpha_plus_beta():
    # Equal logits: P and Q uniform, so alpha*n*sum f_i/n + beta*m*sum f_j/m = alpha+beta
    # ("min loss_lb = alpha + beta"; 0.01 at alpha = beta = 0.005).
    for n, m, e in [(2, 4, 1), (4, 2, 1), (2, 4, 8)]:
        cfg = oracle.Config(n, m, e, T=32)
        r = oracle.route(cfg, np.zeros((cfg.G, 32, cfg.logit_width), np.float32))
        np.testing.assert_allclose(r.loss, 0.01, rtol=1e-15)
    cfg = oracle.Config(2, 4, 1, T=32, flat=True, alpha=0.01)
    r = oracle.route(cfg, np.zeros((8, 32, 8), np.float32))
    np.testing.assert_allclose(r.loss, 0.01, rtol=1e-15)     # one-hop Switch: alpha


def test_lb_uniform_routing_with_onehot_probabilities():
    # f = P = uniform (each destination chosen by T/K tokens with a margin so large that
    # softmax is one-hot to 1e-17): loss = alpha + beta, the paper's minimum.
    n, m = 4, 2
    cfg = oracle.Config(n, m, 1, T=8)
    lg = np.zeros((cfg.G, 8, n + m), np.float32)
    for t in range(8):
        lg[:, t, t % n] = 40.0
        lg[:, t, n + t % m] = 40.0
    r = oracle.route(cfg, lg)
    np.testing.assert_allclose(r.loss, 0.01, rtol=1e-12)


def test_lb_all_to_node0_onehot():
    # all tokens to node 0 with P one-hot, n = 4, alpha = 0.005, beta = 0 -> 0.02
    cfg = oracle.Config(4, 1, 1, T=6, alpha=0.005, beta=0.0)
    lg = np.zeros((4, 6, 5), np.float32)
    lg[:, :, 0] = 40.0
    r = oracle.route(cfg, lg)
    np.testing.assert_allclose(r.loss, 0.02, rtol=1e-12)


def test_lb_twice_unscaled_and_cauchy_schwarz():
    # P:L226 "twice the unscaled balancing loss": alpha = beta = 1 at uniform -> 2 = 2 x flat.
    cfg = oracle.Config(2, 4, 1, T=16, alpha=1.0, beta=1.0)
    r = oracle.route(cfg, np.zeros((8, 16, 6), np.float32))
    np.testing.assert_allclose(r.loss, 2.0, rtol=1e-15)
    # For one-hot probability batches f = P, so n*sum f_i^2 >= 1 (Cauchy-Schwarz): loss >= a+b.
    rs = np.random.default_rng(0)
    cfg = oracle.Config(3, 2, 1, T=10)
    for _ in range(50):
        lg = np.zeros((6, 10, 5), np.float32)
        for rk in range(6):
            for t in range(10):
                lg[rk, t, rs.integers(0, 3)] = 40.0
                lg[rk, t, 3 + rs.integers(0, 2)] = 40.0
        r = oracle.route(cfg, lg)
        assert (r.loss >= 0.01 - 1e-15).all()


def test_lb_definition_counts():
    # f and P as printed at P:L129-130: A = argmax counts before capacity, S = prob sums.
    cfg = oracle.Config(2, 4, 1, T=64, cf=0.5)
    lg = synth.supplied_logits(8, 64, 6, seed=11, dist="skewed", K1=2)
    r = oracle.route(cfg, lg)
    for rk in range(8):
        np.testing.assert_array_equal(r.A1[rk], np.bincount(np.argmax(lg[rk, :, :2], -1), minlength=2))
        np.testing.assert_array_equal(r.A2[rk], np.bincount(np.argmax(lg[rk, :, 2:], -1), minlength=4))
    assert (r.keep1 == 0).any()      # drops happened; f still counts them (R13)
