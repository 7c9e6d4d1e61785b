"""Pins of the oracle's top-k layer (oracle_route_topk / oracle_out_rows_topk; Eq. (2),
P:L43-47; readings R29-R32 in DESIGN.md) against things other than itself: the k = 1
collapse onto the pinned top-1 router, numpy's stable descending argsort for the choices,
scipy's softmax for the weights, an O((kT)^2) brute-force definition of the choice-major
capacity rule, a closed-form worked example, and the identity-expert output.  CPU only."""
import itertools

import numpy as np
import pytest
from scipy.special import softmax

import oracle
import synth


def _cfg(n, m, e, T, cf):
    return oracle.Config(n, m, e, T, cf, flat=True, alpha=0.01)


@pytest.mark.parametrize("dist", ["balanced", "skewed", "ties", "signed_zero"])
def test_k1_equals_top1_router(dist):
    cfg = _cfg(2, 2, 2, 300, 0.75)
    lg = synth.supplied_logits(4, 300, 8, seed=3, dist=dist)
    a = oracle.route(cfg, lg)
    b = oracle.route_topk(cfg, 1, lg)
    np.testing.assert_array_equal(b.dest[0], a.dest1)
    np.testing.assert_array_equal(b.slot[0], a.slot1)
    np.testing.assert_array_equal(b.keep[0], a.keep)
    np.testing.assert_array_equal(b.w[0], a.gate)          # flat: gate = p (q = 1)
    np.testing.assert_array_equal(b.counts, a.counts1)
    np.testing.assert_array_equal(b.loss, a.loss)


@pytest.mark.parametrize("k", [2, 3])
@pytest.mark.parametrize("dist", ["balanced", "skewed", "ties"])
def test_choices_weights_and_capacity_brute_force(k, dist):
    G, e, T, cf = 4, 2, 60, 0.75
    cfg = _cfg(2, 2, e, T, cf)
    K = G * e
    lg = synth.supplied_logits(G, T, K, seed=5, dist=dist)
    r = oracle.route_topk(cfg, k, lg)
    # R29: stable descending order == repeated first argmax
    order = np.argsort(-lg, axis=-1, kind="stable")[:, :, :k]
    np.testing.assert_array_equal(np.moveaxis(r.dest, 0, -1), order)
    # R30: weights = full softmax entries (fp64 rounded to fp32)
    p = softmax(lg.astype(np.float64), axis=-1)
    np.testing.assert_allclose(np.moveaxis(r.w, 0, -1), np.take_along_axis(p, order, -1).astype(np.float32),
                               rtol=1e-6, atol=0)
    # R31: choice-major capacity, by definition over the item sequence
    C = int(np.ceil(cf * k * T / K))
    for g in range(G):
        seq = [(j, t) for j in range(k) for t in range(T)]
        for idx, (j, t) in enumerate(seq):
            e_ = r.dest[j, g, t]
            before = sum(1 for (jj, tt) in seq[:idx] if r.dest[jj, g, tt] == e_)
            assert r.slot[j, g, t] == before
            assert r.keep[j, g, t] == (before < C)
        for q in range(K):
            assert r.counts[g, q] == min(int((r.dest[:, g] == q).sum()), C)
    assert (r.keep == 0).any() and (r.keep == 1).any()


def test_worked_example_and_identity_expert():
    """Logits (ln 4, ln 2, 0, 0) over 4 experts: p = (1/2, 1/4, 1/8, 1/8); top-2 = experts 0, 1
    with weights 1/2, 1/4; with no drops the identity expert returns 3/4 x (Eq. 2)."""
    cfg = _cfg(1, 4, 1, 1, 8.0)
    lg = np.array([[[np.log(4.0), np.log(2.0), 0.0, 0.0]]], np.float32).repeat(4, 0)
    r = oracle.route_topk(cfg, 2, lg)
    assert (r.dest[:, 0, 0] == [0, 1]).all()
    np.testing.assert_allclose(r.w[:, 0, 0], [0.5, 0.25], rtol=1e-7)
    x = synth.tokens(4, 1, 8, seed=1)
    out = oracle.out_rows_topk(cfg, r, x, identity=True)
    np.testing.assert_allclose(out, 0.75 * x.reshape(4, 8).astype(np.float64), rtol=1e-7)


def test_identity_expert_drops_and_ties():
    """Identity expert: out = sum over kept choices of w_j x (dropped choices add nothing);
    a tie between the two largest logits takes the lower index first."""
    cfg = _cfg(2, 2, 1, 50, 0.5)
    lg = synth.supplied_logits(4, 50, 4, seed=9, dist="skewed")
    lg[0, 0] = [1.0, 3.0, 3.0, 0.0]
    r = oracle.route_topk(cfg, 2, lg)
    assert (r.dest[:, 0, 0] == [1, 2]).all()
    x = synth.tokens(4, 50, 16, seed=2)
    out = oracle.out_rows_topk(cfg, r, x, identity=True)
    ref = (r.keep * r.w).sum(0).reshape(-1, 1).astype(np.float64) * x.reshape(-1, 16).astype(np.float64)
    np.testing.assert_allclose(out, ref, rtol=1e-6)
    assert (r.keep == 0).any()


def test_ffn_output_is_sum_of_weighted_experts():
    """Eq. (2) with real experts: out = sum_j keep_j w_j E_{e_j}(x), each E the pinned
    oracle_ffn_row (tests/test_oracle_ffn_loss.py)."""
    cfg = _cfg(2, 1, 2, 30, 1.0)
    lg = synth.supplied_logits(2, 30, 4, seed=4, dist="balanced")
    r = oracle.route_topk(cfg, 2, lg)
    x = synth.tokens(2, 30, 8, seed=4)
    W1, b1, W2, b2 = synth.expert_weights(4, 8, 16, seed=4)
    out = oracle.out_rows_topk(cfg, r, x, W1, b1, W2, b2)
    for g in (0, 17, 31, 59):
        ref = np.zeros(8)
        for j in range(2):
            rr, t = divmod(g, 30)
            if r.keep[j, rr, t]:
                ex = r.dest[j, rr, t]
                ref += float(r.w[j, rr, t]) * oracle.ffn_row(x[rr, t], W1[ex], b1[ex], W2[ex], b2[ex])
        np.testing.assert_allclose(out[g], ref, rtol=1e-12, atol=1e-14)


def test_backward_topk_k1_equals_top1_backward():
    """k = 1: the top-k backward equals the FD-pinned top-1 flat backward (oracle_backward)."""
    cfg = _cfg(2, 2, 2, 40, 0.75)
    G, K, T, d, d_ff = 4, 8, 40, 8, 12
    x = synth.tokens(G, T, d, seed=7, dtype="bf16")
    W = synth.router_weights(K, d, seed=7)
    lg = oracle.logits(x.reshape(-1, d), W).reshape(G, T, K)
    W1, b1, W2, b2 = synth.expert_weights(K, d, d_ff, seed=7)
    gout = np.random.default_rng(3).normal(size=(G, T, d)).astype(np.float32)
    r1 = oracle.route(cfg, lg)
    rk = oracle.route_topk(cfg, 1, lg)
    a = oracle.backward(cfg, r1, x, W1, b1, W2, b2, gout, lam=2.0, W=W)
    b = oracle.backward_topk(cfg, rk, x, W1, b1, W2, b2, gout, lam=2.0, W=W)
    for key in ("dlogits", "dx", "dW", "dW1", "db1", "dW2", "db2"):
        np.testing.assert_allclose(b[key], a[key], rtol=1e-12, atol=1e-14, err_msg=key)


@pytest.mark.parametrize("k,cf", [(2, 8.0), (3, 0.6)])
def test_backward_topk_finite_differences(k, cf):
    """Central finite differences of the top-k objective (routing decisions held fixed) along
    random directions of every input: x, the router W, W1, b1, W2, b2."""
    cfg = _cfg(2, 1, 2, 5, cf)
    G, K, T, d, d_ff = 2, 4, 5, 4, 6
    rs = np.random.default_rng(11)
    x = rs.normal(size=(G, T, d)).astype(np.float32)
    W = (0.5 * rs.normal(size=(K, d))).astype(np.float32)
    W1 = (0.5 * rs.normal(size=(K, d, d_ff))).astype(np.float32)
    b1 = (0.1 * rs.normal(size=(K, d_ff))).astype(np.float32)
    W2 = (0.5 * rs.normal(size=(K, d_ff, d))).astype(np.float32)
    b2 = (0.1 * rs.normal(size=(K, d))).astype(np.float32)
    gout = rs.normal(size=(G, T, d)).astype(np.float32)
    lg = oracle.logits(x.reshape(-1, d), W).reshape(G, T, K)
    r = oracle.route_topk(cfg, k, lg)
    if cf < 1:
        assert (r.keep == 0).any()
    grad = oracle.backward_topk(cfg, r, x, W1, b1, W2, b2, gout, lam=3.0, W=W)
    base = dict(x=x, W=W, W1=W1, b1=b1, W2=W2, b2=b2)
    names = dict(x="dx", W="dW", W1="dW1", b1="db1", W2="dW2", b2="db2")
    eps = 1e-6
    for p, gk in names.items():
        u = rs.normal(size=base[p].shape)
        def J(sign):
            q = {kk: vv.astype(np.float64) for kk, vv in base.items()}
            q[p] = q[p] + sign * eps * u
            return oracle.objective_topk(cfg, r, q["x"], q["W1"], q["b1"], q["W2"], q["b2"], gout, lam=3.0, W=q["W"])
        fd = (J(1) - J(-1)) / (2 * eps)
        an = float((grad[gk] * u).sum())
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (p, fd, an)
