"""Pins for the oracle's routing (oracle_route / oracle_capacity): closed forms from the
paper and SPEC, brute-force definitions on tiny inputs, exhaustive enumeration,
invariants, and the n=1 / K2=1 collapse to flat Switch routing.

None of these checks call the oracle to produce an expected value: expected values come
from the paper's printed examples, from O(T^2) brute-force definitions written here with
numpy's argmax (first maximal index), or from scipy's softmax.
"""
import itertools
import math

import numpy as np
import pytest
from scipy.special import softmax

import oracle
import synth


def one_hot_logits(cfg, assign, gap=1.0):
    """Logits realising an assignment [(i, j)] per (rank, token); gap sets the margin."""
    K1, K2, _, _ = cfg.sizes()
    lg = np.zeros((cfg.G, cfg.T, cfg.logit_width), np.float32)
    for r in range(cfg.G):
        for t in range(cfg.T):
            i, j = assign[r][t]
            lg[r, t, i] = gap
            if not cfg.flat:
                lg[r, t, K1 + j] = gap
    return lg


def brute_force(cfg, lg):
    """Independent O(T^2) definition of both routing levels (readings R2, R5-R8,
    R10).  Returns dicts of expected arrays."""
    G, T, n, m = cfg.G, cfg.T, cfg.n, cfg.m
    K1 = cfg.n if not cfg.flat else cfg.G * cfg.e
    K2 = cfg.m * cfg.e if not cfg.flat else 1
    C1 = T if K1 == 1 else math.ceil(cfg.cf * T / K1)
    C2 = (n * C1 if K2 == 1 else math.ceil(cfg.cf * T / K2))
    i = np.argmax(lg[:, :, :K1], axis=-1)
    j = np.zeros_like(i) if cfg.flat else np.argmax(lg[:, :, K1:], axis=-1)
    slot1 = np.array([[np.sum(i[r, :t] == i[r, t]) for t in range(T)] for r in range(G)], dtype=np.int64)
    keep1 = slot1 < C1
    keep = keep1.copy()
    jin = np.full((G, max(n * C1, 1)), -1)
    slot2 = np.full_like(jin, -1)
    keep2 = np.zeros_like(jin, dtype=bool)
    if not cfg.flat:
        for u in range(G):
            ii, l = divmod(u, m)
            recv = []  # (s, c, r, t, j) in received order
            for s in range(n):
                r = s * m + l
                toks = [t for t in range(T) if i[r, t] == ii and keep1[r, t]]
                for c, t in enumerate(toks):
                    recv.append((s, c, r, t, j[r, t]))
            for a, (s, c, r, t, jj) in enumerate(recv):
                x = s * C1 + c
                jin[u, x] = jj
                slot2[u, x] = sum(1 for b in recv[:a] if b[4] == jj)
                keep2[u, x] = slot2[u, x] < C2
                keep[r, t] = keep2[u, x]
    return dict(dest1=i, dest2=j, slot1=slot1, keep1=keep1, keep=keep, jin=jin, slot2=slot2,
                keep2=keep2, C1=C1, C2=C2)


def check_against_brute(cfg, lg):
    r = oracle.route(cfg, lg)
    b = brute_force(cfg, lg)
    assert (r.C1, r.C2 if not cfg.flat else b["C2"]) == (b["C1"], b["C2"])
    np.testing.assert_array_equal(r.dest1, b["dest1"])
    np.testing.assert_array_equal(r.dest2, b["dest2"])
    np.testing.assert_array_equal(r.slot1, b["slot1"])
    np.testing.assert_array_equal(r.keep1.astype(bool), b["keep1"])
    np.testing.assert_array_equal(r.keep.astype(bool), b["keep"])
    if not cfg.flat:
        np.testing.assert_array_equal(r.jin, b["jin"])
        np.testing.assert_array_equal(r.slot2, b["slot2"])
        np.testing.assert_array_equal(r.keep2.astype(bool), b["keep2"])
    return r


# ---- capacity (SPEC dispatch examples S:L281-283; R5, R20) -------------------------

def test_capacity_spec_examples():
    assert oracle.capacity(8, 4, 2.0) == 4
    assert oracle.capacity(0, 4, 2.0) == 0
    assert oracle.capacity(7, 2, 1.0) == 4      # S:L283 (ceiling)
    assert oracle.capacity(16384, 2, 2.0) == 16384
    assert oracle.capacity(16384, 4, 2.0) == 8192
    assert oracle.capacity(32768, 8, 1.25) == 5120
    assert oracle.capacity(5, 1, 0.5) == 5      # single destination: no capacity (R20)


def test_sizes_configs():
    # C2: 2x4, e=1, T=16K, cf 2 -> C1 = 16384, C2 = 8192, flat C = 4096
    assert oracle.Config(2, 4, 1, 16384, 2.0).sizes() == (2, 4, 16384, 8192)
    assert oracle.Config(2, 4, 1, 16384, 2.0, flat=True).sizes()[:3] == (8, 1, 4096)
    # C4: 2x4, e=8 -> K2 = 32, C2 = 4096; flat K = 64, C = 2048
    assert oracle.Config(2, 4, 8, 65536, 2.0).sizes() == (2, 32, 65536, 4096)
    assert oracle.Config(2, 4, 8, 65536, 2.0, flat=True).sizes()[:3] == (64, 1, 2048)


# ---- probabilities: closed forms, shift invariance ----

def test_softmax_ln2_closed_form():
    cfg = oracle.Config(1, 1, 4, T=1, flat=True, alpha=0.01)
    lg = np.array([[[np.log(2.0), 0, 0, 0]]], np.float32)
    r = oracle.route(cfg, lg)
    assert r.dest1[0, 0] == 0
    assert abs(r.p[0, 0] - 0.4) < 1e-7
    np.testing.assert_allclose(r.S1[0], [0.4, 0.2, 0.2, 0.2], rtol=0, atol=1e-7)


def test_bilevel_gate_054():
    cfg = oracle.Config(2, 2, 1, T=1)
    lg = np.zeros((4, 1, 4), np.float32)
    lg[:, 0] = np.log([0.9, 0.1, 0.6, 0.4]).astype(np.float32)
    r = oracle.route(cfg, lg)
    assert (r.dest1 == 0).all() and (r.dest2 == 0).all()
    np.testing.assert_allclose(r.p, 0.9, atol=1e-7)
    np.testing.assert_allclose(r.q, 0.6, atol=1e-7)
    np.testing.assert_allclose(r.gate, 0.54, atol=1e-7)


@pytest.mark.parametrize("n,m,e", [(2, 4, 1), (4, 2, 1), (3, 2, 2)])
def test_equal_rows_tie_to_expert00(n, m, e):
    cfg = oracle.Config(n, m, e, T=5)
    lg = np.full((cfg.G, 5, cfg.logit_width), 0.25, np.float32)
    r = oracle.route(cfg, lg)
    assert (r.dest1 == 0).all() and (r.dest2 == 0).all()
    np.testing.assert_allclose(r.gate, 1.0 / (n * m * e), rtol=1e-7)


def test_signed_zero_is_a_tie():
    cfg = oracle.Config(1, 1, 3, T=1, flat=True)
    r = oracle.route(cfg, np.array([[[-0.0, 0.0, -1.0]]], np.float32))
    assert r.dest1[0, 0] == 0          # R28: -0.0 == +0.0 under '>', lowest index wins


def test_shift_invariance_and_scipy_softmax():
    cfg = oracle.Config(2, 4, 2, T=64)
    lg = synth.supplied_logits(cfg.G, cfg.T, cfg.logit_width, seed=3)
    lg = np.round(lg * 1024) / np.float32(1024)     # multiples of 2^-10: the shift is exact
    r0 = oracle.route(cfg, lg)
    r1 = oracle.route(cfg, lg + np.float32(8.0))
    np.testing.assert_array_equal(r0.dest1, r1.dest1)
    np.testing.assert_array_equal(r0.p, r1.p)
    np.testing.assert_array_equal(r0.gate, r1.gate)
    K1 = cfg.n
    sm1 = softmax(lg[:, :, :K1].astype(np.float64), axis=-1)
    sm2 = softmax(lg[:, :, K1:].astype(np.float64), axis=-1)
    np.testing.assert_allclose(r0.S1, sm1.sum(1), rtol=1e-12)
    np.testing.assert_allclose(r0.S2, sm2.sum(1), rtol=1e-12)
    np.testing.assert_allclose(r0.p, sm1.max(-1), rtol=1e-7)
    np.testing.assert_allclose(r0.q, sm2.max(-1), rtol=1e-7)
    np.testing.assert_allclose(r0.gate, sm1.max(-1) * sm2.max(-1), rtol=3e-7)


def test_nonfinite_logits_rejected():
    cfg = oracle.Config(1, 2, 1, T=2)
    lg = np.zeros((2, 2, 3), np.float32)
    lg[1, 1, 2] = np.nan
    with pytest.raises(ValueError):
        oracle.route(cfg, lg)


# ---- slots, keep masks: brute force and exhaustive enumeration ---------------------

@pytest.mark.parametrize("dist", ["balanced", "skewed", "ties"])
@pytest.mark.parametrize("n,m,e,cf", [(2, 4, 1, 1.0), (4, 2, 1, 1.25), (2, 2, 2, 0.5), (3, 1, 2, 1.0)])
def test_brute_force_random(dist, n, m, e, cf):
    for seed in range(3):
        cfg = oracle.Config(n, m, e, T=24, cf=cf)
        lg = synth.supplied_logits(cfg.G, cfg.T, cfg.logit_width, seed=seed, dist=dist, K1=n)
        check_against_brute(cfg, lg)
        fcfg = oracle.Config(n, m, e, T=24, cf=cf, flat=True)
        flg = synth.supplied_logits(cfg.G, cfg.T, fcfg.logit_width, seed=seed, dist=dist)
        check_against_brute(fcfg, flg)


def test_exhaustive_tiny():
    """Every assignment of (i, j) to every token, for n, m, e in {1, 2}, T <= 2 per rank
    (sampled when the space exceeds 4096), at cf in {0.5, 1, 2}."""
    rs = np.random.default_rng(0)
    for n, m, e, T in itertools.product((1, 2), (1, 2), (1, 2), (1, 2)):
        G = n * m
        choices = [(i, j) for i in range(n) for j in range(m * e)]
        space = len(choices) ** (G * T)
        if space <= 4096:
            assigns = itertools.product(choices, repeat=G * T)
        else:
            assigns = (tuple(choices[k] for k in rs.integers(0, len(choices), G * T)) for _ in range(300))
        for flat_assign in assigns:
            A = [list(flat_assign[r * T:(r + 1) * T]) for r in range(G)]
            for cf in (0.5, 1.0, 2.0):
                cfg = oracle.Config(n, m, e, T=T, cf=cf)
                check_against_brute(cfg, one_hot_logits(cfg, A))


def test_spec_plan_example_all_to_node0():
    # n=2, m=1, T=8, all tokens to node 0, cf=1.0 -> capacity 4, 4 drops
    cfg = oracle.Config(2, 1, 1, T=8, cf=1.0)
    A = [[(0, 0)] * 8, [(0, 0)] * 8]
    r = oracle.route(cfg, one_hot_logits(cfg, A))
    assert r.C1 == 4
    assert (r.keep1 == 0).sum(axis=1).tolist() == [4, 4]
    assert r.counts1.tolist() == [[4, 0], [4, 0]]


# ---- invariants: conservation, capacity bound, monotone drops ----------

@pytest.mark.parametrize("flat", [False, True])
def test_invariants(flat):
    cfg0 = oracle.Config(2, 4, 2, T=200, flat=flat)
    lg = synth.supplied_logits(cfg0.G, cfg0.T, cfg0.logit_width, seed=7, dist="skewed", K1=cfg0.n)
    prev = None
    for cf in (0.25, 0.5, 1.0, 1.25, 2.0, 4.0, 8.0):
        cfg = oracle.Config(2, 4, 2, T=200, cf=cf, flat=flat)
        r = oracle.route(cfg, lg)
        # conservation at level 1: kept + dropped = T, kept per dest = counts1 <= C1
        assert (r.counts1.sum(1) == r.keep1.sum(1)).all()
        assert (r.counts1 <= r.C1).all()
        assert (r.A1.sum(1) == cfg.T).all() and (r.A2.sum(1) == cfg.T).all()
        if not flat:
            valid = r.jin >= 0
            assert (r.counts2.sum(1) == (r.keep2.astype(bool) & valid).sum(1)).all()
            assert (r.counts2 <= r.C2).all()
            # every token that arrived is received exactly once
            assert valid.sum() == r.keep1.sum()
        drops = int((r.keep == 0).sum())
        if prev is not None:
            assert drops <= prev                        # monotone in cf
        prev = drops
    assert prev == 0                                    # cf = 8 drops nothing here


def test_received_count_matches_sent():
    cfg = oracle.Config(2, 4, 1, T=100, cf=1.0)
    lg = synth.supplied_logits(cfg.G, cfg.T, cfg.logit_width, seed=1, dist="skewed", K1=2)
    r = oracle.route(cfg, lg)
    for u in range(cfg.G):
        i, l = divmod(u, cfg.m)
        for s in range(cfg.n):
            sent = r.counts1[s * cfg.m + l, i]
            got = (r.jin[u, s * r.C1:(s + 1) * r.C1] >= 0).sum()
            assert sent == got
            assert (r.jin[u, s * r.C1:s * r.C1 + sent] >= 0).all()   # packed prefix


# ---- collapse to flat Switch (R20; SURVEY §8(c) "collapse") -------------------------

@pytest.mark.parametrize("m,e,cf", [(4, 1, 1.0), (2, 2, 0.5), (8, 1, 2.0)])
def test_collapse_n1(m, e, cf):
    T = 50
    bi = oracle.Config(1, m, e, T=T, cf=cf, alpha=0.005, beta=0.005)
    fl = oracle.Config(1, m, e, T=T, cf=cf, flat=True, alpha=0.005)
    lq = synth.supplied_logits(m, T, m * e, seed=5, dist="skewed")
    lp = synth.supplied_logits(m, T, 1, seed=6)
    rb = oracle.route(bi, np.concatenate([lp, lq], axis=-1))
    rf = oracle.route(fl, lq)
    np.testing.assert_array_equal(rb.dest2, rf.dest1)
    np.testing.assert_array_equal(rb.keep, rf.keep)
    np.testing.assert_array_equal(rb.gate, rf.gate)         # bit-exact: p = 1
    for u in range(m):                                        # slot2 at u equals flat slot
        valid = rb.jin[u] >= 0
        np.testing.assert_array_equal(rb.slot2[u][valid], rf.slot1[u])
    np.testing.assert_allclose(rb.loss, 0.005 + rf.loss, rtol=1e-15)


@pytest.mark.parametrize("n,cf", [(2, 1.0), (4, 1.25), (8, 0.5)])
def test_collapse_k2_1(n, cf):
    T = 50
    bi = oracle.Config(n, 1, 1, T=T, cf=cf, alpha=0.005, beta=0.005)
    fl = oracle.Config(n, 1, 1, T=T, cf=cf, flat=True, alpha=0.005)
    lp = synth.supplied_logits(n, T, n, seed=8, dist="skewed")
    lq = synth.supplied_logits(n, T, 1, seed=9)
    rb = oracle.route(bi, np.concatenate([lp, lq], axis=-1))
    rf = oracle.route(fl, lp)
    for k in ("dest1", "slot1", "keep1", "keep", "gate"):
        np.testing.assert_array_equal(getattr(rb, k), getattr(rf, k))
    assert (rb.keep2[rb.jin >= 0] == 1).all()
    np.testing.assert_allclose(rb.loss, rf.loss + 0.005, rtol=1e-15)
