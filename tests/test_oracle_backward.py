"""Pins for the backward oracle (oracle_backward): central finite
differences of the fp64 objective J = sum <gout, OUT> + lam * sum loss (oracle_objective),
which is itself pinned to the forward oracle; and the corrected W_p = 0 closed form
(SURVEY §0 finding 4: the LB gradient there is (alpha/T)(f - 1/n) sum x, not zero)."""
import numpy as np
import pytest

import oracle
import synth


def q12(a):
    """Round to multiples of 2^-12 so the values are exact in fp32 and fp64."""
    return np.round(np.asarray(a, np.float64) * 4096.0) / 4096.0


def setup(n, m, e, T, d, d_ff, cf, flat, seed, fused=True):
    cfg = oracle.Config(n, m, e, T, cf, flat=flat, alpha=0.01 if flat else 0.005, beta=0.005)
    G = n * m
    rs = np.random.default_rng(seed)
    x = q12(rs.normal(size=(G, T, d)))
    W = q12(rs.uniform(-1, 1, size=(cfg.logit_width, d)))
    W1 = q12(rs.uniform(-0.4, 0.4, size=(G * e, d, d_ff)))
    b1 = q12(rs.uniform(-0.1, 0.1, size=(G * e, d_ff)))
    W2 = q12(rs.uniform(-0.3, 0.3, size=(G * e, d_ff, d)))
    b2 = q12(rs.uniform(-0.1, 0.1, size=(G * e, d)))
    gout = q12(rs.normal(size=(G, T, d)))
    return cfg, x, W, W1, b1, W2, b2, gout


def test_objective_matches_forward_oracle():
    cfg, x, W, W1, b1, W2, b2, gout = setup(2, 2, 1, 7, 6, 10, 1.0, False, 0)
    J, keep, _ = oracle.objective(cfg, x, W1, b1, W2, b2, gout, lam=1.0, W=W)
    lg = oracle.logits(x.reshape(-1, 6), W).reshape(cfg.G, cfg.T, -1)
    r = oracle.route(cfg, lg)
    out = oracle.out_rows(cfg, r, x, W1, b1, W2, b2).reshape(cfg.G, cfg.T, 6)
    ref = float((out * gout).sum() + r.loss.sum())
    np.testing.assert_array_equal(keep, r.keep.reshape(-1))
    assert abs(J - ref) <= 1e-6 * max(1.0, abs(ref))      # gate rounded to fp32 in out_rows


@pytest.mark.parametrize("flat", [False, True])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_backward_finite_differences(flat, seed):
    n, m, e, T, d, d_ff = 2, 2, 1, 6, 5, 7
    cfg, x, W, W1, b1, W2, b2, gout = setup(n, m, e, T, d, d_ff, 0.75, flat, seed)
    lg = oracle.logits(x.reshape(-1, d), W).reshape(cfg.G, T, -1)
    r = oracle.route(cfg, lg)
    assert (r.keep == 0).any() and (r.keep == 1).any()
    lam = 3.0                      # make the LB term visible next to the data term
    gr = oracle.backward(cfg, r, x, W1, b1, W2, b2, gout, lam=lam, W=W)
    _, keep0, dest0 = oracle.objective(cfg, x, W1, b1, W2, b2, gout, lam=lam, W=W)
    h = 1e-5
    rs = np.random.default_rng(100 + seed)
    for name, arr, grad in (("x", x, gr["dx"]), ("W", W, gr["dW"]), ("W1", W1, gr["dW1"]), ("b1", b1, gr["db1"]),
                            ("W2", W2, gr["dW2"]), ("b2", b2, gr["db2"])):
        for _ in range(12):
            idx = tuple(rs.integers(0, s) for s in arr.shape)
            args = dict(x=x, W=W, W1=W1, b1=b1, W2=W2, b2=b2)
            vals = []
            for sgn in (+1, -1):
                a2 = arr.copy()
                a2[idx] += sgn * h
                args[name] = a2
                J, keep, dest = oracle.objective(cfg, args["x"], args["W1"], args["b1"], args["W2"], args["b2"], gout,
                                                 lam=lam, W=args["W"])
                assert (keep == keep0).all() and (dest == dest0).all(), "perturbation flipped a decision"
                vals.append(J)
            fd = (vals[0] - vals[1]) / (2 * h)
            an = grad[idx]
            assert abs(fd - an) <= 1e-6 + 1e-5 * abs(fd), (name, idx, fd, an)


def test_backward_supplied_logits_gradient():
    """dlogits against finite differences of the objective in the logits themselves."""
    n, m, e, T, d, d_ff = 2, 2, 2, 5, 4, 6
    cfg, x, W, W1, b1, W2, b2, gout = setup(n, m, e, T, d, d_ff, 1.0, False, 7)
    lg = q12(synth.supplied_logits(cfg.G, T, cfg.logit_width, seed=7))
    r = oracle.route(cfg, lg.astype(np.float32))
    gr = oracle.backward(cfg, r, x, W1, b1, W2, b2, gout, lam=2.0, logits=lg)
    assert gr["dW"] is None
    h = 1e-5
    for idx in [(0, 0, 0), (1, 2, 3), (3, 4, 5), (2, 1, 1), (3, 0, 2)]:
        vals = []
        for sgn in (+1, -1):
            l2 = lg.copy()
            l2[idx] += sgn * h
            vals.append(oracle.objective(cfg, x, W1, b1, W2, b2, gout, lam=2.0, logits=l2)[0])
        fd = (vals[0] - vals[1]) / (2 * h)
        assert abs(fd - gr["dlogits"][idx]) <= 1e-6 + 1e-5 * abs(fd), (idx, fd, gr["dlogits"][idx])


def test_lb_gradient_at_wp_zero_closed_form():
    """W_p = 0: every token ties, goes to node 0 (R2), p is uniform, so the inter LB
    gradient is dW_p[k] = (alpha/T)(f_k - 1/n) sum_t x_t with f = (1, 0, ..., 0) -- NOT the
    zero matrix S:L231 claims (SURVEY §0 finding 4)."""
    n, m, T, d = 4, 1, 9, 3
    cfg = oracle.Config(n, m, 1, T, 8.0, alpha=0.005, beta=0.0)
    rs = np.random.default_rng(3)
    x = q12(rs.normal(size=(n * m, T, d)))
    W = np.zeros((n + 1, d))
    W1 = np.zeros((n, d, 4)); b1 = np.zeros((n, 4)); W2 = np.zeros((n, 4, d)); b2 = np.zeros((n, d))
    gout = np.zeros((n, T, d))
    lg = oracle.logits(x.reshape(-1, d), W).reshape(n, T, -1)
    r = oracle.route(cfg, lg)
    assert (r.dest1 == 0).all()
    gr = oracle.backward(cfg, r, x, W1, b1, W2, b2, gout, lam=1.0, W=W)
    f = np.zeros(n); f[0] = 1.0
    ref = np.zeros((n, d))
    for rk in range(n):                      # tied router: the gradient sums over ranks
        ref += (0.005 / T) * np.outer(f - 1.0 / n, x[rk].sum(0))
    np.testing.assert_allclose(gr["dW"][:n], ref, rtol=1e-12, atol=1e-15)
    assert np.abs(gr["dW"][:n]).max() > 0
