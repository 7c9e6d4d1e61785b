"""The cited worked examples of tests/golden/ against the oracle (-m "not gpu")."""
import json
import math
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "worked_examples.json")))


@pytest.mark.parametrize("c", CASES, ids=[c["id"] for c in CASES])
def test_golden(c):
    k = c["kind"]
    if k == "capacity":
        assert oracle.capacity(*c["args"]) == c["expect"]
    elif k == "softmax_row":
        # one token, n = 4 inter destinations, no level 2 (K2 = 1 is the identity, R20)
        cfg = oracle.Config(4, 1, 1, T=1)
        lg = np.zeros((4, 1, cfg.logit_width), np.float32)
        lg[:, 0, :4] = np.array(c["logits"], np.float32)
        r = oracle.route(cfg, lg)
        assert r.dest1[0, 0] == 0
        np.testing.assert_allclose(r.p[0, 0], c["expect"][0], rtol=1e-6)
    elif k == "bilevel_gate":
        cfg = oracle.Config(c["n"], c["m"], 1, T=1)
        lg = np.zeros((cfg.G, 1, cfg.logit_width), np.float32)
        lg[:, 0, :c["n"]] = np.log(np.array(c["p"], np.float64)).astype(np.float32)
        lg[:, 0, c["n"]:] = np.log(np.array(c["q"], np.float64)).astype(np.float32)
        r = oracle.route(cfg, lg)
        assert r.dest1[0, 0] == c["expect_i"] and r.dest2[0, 0] == c["expect_j"]
        np.testing.assert_allclose(r.gate[0, 0], c["expect_gate"], rtol=1e-6)
    elif k == "bilevel_gate_equal":
        cfg = oracle.Config(c["n"], c["m"], 1, T=3)
        r = oracle.route(cfg, np.zeros((cfg.G, 3, cfg.logit_width), np.float32))
        assert (r.dest1 == c["expect_i"]).all() and (r.dest2 == c["expect_j"]).all()
        np.testing.assert_allclose(r.gate, c["expect_gate"], rtol=1e-6)
    elif k == "lb_uniform":
        cfg = oracle.Config(c["n"], c["m"], 1, T=16, alpha=c["alpha"], beta=c["beta"])
        r = oracle.route(cfg, np.zeros((cfg.G, 16, cfg.logit_width), np.float32))
        np.testing.assert_allclose(r.loss, c["expect"], rtol=1e-15)
    elif k == "lb_all_to_node0":
        cfg = oracle.Config(c["n"], 1, 1, T=6, alpha=c["alpha"], beta=0.0)
        lg = np.zeros((cfg.G, 6, cfg.logit_width), np.float32)
        lg[:, :, 0] = 40.0                           # one-hot P at node 0
        r = oracle.route(cfg, lg)
        np.testing.assert_allclose(r.loss, c["expect"], rtol=1e-12)
    elif k == "drops_all_to_node0":
        cfg = oracle.Config(c["n"], c["m"], 1, T=c["T"], cf=c["cf"])
        assert oracle.capacity(c["T"], c["n"], c["cf"]) == c["expect_capacity"]
        lg = np.zeros((cfg.G, c["T"], cfg.logit_width), np.float32)
        lg[:, :, 0] = 1.0
        r = oracle.route(cfg, lg)
        keep = r.keep.reshape(cfg.G, c["T"]).astype(bool)
        assert (~keep[0]).sum() == c["expect_drops"]
        assert keep[0, :c["expect_capacity"]].all() and not keep[0, c["expect_capacity"]:].any()
    elif k == "ffn_row":
        f32 = lambda v: np.array(v, np.float32)
        y = oracle.ffn_row(f32(c["x"]), f32(c["W1"]), f32(c["b1"]), f32(c["W2"]), f32(c["b2"]))
        np.testing.assert_allclose(y, c["expect"], rtol=0, atol=1e-14)
        # the hand evaluation itself, with math.erf (not the oracle's code)
        g = lambda a: 0.5 * a * (1 + math.erf(a / math.sqrt(2)))
        assert abs(c["expect"][0] - (g(1) + g(2) + 0.5)) < 1e-15 and abs(c["expect"][1] + g(2)) < 1e-15
    else:
        raise AssertionError(f"unknown kind {k}")
