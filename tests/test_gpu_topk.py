"""The FLAT top-k layer (Eq. (2); readings R29-R32) against
the pinned top-k oracle (tests/test_oracle_topk.py): every choice's expert, capacity slot
(choice-major, R31) and the per-expert counts bit-exactly on supplied fp32 logits; the
Eq. (2) output within the north-star tolerance; the fused tensor-core router (both gate
kernels) routes exactly like the oracle on the GPU's own logits."""
import numpy as np
import pytest
import torch

import oracle
import synth
from harness import assert_close_scaled

pytestmark = pytest.mark.gpu


def _run(n, m, e, T, d, d_ff, cf, k, dtype, peer, fused, seed, dist="skewed"):
    from paper_2212_05191_b200 import SmileLayer
    G = n * m
    K = G * e
    cfg = oracle.Config(n, m, e, T, cf, flat=True, alpha=0.01)
    x = synth.tokens(G, T, d, seed=seed, dtype=dtype)
    W1, b1, W2, b2 = synth.expert_weights(G * e, d, d_ff, seed=seed, dtype=dtype)
    layer = SmileLayer(n, m, e, d, d_ff, T, cf, dtype, "flat", topk=k)
    layer.alloc_workspace()
    layer.ws.fill_(0x7f)
    if peer:
        layer.enable_peer_exchange()
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    t = lambda a, dt=tdt: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dt)
    xg = t(x)
    out = torch.full_like(xg, float("nan"))
    loss = torch.empty(G, dtype=torch.float64, device="cuda")
    if fused:
        W = synth.router_weights(K, d, seed=seed)
        lg_gpu = torch.empty(G, T, K, dtype=torch.float32, device="cuda")
        w = layer._view

        class P:
            def __init__(s, a): s.a = a
            def data_ptr(s): return s.a
        layer.gate_inter(xg, w.route, w.stats, P(w.counts1), w_router=t(W, torch.float32), logits_out=lg_gpu)
        torch.cuda.synchronize()
        lg = lg_gpu.cpu().numpy()
        np.testing.assert_allclose(lg, oracle.logits(x.reshape(-1, d), W).reshape(G, T, K), rtol=0, atol=2e-5)
        layer.forward(xg, t(W1.transpose(0, 2, 1)), t(b1, torch.float32), t(W2.transpose(0, 2, 1)),
                      t(b2, torch.float32), out, loss, w_router=t(W, torch.float32), alpha=0.01, beta=0.0)
    else:
        lg = synth.supplied_logits(G, T, K, seed=seed, dist=dist)
        layer.forward(xg, t(W1.transpose(0, 2, 1)), t(b1, torch.float32), t(W2.transpose(0, 2, 1)),
                      t(b2, torch.float32), out, loss, logits=t(lg, torch.float32), alpha=0.01, beta=0.0)
    torch.cuda.synchronize()
    assert layer.get_error() == 0
    r = oracle.route_topk(cfg, k, lg)
    v = {kk: tt.cpu().numpy() for kk, tt in layer.view().items()}
    np.testing.assert_array_equal(v["dest1"], r.dest)
    np.testing.assert_array_equal(v["slot1"], r.slot)
    np.testing.assert_array_equal(v["counts1"], r.counts)
    np.testing.assert_array_equal(v["hist1"], r.A1)
    np.testing.assert_allclose(v["gate"], r.w, rtol=1e-6, atol=0)
    np.testing.assert_allclose(v["psum1"], r.S1, rtol=1e-6)
    np.testing.assert_allclose(loss.cpu().numpy(), r.loss, rtol=1e-6)
    ref = oracle.out_rows_topk(cfg, r, x, W1, b1, W2, b2)
    got = out.float().cpu().numpy().reshape(-1, d)
    assert_close_scaled(got, ref, 2e-2 if dtype == "bf16" else 1e-5, f"top-{k} output")
    alldrop = (r.keep.sum(0) == 0).reshape(-1)
    assert (got[alldrop] == 0).all()
    layer.close()
    return r


@pytest.mark.parametrize("k,dtype,peer", [(2, "bf16", False), (2, "bf16", True), (3, "fp32", False),
                                          (2, "fp32", True), (4, "bf16", True)])
def test_topk_supplied_logits(k, dtype, peer):
    r = _run(2, 2, 2, 500, 64, 128, 0.75, k, dtype, peer, False, 71)
    assert (r.keep == 0).any() and (r.keep[1:] == 1).any()


@pytest.mark.parametrize("n,m,e,d", [(2, 2, 2, 128), (2, 4, 8, 128)])   # KW 8 (swapped gate), 64 (128-token gate)
def test_topk_fused_router(n, m, e, d):
    _run(n, m, e, 600, d, 256, 1.0, 2, "bf16", True, True, 72, dist=None)


def test_topk_c2_widths():
    """C2's widths (d 768, d_ff 3072) at reduced T, the tcgen05 FFN, top-2 over 8 experts."""
    _run(2, 4, 1, 2048, 768, 3072, 1.25, 2, "bf16", True, False, 73, dist="balanced")


def test_topk_rejections():
    from paper_2212_05191_b200 import SmileLayer, SmileError
    with pytest.raises(SmileError):
        SmileLayer(2, 2, 1, 64, 128, 100, 1.0, "bf16", "bilevel", topk=2)    # bi-level is top-1 (Eq. 3)
    with pytest.raises(SmileError):
        SmileLayer(1, 2, 1, 64, 128, 100, 1.0, "bf16", "flat", topk=3)       # k > K


@pytest.mark.parametrize("k,dtype,peer,fused,ffn", [(2, "bf16", False, True, "tcgen05"), (2, "bf16", True, False, "tcgen05"),
                                                    (3, "fp32", False, True, "simt"), (2, "fp32", True, True, "simt")])
def test_topk_backward(k, dtype, peer, fused, ffn):
    """Training step of the FLAT top-k layer (forward with GELU' saved + smile_backward)
    against the pinned top-k backward oracle (tests/test_oracle_topk.py): dlogits, dx, the
    router gradient and every expert weight / bias gradient; tolerances as the top-1
    backward (bf16 3e-2, fp32 1e-4, atol = rtol * max|ref|)."""
    from paper_2212_05191_b200 import SmileLayer
    n, m, e, T, d, d_ff, cf = 2, 2, 2, 400, 128, 256, 0.75
    G, K = n * m, n * m * e
    cfg = oracle.Config(n, m, e, T, cf, flat=True, alpha=0.01)
    x = synth.tokens(G, T, d, seed=77, dtype=dtype)
    W1, b1, W2, b2 = synth.expert_weights(K, d, d_ff, seed=77, dtype=dtype)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    t = lambda a, dt=tdt: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dt)
    layer = SmileLayer(n, m, e, d, d_ff, T, cf, dtype, "flat", topk=k, ffn_impl=ffn)
    if peer:
        layer.enable_peer_exchange()
    W = synth.router_weights(K, d, seed=77) if fused else None
    lg_in = None if fused else synth.supplied_logits(G, T, K, seed=77, dist="skewed")
    # every input stays alive until the backward (it reads x, the router and the logits again)
    keep = dict(x=t(x), W1t=t(W1.transpose(0, 2, 1)), b1=t(b1, torch.float32), W2t=t(W2.transpose(0, 2, 1)),
                b2=t(b2, torch.float32), lg=None if fused else t(lg_in, torch.float32),
                W=t(W, torch.float32) if fused else None)
    out = torch.empty_like(keep["x"])
    loss = torch.empty(G, dtype=torch.float64, device="cuda")
    layer.forward(keep["x"], keep["W1t"], keep["b1"], keep["W2t"], keep["b2"], out, loss, logits=keep["lg"],
                  w_router=keep["W"], alpha=0.01, beta=0.0, train=True)
    rs = np.random.default_rng(5)
    gout_np = rs.normal(size=(G, T, d)).astype(np.float32)
    if dtype == "bf16":
        gout_np = synth.round_bf16(gout_np)
    f32 = dict(dtype=torch.float32, device="cuda")
    dx = torch.empty_like(out)
    dW1 = torch.empty(K, d, d_ff, **f32); db1 = torch.empty(K, d_ff, **f32)
    dW2 = torch.empty(K, d_ff, d, **f32); db2 = torch.empty(K, d, **f32)
    dWr = torch.empty(K, d, **f32) if fused else None
    layer.backward(t(gout_np), dx, t(W1), t(W2), dW1, db1, dW2, db2, dW_router=dWr, lam=2.0)
    torch.cuda.synchronize()
    assert layer.get_error() == 0
    lg = layer.view()["logits"].cpu().numpy() if fused else lg_in      # route on the GPU's logits (R3)
    r = oracle.route_topk(cfg, k, lg)
    np.testing.assert_array_equal(layer.view()["dest1"].cpu().numpy(), r.dest)
    assert (r.keep == 0).any()
    ref = oracle.backward_topk(cfg, r, x, W1, b1, W2, b2, gout_np, lam=2.0, W=W, logits=None if fused else lg_in)
    tol = 3e-2 if dtype == "bf16" else 1e-4
    got = dict(dlogits=layer.view()["dlogits"].cpu().numpy(), dx=dx.float().cpu().numpy(), dW1=dW1.cpu().numpy(),
               db1=db1.cpu().numpy(), dW2=dW2.cpu().numpy(), db2=db2.cpu().numpy())
    if fused:
        got["dW"] = dWr.cpu().numpy()
    for key, gv in got.items():
        assert_close_scaled(gv, ref[key], tol, f"top-{k} backward {key}")
    assert_close_scaled(out.float().cpu().numpy().reshape(-1, d), oracle.out_rows_topk(cfg, r, x, W1, b1, W2, b2),
                        2e-2 if dtype == "bf16" else 1e-5, "top-k training forward output")
    layer.close()
