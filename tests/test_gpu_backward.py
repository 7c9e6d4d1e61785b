"""GPU parity of the backward pass (configuration C3) against the
pinned fp64 backward oracle (tests/test_oracle_backward.py): router dlogits, dx, the
router weight gradient and every expert weight / bias gradient, on seeded inputs with
drops at both levels.  Tolerances (atol = rtol * max|ref|): fp32 1e-4 (fp32 GEMMs and
softmax derivatives against fp64), bf16 3e-2 (bf16 dY / dZ / H / returned expert rows).
bf16 cases with d, d_ff multiples of 128 run the tcgen05 weight gradients (MN-major
operands, wgrad_tcgen05.cu); the others the SIMT ones."""
import numpy as np
import pytest
import torch

import oracle
from harness import Case, assert_close_scaled

pytestmark = pytest.mark.gpu


def run_bwd(case, lam=2.0, seed=0, peer=False):
    from paper_2212_05191_b200 import SmileLayer
    G, T, d, d_ff, e = case.G, case.T, case.d, case.d_ff, case.e
    layer = SmileLayer(case.n, case.m, e, d, d_ff, T, case.cf, case.dtype, case.mode, ffn_impl=case.ffn_impl)
    if peer:
        layer.enable_peer_exchange()
    g = case.gpu_tensors()
    tdt = g["x"].dtype
    rs = np.random.default_rng(100 + seed)
    gout_np = rs.normal(size=(G, T, d)).astype(np.float32)
    if case.dtype == "bf16":
        import synth
        gout_np = synth.round_bf16(gout_np)
    gout = torch.from_numpy(gout_np).cuda().to(tdt)
    W1 = torch.from_numpy(case.W1).cuda().to(tdt).contiguous()
    W2 = torch.from_numpy(case.W2).cuda().to(tdt).contiguous()
    out = torch.empty_like(g["x"])
    loss = torch.empty(G, dtype=torch.float64, device="cuda")
    layer.forward(g["x"], g["W1t"], g["b1"], g["W2t"], g["b2"], out, loss, logits=g["logits"], w_router=g["w_router"],
                  alpha=case.alpha, beta=case.beta, train=True)
    dx = torch.empty_like(g["x"])
    NE = G * e
    f32 = dict(dtype=torch.float32, device="cuda")
    dW1 = torch.empty(NE, d, d_ff, **f32); db1 = torch.empty(NE, d_ff, **f32)
    dW2 = torch.empty(NE, d_ff, d, **f32); db2 = torch.empty(NE, d, **f32)
    dWr = torch.empty(case.cfg.logit_width, d, **f32) if case.fused else None
    layer.backward(gout, dx, W1, W2, dW1, db1, dW2, db2, dW_router=dWr, lam=lam)
    torch.cuda.synchronize()
    assert layer.get_error() == 0
    lg = case.logits
    if case.fused:
        lg = layer.view()["logits"].cpu().numpy()      # route on the GPU's own logits (R3)
    r = oracle.route(case.cfg, lg)
    v = layer.view()
    np.testing.assert_array_equal(v["dest1"].cpu().numpy(), r.dest1)
    ref = oracle.backward(case.cfg, r, case.x, case.W1, case.b1, case.W2, case.b2, gout_np, lam=lam,
                          W=case.w_router if case.fused else None, logits=None if case.fused else case.logits)
    tol = 3e-2 if case.dtype == "bf16" else 1e-4
    got = dict(dlogits=v["dlogits"].cpu().numpy(), dx=dx.float().cpu().numpy(), dW1=dW1.cpu().numpy(),
               db1=db1.cpu().numpy(), dW2=dW2.cpu().numpy(), db2=db2.cpu().numpy())
    if case.fused:
        got["dW"] = dWr.cpu().numpy()
    for k, gv in got.items():
        # dlogits see the expert output only through dgate = <gout, back1>, back1 in the layer dtype
        assert_close_scaled(gv, ref[k], tol, f"backward {k}")
    return r


@pytest.mark.parametrize("n,m,e,T,d,d_ff,cf,dtype,mode,fused,ffn", [
    (2, 4, 1, 300, 64, 128, 1.0, "fp32", "bilevel", False, "simt"),
    (2, 2, 2, 257, 64, 64, 0.75, "fp32", "bilevel", True, "simt"),
    (4, 2, 1, 200, 64, 128, 1.25, "fp32", "flat", True, "simt"),
    (2, 4, 1, 600, 128, 256, 1.25, "bf16", "bilevel", True, "tcgen05"),   # C3-like 2x4, tcgen05 dgrad
    (4, 2, 1, 600, 128, 256, 1.25, "bf16", "bilevel", False, "tcgen05"),  # C3-like 4x2
    (2, 2, 2, 400, 64, 128, 1.0, "bf16", "flat", True, "tcgen05"),
    (2, 2, 2, 700, 128, 384, 1.0, "bf16", "flat", True, "tcgen05"),     # tcgen05 wgrad, e = 2, BN 128 / 192
    (2, 4, 1, 2000, 256, 512, 1.25, "bf16", "bilevel", False, "tcgen05"),  # wgrad over many K blocks
])
@pytest.mark.parametrize("cta_pair", [None, "1"])
def test_backward_parity(n, m, e, T, d, d_ff, cf, dtype, mode, fused, ffn, cta_pair, monkeypatch):
    """cta_pair None: the library's choice (these small capacities get 128-row tiles);
    "1": CTA-pair 256-row tiles forced (SMILE_FFN_CTA_PAIR, the path of C2-C4)."""
    if cta_pair is not None:
        if ffn != "tcgen05":
            pytest.skip("CTA pairs are a tcgen05 path")
        monkeypatch.setenv("SMILE_FFN_CTA_PAIR", cta_pair)
    case = Case(n, m, e, T, d, d_ff, cf, dtype=dtype, mode=mode, dist="skewed", seed=21, fused=fused, ffn_impl=ffn)
    r = run_bwd(case)
    assert (r.keep == 0).any()


@pytest.mark.parametrize("n,m,e,T,d,d_ff,cf,dtype,mode,fused,ffn", [
    (2, 4, 1, 600, 128, 256, 1.25, "bf16", "bilevel", True, "tcgen05"),
    (2, 2, 2, 700, 128, 384, 1.0, "bf16", "flat", True, "tcgen05"),
    (2, 2, 2, 257, 64, 64, 0.75, "fp32", "bilevel", True, "simt"),
])
def test_backward_parity_peer(n, m, e, T, d, d_ff, cf, dtype, mode, fused, ffn, monkeypatch):
    """The training step over the peer-store exchange (gradient rows stored at / loaded
    from their owners, every exchange a barrier): same oracle bar as the copy path."""
    monkeypatch.setenv("SMILE_FFN_CTA_PAIR", "1")
    case = Case(n, m, e, T, d, d_ff, cf, dtype=dtype, mode=mode, dist="skewed", seed=21, fused=fused, ffn_impl=ffn)
    r = run_bwd(case, peer=True)
    assert (r.keep == 0).any()
