"""Full-size parity at EVERY configuration bench.py times (VERDICT r01 "Next round" 1):
C2 (2x4, e = 1, T = 16K), C4 (2x4, e = 8, T = 64K, H workspace > 2^31 bytes), C5 (2x4,
e = 16, d = 1600, d_ff = 6400, T = 8K), bi-level and flat, and the C3 training step (2x4 and
4x2, T = 32K, fwd + bwd), each in the launch configuration the bench uses: fused
tensor-core router (w_router), peer-store exchange, tcgen05 FFN, the layer output bound
(GEMM 2 -> out fusion) for inference.

Routing is compared in FULL and bit-exactly (dest1, dest2, slot1, counts, histograms,
the level-2 received metadata / slots / counts) against the oracle run on the GPU's own
fp32 logits, which must themselves be within fp32 accumulation error (2e-5) of the
oracle's fp64 logits (R3).  Outputs are compared on dense samples (harness.dense_rows:
one row of every 32-row FFN strip of every expert segment, every segment's first and last
row, every dropped token), evaluated by the OpenMP oracle (bit-identical to the serial
one, tests/test_oracle_parallel.py).  Tolerances: bf16 outputs rtol 2e-2, gradients 3e-2
(atol = rtol * max|ref|), loss 1e-6 (north star)."""
import numpy as np
import pytest
import torch

import oracle
from harness import Case, assert_close_scaled, dense_rows

pytestmark = pytest.mark.gpu


class Addr:
    def __init__(self, a):
        self.a = a

    def data_ptr(self):
        return self.a


def _gpu_logits(layer, g, case):
    """The fused router's fp32 logits from the gate kernel (run before the forward on the
    same context -- the forward recomputes them identically, the kernel is deterministic)."""
    lg = torch.empty(case.G, case.T, case.cfg.logit_width, dtype=torch.float32, device="cuda")
    w = layer._view
    layer.gate_inter(g["x"], w.route, w.stats, Addr(w.counts1), w_router=g["w_router"], logits_out=lg)
    torch.cuda.synchronize()
    return lg.cpu().numpy()


def _check_logits(case, lg):
    ref = oracle.logits(case.x.reshape(-1, case.d), case.w_router, threads=True).reshape(lg.shape)
    np.testing.assert_allclose(lg, ref, rtol=0, atol=2e-5)


def _check_route_full(case, layer, r, loss):
    v = {k: t.cpu().numpy() for k, t in layer.view().items()}
    for k, ref in (("dest1", r.dest1), ("slot1", r.slot1), ("counts1", r.counts1), ("hist1", r.A1)):
        np.testing.assert_array_equal(v[k], ref, err_msg=k)
    np.testing.assert_allclose(v["gate"], r.gate, rtol=1e-6, atol=0)
    np.testing.assert_allclose(loss.cpu().numpy(), r.loss, rtol=1e-6)
    if not case.flat:
        np.testing.assert_array_equal(v["dest2"], r.dest2)
        np.testing.assert_array_equal(v["hist2"], r.A2)
        np.testing.assert_array_equal(v["rmeta1"], r.jin)
        valid = r.jin >= 0
        np.testing.assert_array_equal(v["slot2"][valid], r.slot2[valid])
        np.testing.assert_array_equal(v["counts2"], r.counts2)


def _layer(case):
    from paper_2212_05191_b200 import SmileLayer
    L = SmileLayer(case.n, case.m, case.e, case.d, case.d_ff, case.T, case.cf, "bf16", case.mode)
    L.enable_peer_exchange()
    return L


def _forward_check(case):
    layer = _layer(case)
    g = case.gpu_tensors()
    lg = _gpu_logits(layer, g, case)
    _check_logits(case, lg)
    out = torch.full_like(g["x"], float("nan"))               # every row must be written
    loss = torch.empty(layer.V, dtype=torch.float64, device="cuda")
    layer.forward(g["x"], g["W1t"], g["b1"], g["W2t"], g["b2"], out, loss, w_router=g["w_router"],
                  alpha=case.alpha, beta=case.beta)
    torch.cuda.synchronize()
    assert layer.get_error() == 0
    r = case.oracle_route(logits=lg)
    _check_route_full(case, layer, r, loss)
    rows = dense_rows(case, r)
    got = out.view(-1, case.d)[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    ref = oracle.out_rows(case.cfg, r, case.x, case.W1, case.b1, case.W2, case.b2, rows=rows, threads=True)
    assert_close_scaled(got, ref, 2e-2, f"full-size {case.mode} output ({rows.size} rows)")
    keep = r.keep.reshape(-1).astype(bool)[rows]
    assert (got[~keep] == 0).all()
    assert not torch.isnan(out.float()).any()
    layer.close()
    return r, rows


BENCH = {
    "c2": dict(n=2, m=4, e=1, T=16384, d=768, d_ff=3072, cf=2.0),
    "c4": dict(n=2, m=4, e=8, T=65536, d=1024, d_ff=4096, cf=2.0),
    "c5": dict(n=2, m=4, e=16, T=8192, d=1600, d_ff=6400, cf=2.0),
}


@pytest.mark.parametrize("mode", ["bilevel", "flat"])
@pytest.mark.parametrize("cfg", ["c2", "c4", "c5"])
def test_bench_config_full_size(cfg, mode):
    c = BENCH[cfg]
    case = Case(c["n"], c["m"], c["e"], c["T"], c["d"], c["d_ff"], c["cf"], dtype="bf16", mode=mode, fused=True,
                seed=4, bias=False)
    r, rows = _forward_check(case)
    assert rows.size > case.G * case.T // 40


@pytest.mark.parametrize("n,m", [(2, 4), (4, 2)])
def test_c3_training_full_size(n, m):
    """C3 as bench.py --config c3 / c3_4x2 times it: fused router, peer exchange, tcgen05
    forward (GELU' saved) + smile_backward.  Gradients vs oracle_backward_sampled: dlogits and
    dx of ~600 tokens (incl. dropped ones), dW1 columns / db1 entries / dW2 rows at 8
    intermediate columns of every expert, all of db2; the tied-router gradient is checked
    as the property dW = sum_t dlogits[t]^T x[t] (fp64 on the host) over the GPU's
    dlogits, which are themselves pinned on the sampled tokens."""
    from paper_2212_05191_b200 import SmileLayer
    T, d, d_ff, cf, e = 32768, 768, 3072, 1.25, 1
    case = Case(n, m, e, T, d, d_ff, cf, dtype="bf16", fused=True, seed=6)
    layer = _layer(case)
    g = case.gpu_tensors()
    G, NE = case.G, case.G * e
    rs = np.random.default_rng(106)
    import synth
    gout_np = synth.round_bf16(rs.normal(size=(G, T, d)).astype(np.float32))
    gout = torch.from_numpy(gout_np).cuda().to(torch.bfloat16)
    W1 = torch.from_numpy(case.W1).cuda().to(torch.bfloat16).contiguous()
    W2 = torch.from_numpy(case.W2).cuda().to(torch.bfloat16).contiguous()
    out = torch.empty_like(g["x"])
    loss = torch.empty(G, dtype=torch.float64, device="cuda")
    lam = 2.0
    layer.forward(g["x"], g["W1t"], g["b1"], g["W2t"], g["b2"], out, loss, w_router=g["w_router"],
                  alpha=case.alpha, beta=case.beta, train=True)
    f32 = dict(dtype=torch.float32, device="cuda")
    dx = torch.empty_like(g["x"])
    dW1 = torch.empty(NE, d, d_ff, **f32); db1 = torch.empty(NE, d_ff, **f32)
    dW2 = torch.empty(NE, d_ff, d, **f32); db2 = torch.empty(NE, d, **f32)
    dWr = torch.empty(case.cfg.logit_width, d, **f32)
    layer.backward(gout, dx, W1, W2, dW1, db1, dW2, db2, dW_router=dWr, lam=lam)
    torch.cuda.synchronize()
    assert layer.get_error() == 0
    v = layer.view()
    lg = v["logits"].cpu().numpy()
    _check_logits(case, lg)
    r = case.oracle_route(logits=lg)
    _check_route_full(case, layer, r, loss)
    # forward output on dense rows
    rows = dense_rows(case, r)
    got = out.view(-1, d)[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    ref = oracle.out_rows(case.cfg, r, case.x, case.W1, case.b1, case.W2, case.b2, rows=rows, threads=True)
    assert_close_scaled(got, ref, 2e-2, "C3 forward output")
    # gradients: sampled tokens (one per 512 of every rank + dropped ones), 8 columns
    keep = r.keep.reshape(-1).astype(bool)
    toks = np.unique(np.concatenate([np.arange(0, G * T, 509), np.flatnonzero(~keep)[:64], [G * T - 1]]))
    ex = np.where(keep[toks], r.dest1.reshape(-1)[toks] * case.cfg.sizes()[1] + r.dest2.reshape(-1)[toks], -1)
    toks = toks[np.argsort(ex, kind="stable")]               # expert-major: the oracle reuses its weight copy
    cols = np.array([0, 1, 511, 1024, 1535, 2047, 3000, d_ff - 1], np.int32)
    ref = oracle.backward_sampled(case.cfg, r, case.x, case.W1, case.b1, case.W2, case.b2, gout_np, toks, cols,
                                  lam=lam, W=case.w_router)
    tol = 3e-2
    dlg = v["dlogits"].cpu().numpy().reshape(G * T, -1)
    assert_close_scaled(dlg[toks], ref["dlogits"], tol, "C3 dlogits")
    assert_close_scaled(dx.view(G * T, d)[torch.from_numpy(toks).cuda()].float().cpu().numpy(), ref["dx"], tol, "C3 dx")
    cl = torch.from_numpy(cols.astype(np.int64)).cuda()
    assert_close_scaled(dW1[:, :, cl].cpu().numpy(), ref["dW1c"], tol, "C3 dW1 columns")
    assert_close_scaled(db1[:, cl].cpu().numpy(), ref["db1c"], tol, "C3 db1 entries")
    assert_close_scaled(dW2[:, cl, :].cpu().numpy(), ref["dW2r"], tol, "C3 dW2 rows")
    assert_close_scaled(db2.cpu().numpy(), ref["db2"], tol, "C3 db2")
    # tied router gradient (a19): dW = sum over every token of dlogits^T x
    dW_prop = dlg.astype(np.float64).T @ case.x.reshape(G * T, d).astype(np.float64)
    assert_close_scaled(dWr.cpu().numpy(), dW_prop, 1e-3, "C3 dW_router = dlogits^T x")
    layer.close()
