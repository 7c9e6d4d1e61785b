"""smile_forward_chunked (the paper's pipe_overlapping appendix,
P:L391-405): the layer over c chunks of T/c tokens per rank, pipelined on two streams.
Each chunk is its own layer with capacities ceil(cf * (T/c) / K) (R5 per chunk), so the
oracle is run per chunk with T/c tokens; routing bit-exact (supplied logits), outputs
within bf16 tolerance, and bit-identical to running the chunks one by one with
smile_forward."""
import numpy as np
import pytest
import torch

from harness import Case, assert_close_scaled

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,peer,c", [("bilevel", True, 3), ("bilevel", False, 2), ("flat", True, 4),
                                         ("flat", False, 3)])
def test_forward_chunked_matches_per_chunk_oracle(mode, peer, c):
    from paper_2212_05191_b200 import SmileLayer, forward_chunked
    n, m, e, d, d_ff, cf = 2, 4, 1, 128, 256, 1.25
    Tc = 480
    T = Tc * c
    full = Case(n, m, e, T, d, d_ff, cf, dtype="bf16", mode=mode, dist="skewed", seed=51)
    layers = [SmileLayer(n, m, e, d, d_ff, Tc, cf, "bf16", mode) for _ in range(c)]
    for L in layers:
        L.alloc_workspace()
        L.ws.fill_(0x7f)                                    # garbage: every buffer must be rewritten
        if peer:
            L.enable_peer_exchange()
    g = full.gpu_tensors()
    sl = lambda k: slice(k * Tc, (k + 1) * Tc)
    xs = [g["x"][:, sl(k)].contiguous() for k in range(c)]
    lgs = [g["logits"][:, sl(k)].contiguous() for k in range(c)]
    outs = [torch.full_like(xs[k], float("nan")) for k in range(c)]
    losses = [torch.empty(layers[0].V, dtype=torch.float64, device="cuda") for _ in range(c)]
    s2 = torch.cuda.Stream()
    for _ in range(2):                                      # twice: the per-chunk state resets between calls
        forward_chunked(layers, xs, g["W1t"], g["b1"], g["W2t"], g["b2"], outs, losses, logits=lgs,
                        alpha=full.alpha, beta=full.beta, stream2=s2)
    torch.cuda.synchronize()
    for L in layers:
        assert L.get_error() == 0
    for k in range(c):
        ck = Case(n, m, e, Tc, d, d_ff, cf, dtype="bf16", mode=mode, dist="skewed", seed=51)
        ck.x = np.ascontiguousarray(full.x[:, sl(k)])
        ck.logits = np.ascontiguousarray(full.logits[:, sl(k)])
        r = ck.oracle_route()
        v = layers[k].view()
        np.testing.assert_array_equal(v["dest1"].cpu().numpy(), r.dest1)
        np.testing.assert_array_equal(v["slot1"].cpu().numpy(), r.slot1)
        np.testing.assert_array_equal(v["counts1"].cpu().numpy(), r.counts1)
        if mode == "bilevel":
            np.testing.assert_array_equal(v["counts2"].cpu().numpy(), r.counts2)
        assert (r.keep == 0).any()
        assert_close_scaled(outs[k].float().cpu().numpy().reshape(-1, d), ck.oracle_out(r), 2e-2, f"chunk {k}")
        np.testing.assert_allclose(losses[k].cpu().numpy(), r.loss, rtol=1e-6)
        # the same chunk through plain smile_forward: bit-identical
        o2 = torch.empty_like(xs[k])
        l2 = torch.empty_like(losses[k])
        layers[k].forward(xs[k], g["W1t"], g["b1"], g["W2t"], g["b2"], o2, l2, logits=lgs[k], alpha=full.alpha,
                          beta=full.beta)
        torch.cuda.synchronize()
        assert torch.equal(o2, outs[k]) and torch.equal(l2, losses[k])
    for L in layers:
        L.close()


def test_forward_chunked_rejects_bad_arguments():
    from paper_2212_05191_b200 import SmileLayer, SmileError, forward_chunked
    L0 = SmileLayer(2, 2, 1, 64, 128, 100, 1.0, "bf16", "bilevel")
    L1 = SmileLayer(2, 2, 1, 64, 128, 120, 1.0, "bf16", "bilevel")       # other chunk size
    x = torch.zeros(4, 100, 64, dtype=torch.bfloat16, device="cuda")
    W1t = torch.zeros(4, 128, 64, dtype=torch.bfloat16, device="cuda")
    W2t = torch.zeros(4, 64, 128, dtype=torch.bfloat16, device="cuda")
    b1, b2 = torch.zeros(4, 128, device="cuda"), torch.zeros(4, 64, device="cuda")
    wr = torch.zeros(L0.KW, 64, device="cuda")
    loss = torch.empty(4, dtype=torch.float64, device="cuda")
    s2 = torch.cuda.Stream()
    with pytest.raises(SmileError):                                      # shapes differ
        forward_chunked([L0, L1], [x, x], W1t, b1, W2t, b2, [x, x], [loss, loss], w_router=wr, stream2=s2)
    with pytest.raises(SmileError):                                      # one context twice
        forward_chunked([L0, L0], [x, x], W1t, b1, W2t, b2, [x, x], [loss, loss], w_router=wr, stream2=s2)
    L0.close()
    L1.close()
