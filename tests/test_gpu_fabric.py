"""The emulated heterogeneous fabric (smile_set_fabric, SURVEY 8(f) row 1 -- an in-box
EMULATION of a slower inter-node network): cross-node transfers of
the COPY exchange go through per-rank emulated NICs.  It moves the same rows, so outputs
are bit-identical to the plain COPY exchange (and hence to the oracle); and its cost model
is a hard lower bound: every cross-node message occupies its NIC for latency + bytes/BW,
so a layer whose ranks send k cross-node messages per exchange cannot be faster than
k * latency per exchange -- which is where the paper's O(mn) -> O(m + n) message count
 separates the two layers."""
import numpy as np
import pytest
import torch

from harness import Case, assert_close_scaled

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["bilevel", "flat"])
def test_fabric_bit_identical(mode):
    case = Case(2, 4, 2, 600, 64, 128, 1.25, dtype="bf16", mode=mode, dist="skewed", seed=61)
    layer, o_plain, l_plain, err = case.run_gpu()
    assert err == 0
    layer.set_fabric(40.0, 3.0)
    _, o_fab, l_fab, err = case.run_gpu(layer=layer)
    assert err == 0
    assert torch.equal(o_plain, o_fab) and torch.equal(l_plain, l_fab)
    assert_close_scaled(o_fab.float().cpu().numpy().reshape(-1, 64), case.oracle_out(case.oracle_route()), 2e-2,
                        "fabric vs oracle")
    layer.set_fabric(0.0, 0.0)                      # disabled again
    layer.close()


def _forward_ms(case, layer, reps=3):
    g = case.gpu_tensors()
    out = torch.empty_like(g["x"])
    loss = torch.empty(layer.V, dtype=torch.float64, device="cuda")
    run = lambda: layer.forward(g["x"], g["W1t"], g["b1"], g["W2t"], g["b2"], out, loss, logits=g["logits"],
                                alpha=case.alpha, beta=case.beta)
    run()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    assert layer.get_error() == 0
    return min(ts)


def test_fabric_message_count_lower_bound():
    """2 x 4 hierarchy, 1 ms per cross-node message, bandwidth effectively unbounded:
    bi-level sends n - 1 = 1 cross-node message per rank per inter exchange (2 exchanges per
    forward), flat m (n - 1) = 4 per world exchange (2 per forward) -> >= 2 ms vs >= 8 ms."""
    from paper_2212_05191_b200 import SmileLayer
    lat = 1000.0
    t = {}
    for mode in ("bilevel", "flat"):
        case = Case(2, 4, 1, 256, 64, 128, 1.0, dtype="bf16", mode=mode, dist="balanced", seed=62)
        layer = SmileLayer(2, 4, 1, 64, 128, 256, 1.0, "bf16", mode)
        layer.set_fabric(1e6, lat)
        t[mode] = _forward_ms(case, layer)
        layer.close()
    assert t["bilevel"] >= 2 * lat / 1e3 * 0.999
    assert t["flat"] >= 8 * lat / 1e3 * 0.999
    assert t["flat"] > t["bilevel"] + 5.0


def test_fabric_refuses_peer_exchange():
    from paper_2212_05191_b200 import SmileLayer, SmileError
    layer = SmileLayer(2, 2, 1, 64, 128, 100, 1.0, "bf16", "bilevel")
    layer.set_fabric(50.0, 5.0)
    with pytest.raises(SmileError):
        layer.enable_peer_exchange()
    layer.set_fabric(0.0, 0.0)
    layer.enable_peer_exchange()
    with pytest.raises(SmileError):
        layer.set_fabric(50.0, 5.0)
    layer.close()
