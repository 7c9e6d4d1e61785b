"""Multi-GPU parity (torchrun, one process per GPU, NCCL): the exchanges between
processes run as ncclAlltoAll on the split inter / intra communicators (V = 1) or as
grouped ncclSend/ncclRecv (several ranks per process); outputs and losses of every rank
must match the CPU oracle.  Skipped when fewer than 2 GPUs are visible."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cases(ngpu):
    base = dict(T=600, d=64, d_ff=128, dist="skewed", seed=11)
    cs = []
    if ngpu >= 2:
        cs += [dict(n=2, m=1, e=1, cf=1.0, dtype="fp32", mode="bilevel", **base),     # V=1, inter comm
               dict(n=1, m=2, e=2, cf=1.0, dtype="fp32", mode="bilevel", **base),     # V=1, intra comm
               dict(n=2, m=1, e=2, cf=1.25, dtype="bf16", mode="flat", **base),       # V=1, world
               dict(n=2, m=4, e=1, cf=1.0, dtype="bf16", mode="bilevel", **base),     # V=4 mixed
               dict(n=4, m=2, e=1, cf=1.25, dtype="fp32", mode="bilevel", **base),
               dict(n=2, m=4, e=1, cf=1.0, dtype="bf16", mode="flat", **base)]
    if ngpu >= 4:
        cs += [dict(n=2, m=2, e=1, cf=1.0, dtype="bf16", mode="bilevel", **base),     # V=1 all NCCL
               dict(n=2, m=2, e=2, cf=1.0, dtype="fp32", mode="flat", **base),
               dict(n=2, m=4, e=1, cf=2.0, dtype="bf16", mode="bilevel", **base)]     # V=2 mixed
    # the same cases through the fused permute -> peer-store exchange (CUDA IPC + NVLink)
    cs = cs + [dict(c, _peer=True) for c in cs]
    # CUDA-graph replays of the peer exchange (device-side barrier epochs) on new inputs
    if ngpu >= 2:
        cs += [dict(n=2, m=4, e=1, cf=1.0, dtype="bf16", mode="bilevel", _peer=True, _graph=True, **base),
               dict(n=2, m=1, e=2, cf=1.25, dtype="bf16", mode="flat", _peer=True, _graph=True, **base)]
    if ngpu >= 4:
        cs += [dict(n=2, m=2, e=1, cf=1.0, dtype="bf16", mode="bilevel", _peer=True, _graph=True, **base)]
    # the FLAT top-k layer (Eq. 2) across processes, both exchanges
    if ngpu >= 2:
        cs += [dict(n=2, m=2, e=2, cf=1.0, dtype="bf16", mode="flat", _topk=2, **base),
               dict(n=2, m=2, e=2, cf=1.0, dtype="bf16", mode="flat", _topk=2, _peer=True, **base),
               dict(n=2, m=1, e=2, cf=0.75, dtype="fp32", mode="flat", _topk=3, _peer=True, **base)]
    # training steps (a16-a19) over both exchanges
    bw = dict(T=400, d=128, d_ff=256, dist="skewed", seed=12)
    if ngpu >= 2:
        cs += [dict(n=2, m=1, e=1, cf=1.0, dtype="bf16", mode="bilevel", _bwd=True, **bw),
               dict(n=2, m=4, e=1, cf=1.25, dtype="bf16", mode="bilevel", _bwd=True, _peer=True, **bw),
               dict(n=2, m=2, e=2, cf=1.0, dtype="bf16", mode="flat", _bwd=True, _peer=True, **bw)]
    if ngpu >= 4:
        cs += [dict(n=2, m=2, e=1, cf=1.25, dtype="bf16", mode="bilevel", _bwd=True, _peer=True, **bw),
               dict(n=4, m=2, e=1, cf=1.25, dtype="bf16", mode="bilevel", _bwd=True, **bw)]
    return cs


def _run(n, cases, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "mgpu_worker.py"),
           json.dumps(cases)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-4000:]
    res = [ln for ln in r.stdout.splitlines() if ln.startswith("MGPU_RESULT")]
    fails = json.loads(res[-1][len("MGPU_RESULT"):])["failures"] if res else None
    assert r.returncode == 0, f"failures: {fails}\n{tail}"
    assert "MGPU_RESULT" in r.stdout, tail


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multigpu_exact_exchange_2():
    """SMILE_XCHG_EXACT=1: the NCCL exchanges move valid rows only (counts first); same
    oracle bar as the padded exchange, forward and training."""
    base = dict(T=600, d=64, d_ff=128, dist="skewed", seed=11)
    bw = dict(T=400, d=128, d_ff=256, dist="skewed", seed=12)
    cases = [dict(n=2, m=1, e=1, cf=1.0, dtype="fp32", mode="bilevel", **base),
             dict(n=2, m=4, e=1, cf=1.0, dtype="bf16", mode="bilevel", **base),
             dict(n=2, m=1, e=2, cf=1.25, dtype="bf16", mode="flat", **base),
             dict(n=2, m=4, e=2, cf=1.0, dtype="bf16", mode="flat", **base),
             dict(n=2, m=4, e=1, cf=1.25, dtype="bf16", mode="bilevel", _bwd=True, **bw)]
    os.environ["SMILE_XCHG_EXACT"] = "1"
    try:
        _run(2, cases, 29613)
    finally:
        del os.environ["SMILE_XCHG_EXACT"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multigpu_parity_2():
    _run(2, _cases(2), 29611)


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
def test_multigpu_parity_4():
    _run(4, [c for c in _cases(4) if c not in _cases(2)], 29612)
