"""N > 1 host logic on CPU: world_size-2 gloo processes execute libsmile's cross-process
exchange schedule (smile_exchange_plan, the exact op list smile_all2all posts to NCCL)
with torch.distributed send/recv on CPU tensors, plus the in-process device-copy pairs
emulated in numpy, and check that every chunk lands where the level's All2All puts it
(R10): chunk p of rank r arrives at member p as chunk pos(r)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2212_05191_b200 as sm
from paper_2212_05191_b200 import smile as smb


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _code(src, dst, L):
    return np.arange(L, dtype=np.int64) + 1_000_000 * src + 1000 * dst


def _worker(proc, nprocs, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=proc, world_size=nprocs)
    ok = []
    try:
        for (n, m, e, mode, level) in cases:
            G = n * m
            V = G // nprocs
            rank0 = proc * V
            kw = dict(n=n, m=m, e=e, d=8, d_ff=8, T=16, cf=1.0, dtype="fp32", mode=mode, nprocs=nprocs, proc=proc)
            members = [sm.group(n, m, level, rank0 + v) for v in range(V)]
            P = len(members[0])
            L = 5
            send = np.zeros((V, P, L), np.int64)
            for v in range(V):
                for p, qr in enumerate(members[v]):
                    send[v, p] = _code(rank0 + v, qr, L)
            recv = np.full((V, P, L), -1, np.int64)
            # in-process pairs: the device-copy path
            for v in range(V):
                for p, qr in enumerate(members[v]):
                    if qr // V == proc:
                        pos = members[qr - rank0].index(rank0 + v)
                        recv[qr - rank0, pos] = send[v, p]
            ops = smb.exchange_plan(level, **kw)
            reqs, bufs = [], []
            for kind, peer, src, dst, chunk in ops:
                v, p = divmod(chunk, P)
                if kind == 0:
                    assert src == rank0 + v and members[v][p] == dst and peer == dst // V
                    t = torch.from_numpy(send[v, p].copy())
                    reqs.append(dist.isend(t, peer))
                else:
                    assert dst == rank0 + v and members[v][p] == src and peer == src // V
                    t = torch.empty(L, dtype=torch.int64)
                    bufs.append((v, p, t))
                    reqs.append(dist.irecv(t, peer))
            for r in reqs:
                r.wait()
            for v, p, t in bufs:
                recv[v, p] = t.numpy()
            for v in range(V):
                for p, qr in enumerate(members[v]):
                    assert (recv[v, p] == _code(qr, rank0 + v, L)).all(), (n, m, mode, level, v, p)
            ok.append((n, m, e, mode, level))
        q.put((proc, "ok", ok))
    except Exception as ex:  # noqa: BLE001
        q.put((proc, "fail", repr(ex)))
    finally:
        dist.destroy_process_group()


CASES = [
    (2, 4, 1, "bilevel", 1), (2, 4, 1, "bilevel", 2),       # V = 4: inter remote, intra local
    (4, 2, 1, "bilevel", 1), (4, 2, 1, "bilevel", 2),       # V = 4: 4x2
    (2, 4, 2, "flat", 0),                                   # world exchange
    (2, 1, 1, "bilevel", 1), (1, 2, 1, "bilevel", 2),       # V = 1 collapses
    (2, 2, 1, "bilevel", 1), (2, 2, 1, "bilevel", 2), (2, 2, 1, "flat", 0),
]


def test_exchange_plan_two_processes_gloo():
    from paper_2212_05191_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, CASES, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for proc, status, info in res:
        assert status == "ok", (proc, info)
        assert len(info) == len(CASES)


def test_exchange_plan_counts():
    # V = 1 (one rank per process): every non-self member is remote; 2((n-1)+(m-1)) p2p
    # sends per rank for bi-level vs 2(G-1) flat over a forward+reverse pair (A12)
    for n, m in [(2, 4), (4, 2), (2, 2)]:
        G = n * m
        kw = dict(n=n, m=m, e=1, d=8, d_ff=8, T=16, cf=1.0, dtype="fp32", nprocs=G)
        bi = sum(sum(1 for o in smb.exchange_plan(lv, mode="bilevel", proc=0, **kw) if o[0] == 0) for lv in (1, 2))
        fl = sum(1 for o in smb.exchange_plan(0, mode="flat", proc=0, **kw) if o[0] == 0)
        assert 2 * bi == 2 * ((n - 1) + (m - 1))
        assert 2 * fl == 2 * (G - 1)
