"""CPU tests of libsmile's host side: the library loads, exports every symbol declared in
include/smile.h, and its pure-host functions (smile_plan, smile_group) follow the
paper's process-group layout (R10) and the capacity readings (R5, R7, R20).
No compute call is made (no GPU here)."""
import os
import re

import pytest

import paper_2212_05191_b200 as sm
from paper_2212_05191_b200 import smile as smb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2212_05191_b200 import build
    build.build()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "smile.h")).read()
    return sorted(set(re.findall(r"^\s*(?:smile_status|int|int64_t|const char\s*\*)\s*\*?\s*(smile_[a-z0-9_]+)\s*\(",
                                 src, re.M)))


def test_exports_every_declared_symbol():
    L = sm.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert L.smile_version() == 100
    assert L.smile_strerror(3) == b"non-finite router logit"
    assert smb.launch_count() == 0          # no kernel has been launched on this CPU-only host


def test_group_examples_spec():
    # (n=2, m=8) rank 9 -> intra {8..15}, inter {1, 9}; (n=3, m=2) rank 4 ->
    # intra {4, 5}, inter {0, 2, 4}; (n=1, m=4) -> inter groups are singletons.
    assert sm.group(2, 8, 2, 9) == list(range(8, 16))
    assert sm.group(2, 8, 1, 9) == [1, 9]
    assert sm.group(3, 2, 2, 4) == [4, 5]
    assert sm.group(3, 2, 1, 4) == [0, 2, 4]
    assert sm.group(1, 4, 1, 2) == [2]
    assert sm.group(2, 4, 0, 5) == list(range(8))


def test_groups_partition_exhaustive():
    # every rank in exactly one intra and one inter group; the two are orthogonal
    for n in range(1, 9):
        for m in range(1, 9):
            if n * m > 64:
                continue
            G = n * m
            for lvl in (1, 2):
                seen = {}
                for r in range(G):
                    g = tuple(sm.group(n, m, lvl, r))
                    assert r in g
                    for q in g:
                        assert tuple(sm.group(n, m, lvl, q)) == g
                    seen[g] = True
                assert sum(len(g) for g in seen) == G
            for r in range(G):
                assert set(sm.group(n, m, 1, r)) & set(sm.group(n, m, 2, r)) == {r}


def test_plan_sizes_and_validation():
    z = sm.plan(n=2, m=4, e=1, d=768, d_ff=3072, T=16384, cf=2.0, dtype="bf16", mode="bilevel")
    assert (z.G, z.V, z.K1, z.K2, z.KW, z.C1, z.C2, z.S, z.Cseg) == (8, 8, 2, 4, 6, 16384, 8192, 4, 8192)
    z = sm.plan(n=2, m=4, e=1, d=768, d_ff=3072, T=16384, cf=2.0, dtype="bf16", mode="flat")
    assert (z.K1, z.K2, z.KW, z.C1, z.C2, z.S, z.Cseg) == (8, 1, 8, 4096, 0, 8, 4096)
    z = sm.plan(n=2, m=4, e=8, d=1024, d_ff=4096, T=65536, cf=2.0, dtype="bf16", mode="bilevel", nprocs=8, proc=5)
    assert (z.V, z.rank0, z.K2, z.C2) == (1, 5, 32, 4096)
    z = sm.plan(n=4, m=1, e=1, d=64, d_ff=64, T=10, cf=0.5, dtype="fp32", mode="bilevel")
    assert (z.K2, z.C1, z.C2) == (1, 2, 8)         # ceil(0.5*10/4); K2 = 1: identity level holds n*C1 (R20)
    bad = dict(n=2, m=4, e=1, d=64, d_ff=64, T=10, cf=1.0, dtype="fp32", mode="bilevel")
    for k, v in (("n", 0), ("m", 0), ("e", 0), ("T", -1), ("cf", 0.0), ("nprocs", 3)):
        with pytest.raises(smb.SmileError) as ei:
            sm.plan(**{**bad, k: v})
        assert ei.value.code == 1
    with pytest.raises(smb.SmileError) as ei:
        sm.plan(**{**bad, "d": 6})                  # rows must be 16-byte multiples
    assert ei.value.code == 2


def test_capacity_matches_oracle():
    """smile_capacity: ceil(cf*T/dests) per (sending rank, destination),
    P:L207 + R5 / R20, against the pinned oracle_capacity (tests/test_oracle_routing.py)
    over the paper's capacity factors, ragged T and the single-destination identity."""
    import oracle
    for T in (0, 1, 7, 8, 255, 1000, 16384, 32768, 65536, 1 << 30):
        for dests in (1, 2, 3, 4, 7, 8, 32, 64, 128):
            for cf in (0.5, 1.0, 1.25, 2.0, 8.0):
                assert smb.capacity(T, dests, cf) == oracle.capacity(T, dests, cf), (T, dests, cf)
    assert smb.capacity(8, 4, 2.0) == 4 and smb.capacity(7, 2, 1.0) == 4
    assert smb.capacity(16384, 1, 2.0) == 16384                                 # R20: no capacity
    for bad in ((-1, 2, 1.0), (10, 0, 1.0), (10, 2, 0.0), (10, 2, -1.0), (10, 2, float("nan"))):
        assert smb.capacity(*bad) == -1, bad
