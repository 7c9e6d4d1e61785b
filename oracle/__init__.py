"""CPU oracle for the SMILE bi-level MoE layer -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_2212_05191_b200`` never imports it; the two share no code.

This module is argument marshalling around ``oracle/smile_oracle.c`` (plain C, fp64): it
compiles the C file with gcc on first use and calls it through ctypes with numpy arrays.
Every function of the arithmetic, and the passage of PAPER.md it follows, is documented
in the C file.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smile_oracle.c")
_LIB = os.path.join(_HERE, "libsmile_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math: IEEE semantics are part of the
    contract, e.g. the strict '>' argmax and the fp64 softmax)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        base = ["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-fno-fast-math", "-ffp-contract=off", "-o", tmp, _SRC]
        try:   # OpenMP only distributes independent rows of the _mt functions (bit-identical results)
            subprocess.check_call(base + ["-fopenmp", "-lm"], stderr=subprocess.DEVNULL)
        except subprocess.CalledProcessError:
            subprocess.check_call(base + ["-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("e", C.c_int32), ("flat", C.c_int32),
                ("T", C.c_int64), ("cf", C.c_double), ("alpha", C.c_double), ("beta", C.c_double)]


_P = C.c_void_p


class _Route(C.Structure):
    _fields_ = [(k, _P) for k in ("dest1", "dest2", "slot1", "keep1", "keep", "p", "q", "gate",
                                   "counts1", "A1", "A2", "S1", "S2", "loss",
                                   "jin", "slot2", "keep2", "counts2")]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_capacity.restype = C.c_int64
        _lib.oracle_capacity.argtypes = [C.c_int64, C.c_int64, C.c_double]
        _lib.oracle_sizes.argtypes = [C.POINTER(_Cfg)] + [C.POINTER(C.c_int64)] * 4
        _lib.oracle_logits.argtypes = [C.c_int64, C.c_int32, C.c_int32, _P, _P, _P]
        _lib.oracle_route.restype = C.c_int
        _lib.oracle_route.argtypes = [C.POINTER(_Cfg), _P, C.POINTER(_Route)]
        _lib.oracle_ffn_row.argtypes = [C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P]
        _lib.oracle_out_rows.argtypes = [C.POINTER(_Cfg), C.c_int32, C.c_int32, _P, C.POINTER(_Route),
                                         _P, _P, _P, _P, C.c_int32, C.c_int64, _P, _P]
        _lib.oracle_objective.restype = C.c_double
        _lib.oracle_objective.argtypes = [C.POINTER(_Cfg), C.c_int32, C.c_int32] + [_P] * 8 + [C.c_double, _P, _P]
        _lib.oracle_backward.argtypes = [C.POINTER(_Cfg), C.c_int32, C.c_int32, _P, _P, _P, C.POINTER(_Route),
                                         _P, _P, _P, _P, _P, C.c_double] + [_P] * 7
        _lib.oracle_route_topk.restype = C.c_int
        _lib.oracle_route_topk.argtypes = [C.POINTER(_Cfg), C.c_int32, _P] + [_P] * 8
        _lib.oracle_out_rows_topk.argtypes = [C.POINTER(_Cfg), C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P,
                                              _P, _P, _P, _P, C.c_int32, C.c_int64, _P, _P]
        _lib.oracle_backward_topk.argtypes = [C.POINTER(_Cfg), C.c_int32, C.c_int32, C.c_int32] + [_P] * 11 + \
            [C.c_double] + [_P] * 7
        _lib.oracle_objective_topk.restype = C.c_double
        _lib.oracle_objective_topk.argtypes = [C.POINTER(_Cfg), C.c_int32, C.c_int32, C.c_int32] + [_P] * 11 + \
            [C.c_double]
        _lib.oracle_logits_mt.argtypes = [C.c_int64, C.c_int32, C.c_int32, _P, _P, _P]
        _lib.oracle_out_rows_mt.argtypes = _lib.oracle_out_rows.argtypes
        _lib.oracle_threads.restype = C.c_int32
        _lib.oracle_backward_sampled.argtypes = [C.POINTER(_Cfg), C.c_int32, C.c_int32, _P, _P, _P, C.POINTER(_Route),
                                                 _P, _P, _P, _P, _P, C.c_double, C.c_int64, _P, C.c_int32, _P] + [_P] * 6
    return _lib


@dataclass
class Config:
    """n groups x m ranks, e experts per rank, T tokens per rank (see smile_oracle.c)."""
    n: int
    m: int
    e: int = 1
    T: int = 8
    cf: float = 2.0
    flat: bool = False
    alpha: float = 0.005
    beta: float = 0.005

    @property
    def G(self) -> int:
        return self.n * self.m

    def _c(self) -> _Cfg:
        return _Cfg(self.n, self.m, self.e, int(self.flat), self.T, self.cf, self.alpha, self.beta)

    def sizes(self):
        """(K1, K2, C1, C2) of the configuration."""
        v = [C.c_int64() for _ in range(4)]
        lib().oracle_sizes(C.byref(self._c()), *[C.byref(x) for x in v])
        return tuple(int(x.value) for x in v)

    @property
    def logit_width(self) -> int:
        K1, K2, _, _ = self.sizes()
        return K1 if self.flat else K1 + K2


def capacity(T: int, dests: int, cf: float) -> int:
    return int(lib().oracle_capacity(T, dests, cf))


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def logits(x: np.ndarray, W: np.ndarray, threads: bool = False) -> np.ndarray:
    """Eq. (1) logits, fp32 of an fp64 accumulation.  x [rows, d], W [K, d].
    threads=True: oracle_logits_mt (rows over OpenMP threads, bit-identical)."""
    x = np.ascontiguousarray(x, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    out = np.empty((x.shape[0], W.shape[0]), np.float32)
    fn = lib().oracle_logits_mt if threads else lib().oracle_logits
    fn(x.shape[0], x.shape[1], W.shape[0], _ptr(x), _ptr(W), _ptr(out))
    return out


def threads() -> int:
    """OpenMP threads of the _mt functions (1 when the oracle was built without OpenMP)."""
    return int(lib().oracle_threads())


class Route:
    """All outputs of oracle_route (numpy arrays, shapes as in smile_oracle.c)."""

    def __init__(self, cfg: Config):
        K1, K2, C1, C2 = cfg.sizes()
        G, T, n = cfg.G, cfg.T, cfg.n
        self.cfg, self.K1, self.K2, self.C1, self.C2 = cfg, K1, K2, C1, C2
        z = lambda shape, dt: np.zeros(shape, dt)
        self.dest1, self.dest2, self.slot1 = z((G, T), np.int32), z((G, T), np.int32), z((G, T), np.int32)
        self.keep1, self.keep = z((G, T), np.uint8), z((G, T), np.uint8)
        self.p, self.q, self.gate = z((G, T), np.float32), z((G, T), np.float32), z((G, T), np.float32)
        self.counts1 = z((G, K1), np.int32)
        self.A1, self.A2 = z((G, K1), np.int64), z((G, K2), np.int64)
        self.S1, self.S2 = z((G, K1), np.float64), z((G, K2), np.float64)
        self.loss = z((G,), np.float64)
        nc = max(n * C1, 1)
        self.jin, self.slot2 = z((G, nc), np.int32), z((G, nc), np.int32)
        self.keep2 = z((G, nc), np.uint8)
        self.counts2 = z((G, K2), np.int32)
        self._s = _Route(*[self.__dict__[k].ctypes.data_as(C.c_void_p) for k, _ in _Route._fields_])


def route(cfg: Config, lg: np.ndarray) -> Route:
    """Run the bi-level (or flat) routing of every rank.  lg [G, T, logit_width] fp32."""
    lg = np.ascontiguousarray(lg, np.float32)
    assert lg.shape == (cfg.G, cfg.T, cfg.logit_width), lg.shape
    r = Route(cfg)
    rc = lib().oracle_route(C.byref(cfg._c()), _ptr(lg), C.byref(r._s))
    if rc == 3:
        raise ValueError("non-finite logits")
    if rc != 0:
        raise ValueError(f"invalid configuration ({rc})")
    return r


def ffn_row(x, W1, b1, W2, b2) -> np.ndarray:
    """One expert, one token: W2^T GELU(W1^T x + b1) + b2 in fp64.  W1 [d, d_ff]."""
    f = lambda a: np.ascontiguousarray(a, np.float32)
    x, W1, b1, W2, b2 = map(f, (x, W1, b1, W2, b2))
    y = np.empty(W1.shape[0], np.float64)
    lib().oracle_ffn_row(W1.shape[0], W1.shape[1], _ptr(x), _ptr(W1), _ptr(b1), _ptr(W2), _ptr(b2), _ptr(y))
    return y


def out_rows(cfg: Config, r: Route, x: np.ndarray, W1=None, b1=None, W2=None, b2=None,
             rows=None, identity: bool = False, threads: bool = False) -> np.ndarray:
    """Eq. (3) layer output (fp64) for the global token rows g = rank*T + t.
    x [G, T, d]; W1 [G*e, d, d_ff], b1 [G*e, d_ff], W2 [G*e, d_ff, d], b2 [G*e, d].
    threads=True: oracle_out_rows_mt (rows over OpenMP threads, bit-identical)."""
    x = np.ascontiguousarray(x, np.float32)
    d = x.shape[-1]
    if identity:
        W1 = b1 = W2 = b2 = np.zeros(1, np.float32)
        d_ff = 0
    else:
        W1, b1, W2, b2 = (np.ascontiguousarray(a, np.float32) for a in (W1, b1, W2, b2))
        d_ff = W1.shape[-1]
    rows = np.arange(cfg.G * cfg.T, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    out = np.empty((rows.shape[0], d), np.float64)
    fn = lib().oracle_out_rows_mt if threads else lib().oracle_out_rows
    fn(C.byref(cfg._c()), d, d_ff, _ptr(x), C.byref(r._s), _ptr(W1), _ptr(b1),
       _ptr(W2), _ptr(b2), int(identity), rows.shape[0], _ptr(rows), _ptr(out))
    return out


def _ptr_or_none(a):
    return None if a is None else _ptr(a)


def objective(cfg: Config, x, W1, b1, W2, b2, gout, lam=1.0, W=None, logits=None):
    """fp64 objective J = sum <gout, OUT> + lam * sum_r loss_r (smile_oracle.c).  Arrays are
    taken as fp64 (x [G,T,d]; W [KW,d] or logits [G,T,KW]).  Returns (J, keep, dest)."""
    f = lambda a: None if a is None else np.ascontiguousarray(a, np.float64)
    x, W1, b1, W2, b2, gout, W, logits = map(f, (x, W1, b1, W2, b2, gout, W, logits))
    keep = np.zeros(cfg.G * cfg.T, np.uint8)
    dest = np.zeros(cfg.G * cfg.T * 2, np.int32)
    J = lib().oracle_objective(C.byref(cfg._c()), x.shape[-1], W1.shape[-1], _ptr(x), _ptr_or_none(W),
                               _ptr_or_none(logits), _ptr(W1), _ptr(b1), _ptr(W2), _ptr(b2), _ptr(gout), lam,
                               _ptr(keep), _ptr(dest))
    return J, keep, dest


def backward(cfg: Config, r: Route, x, W1, b1, W2, b2, gout, lam=1.0, W=None, logits=None):
    """Gradients of the objective (smile_oracle.c oracle_backward), fp64.  Returns a dict
    with dlogits [G,T,KW], dx [G,T,d], dW [KW,d] (None without W), dW1, db1, dW2, db2."""
    f = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)
    x, W1, b1, W2, b2, gout, W, logits = map(f, (x, W1, b1, W2, b2, gout, W, logits))
    G, T, d = x.shape
    d_ff = W1.shape[-1]
    NE = W1.shape[0]
    KW = cfg.logit_width
    out = dict(dlogits=np.zeros((G, T, KW)), dx=np.zeros((G, T, d)), dW=None if W is None else np.zeros((KW, d)),
               dW1=np.zeros((NE, d, d_ff)), db1=np.zeros((NE, d_ff)), dW2=np.zeros((NE, d_ff, d)),
               db2=np.zeros((NE, d)))
    lib().oracle_backward(C.byref(cfg._c()), d, d_ff, _ptr(x), _ptr_or_none(W), _ptr_or_none(logits), C.byref(r._s),
                          _ptr(W1), _ptr(b1), _ptr(W2), _ptr(b2), _ptr(gout), lam, _ptr(out["dlogits"]),
                          _ptr(out["dx"]), _ptr_or_none(out["dW"]), _ptr(out["dW1"]), _ptr(out["db1"]),
                          _ptr(out["dW2"]), _ptr(out["db2"]))
    return out


def backward_sampled(cfg: Config, r: Route, x, W1, b1, W2, b2, gout, tokens, cols, lam=1.0, W=None, logits=None):
    """oracle_backward_sampled: the entries of oracle_backward a full-size test can afford
    -- dlogits / dx of the listed global token rows, dW1[:, :, cols], db1[:, cols],
    dW2[:, cols, :] and all of db2 -- bit-identical to the full function's.  Returns a dict
    of fp64 arrays: dlogits [ntok, KW], dx [ntok, d], dW1c [NE, d, ncol], db1c [NE, ncol],
    dW2r [NE, ncol, d], db2 [NE, d]."""
    f = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)
    x, W1, b1, W2, b2, gout, W, logits = map(f, (x, W1, b1, W2, b2, gout, W, logits))
    G, T, d = x.shape
    d_ff = W1.shape[-1]
    NE = W1.shape[0]
    KW = cfg.logit_width
    tokens = np.ascontiguousarray(tokens, np.int64)
    cols = np.ascontiguousarray(cols, np.int32)
    nt, nc = tokens.shape[0], cols.shape[0]
    out = dict(dlogits=np.zeros((nt, KW)), dx=np.zeros((nt, d)), dW1c=np.zeros((NE, d, nc)), db1c=np.zeros((NE, nc)),
               dW2r=np.zeros((NE, nc, d)), db2=np.zeros((NE, d)))
    lib().oracle_backward_sampled(C.byref(cfg._c()), d, d_ff, _ptr(x), _ptr_or_none(W), _ptr_or_none(logits),
                                  C.byref(r._s), _ptr(W1), _ptr(b1), _ptr(W2), _ptr(b2), _ptr(gout), lam, nt,
                                  _ptr(tokens), nc, _ptr(cols), _ptr(out["dlogits"]), _ptr(out["dx"]),
                                  _ptr(out["dW1c"]), _ptr(out["db1c"]), _ptr(out["dW2r"]), _ptr(out["db2"]))
    return out


class RouteTopk:
    """Outputs of oracle_route_topk (flat top-k layer, Eq. 2): choice-major arrays [k, G, T]."""

    def __init__(self, cfg: Config, k: int):
        G, T = cfg.G, cfg.T
        K = G * cfg.e
        self.cfg, self.k, self.K = cfg, k, K
        self.dest = np.zeros((k, G, T), np.int32)
        self.slot = np.zeros((k, G, T), np.int32)
        self.keep = np.zeros((k, G, T), np.uint8)
        self.w = np.zeros((k, G, T), np.float32)
        self.counts = np.zeros((G, K), np.int32)
        self.A1 = np.zeros((G, K), np.int64)
        self.S1 = np.zeros((G, K), np.float64)
        self.loss = np.zeros(G, np.float64)


def route_topk(cfg: Config, k: int, lg: np.ndarray) -> RouteTopk:
    """Top-k routing of the flat layer (oracle_route_topk).  lg [G, T, G*e] fp32."""
    assert cfg.flat
    lg = np.ascontiguousarray(lg, np.float32)
    assert lg.shape == (cfg.G, cfg.T, cfg.G * cfg.e), lg.shape
    r = RouteTopk(cfg, k)
    rc = lib().oracle_route_topk(C.byref(cfg._c()), k, _ptr(lg), *[_ptr(a) for a in (
        r.dest, r.slot, r.keep, r.w, r.counts, r.A1, r.S1, r.loss)])
    if rc == 3:
        raise ValueError("non-finite logits")
    if rc != 0:
        raise ValueError(f"invalid configuration ({rc})")
    return r


def out_rows_topk(cfg: Config, r: RouteTopk, x, W1=None, b1=None, W2=None, b2=None, rows=None,
                  identity: bool = False) -> np.ndarray:
    """Eq. (2) output of the top-k layer (fp64) for global token rows g = rank*T + t."""
    x = np.ascontiguousarray(x, np.float32)
    d = x.shape[-1]
    if identity:
        W1 = b1 = W2 = b2 = np.zeros(1, np.float32)
        d_ff = 0
    else:
        W1, b1, W2, b2 = (np.ascontiguousarray(a, np.float32) for a in (W1, b1, W2, b2))
        d_ff = W1.shape[-1]
    rows = np.arange(cfg.G * cfg.T, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    out = np.empty((rows.shape[0], d), np.float64)
    lib().oracle_out_rows_topk(C.byref(cfg._c()), r.k, d, d_ff, _ptr(x), _ptr(r.dest), _ptr(r.keep), _ptr(r.w),
                               _ptr(W1), _ptr(b1), _ptr(W2), _ptr(b2), int(identity), rows.shape[0], _ptr(rows),
                               _ptr(out))
    return out


def backward_topk(cfg: Config, r: RouteTopk, x, W1, b1, W2, b2, gout, lam=1.0, W=None, logits=None):
    """oracle_backward_topk: gradients of the top-k objective (fp64).  Returns a dict like
    backward(): dlogits [G,T,K], dx [G,T,d], dW [K,d] or None, dW1, db1, dW2, db2."""
    f = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)
    x, W1, b1, W2, b2, gout, W, logits = map(f, (x, W1, b1, W2, b2, gout, W, logits))
    G, T, d = x.shape
    d_ff = W1.shape[-1]
    NE = W1.shape[0]
    K = r.K
    out = dict(dlogits=np.zeros((G, T, K)), dx=np.zeros((G, T, d)), dW=None if W is None else np.zeros((K, d)),
               dW1=np.zeros((NE, d, d_ff)), db1=np.zeros((NE, d_ff)), dW2=np.zeros((NE, d_ff, d)),
               db2=np.zeros((NE, d)))
    lib().oracle_backward_topk(C.byref(cfg._c()), r.k, d, d_ff, _ptr(x), _ptr_or_none(W), _ptr_or_none(logits),
                               _ptr(r.dest), _ptr(r.keep), _ptr(r.A1), _ptr(W1), _ptr(b1), _ptr(W2), _ptr(b2),
                               _ptr(gout), lam, _ptr(out["dlogits"]), _ptr(out["dx"]), _ptr_or_none(out["dW"]),
                               _ptr(out["dW1"]), _ptr(out["db1"]), _ptr(out["dW2"]), _ptr(out["db2"]))
    return out


def objective_topk(cfg: Config, r: RouteTopk, x, W1, b1, W2, b2, gout, lam=1.0, W=None, logits=None) -> float:
    """oracle_objective_topk: J with the routing decisions of r held fixed (fp64 inputs)."""
    f = lambda a: None if a is None else np.ascontiguousarray(a, np.float64)
    x, W1, b1, W2, b2, gout, W, logits = map(f, (x, W1, b1, W2, b2, gout, W, logits))
    d = x.shape[-1]
    return float(lib().oracle_objective_topk(C.byref(cfg._c()), r.k, d, W1.shape[-1], _ptr(x), _ptr_or_none(W),
                                             _ptr_or_none(logits), _ptr(r.dest), _ptr(r.keep), _ptr(r.A1), _ptr(W1),
                                             _ptr(b1), _ptr(W2), _ptr(b2), _ptr(gout), lam))
