"""ctypes binding of libsmile (include/smile.h).  Argument marshalling only.

PyTorch supplies device memory, streams and (for bootstrap) torch.distributed; every
step of the layer runs in libsmile's kernels.  Names follow the C ABI: gate_inter,
dispatch, all2all_inter / all2all_intra / all2all, gate_intra, expert_ffn, combine,
aux_loss, forward, forward_host.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SMILE_LIB_PATH: load another build of the library (same-box A/B measurements only)
LIB_PATH = os.environ.get("SMILE_LIB_PATH") or os.path.join(_HERE, "libsmile.so")
_lib = None

BILEVEL, FLAT = 0, 1
FP32, BF16 = 0, 1
FFN_AUTO, FFN_SIMT, FFN_TCGEN05 = 0, 1, 2
XCHG_COPY, XCHG_PEER = 0, 1
TCGEN05_DEFAULT = True    # AUTO resolves bf16 to the tcgen05 FFN (api.cu smile_expert_ffn)
_STATUS = {0: "ok", 1: "invalid argument", 2: "shape or layout mismatch", 3: "non-finite router logit",
           4: "CUDA error", 5: "NCCL error", 6: "unsupported configuration", 7: "routing index out of range",
           8: "peer-exchange barrier timed out"}


class SmileError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {_STATUS.get(code, code)} ({code})")
        self.code = code


class Shape(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("e", C.c_int32), ("mode", C.c_int32),
                ("dtype", C.c_int32), ("d", C.c_int32), ("d_ff", C.c_int32), ("T", C.c_int64),
                ("cf", C.c_double), ("nprocs", C.c_int32), ("proc", C.c_int32), ("device", C.c_int32),
                ("ffn_impl", C.c_int32), ("topk", C.c_int32)]


class Sizes(C.Structure):
    _fields_ = [("G", C.c_int32), ("V", C.c_int32), ("rank0", C.c_int32), ("K1", C.c_int32),
                ("K2", C.c_int32), ("KW", C.c_int32), ("C1", C.c_int64), ("C2", C.c_int64),
                ("S", C.c_int32), ("Cseg", C.c_int64), ("ws_bytes", C.c_size_t), ("router_partial_bytes", C.c_size_t)]


_P = C.c_void_p


class Route(C.Structure):
    _fields_ = [(k, _P) for k in ("dest1", "dest2", "slot1", "p", "q", "gate")]


class Stats(C.Structure):
    _fields_ = [(k, _P) for k in ("hist1", "hist2", "psum1", "psum2")]


class Fabric(C.Structure):
    _fields_ = [("inter_gbps", C.c_double), ("inter_latency_us", C.c_double)]


class LayerIO(C.Structure):
    _fields_ = [("x", _P), ("logits", _P), ("w_router", _P), ("W1t", _P), ("b1", _P), ("W2t", _P),
                ("b2", _P), ("out", _P), ("loss", _P), ("alpha", C.c_double), ("beta", C.c_double),
                ("ws", _P), ("train", C.c_int32)]


class GradIO(C.Structure):
    _fields_ = [("gout", _P), ("dx", _P), ("dW_router", _P), ("W1", _P), ("W2", _P), ("dW1", _P), ("db1", _P),
                ("dW2", _P), ("db2", _P), ("lam", C.c_double)]


class WsView(C.Structure):
    _fields_ = [("route", Route), ("stats", Stats)] + [(k, _P) for k in (
        "counts1", "send1", "meta1", "recv1", "rmeta1", "slot2", "counts2", "send2", "recv2", "rcounts",
        "ffn_in", "H", "Y", "ret2", "ret1", "back1", "A1", "logits", "dlogits", "rpartial", "flags")]


def lib():
    """Load the in-tree libsmile.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2212_05191_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.smile_version.restype = C.c_int
        L.smile_strerror.restype = C.c_char_p
        L.smile_launch_count.restype = C.c_int64
        L.smile_capacity.restype = C.c_int64
        L.smile_capacity.argtypes = [C.c_int64, C.c_int64, C.c_double]
        for name in ("smile_plan", "smile_group", "smile_exchange_plan", "smile_get_unique_id", "smile_create", "smile_destroy",
                     "smile_query", "smile_get_error", "smile_gate_inter", "smile_dispatch", "smile_gate_intra",
                     "smile_all2all", "smile_all2all_inter", "smile_all2all_intra", "smile_expert_ffn",
                     "smile_combine", "smile_aux_loss", "smile_forward_ws", "smile_forward", "smile_forward_host",
                     "smile_gate_dispatch_inter",
                     "smile_expert_ffn_train", "smile_combine_bwd", "smile_dispatch_grad", "smile_expert_ffn_bwd",
                     "smile_combine_grad", "smile_router_bwd", "smile_backward", "smile_ipc_handle",
                     "smile_register_workspace", "smile_struct_sizes", "smile_forward_host_stream", "smile_set_output",
                     "smile_forward_chunked", "smile_set_fabric"):
            getattr(L, name).restype = C.c_int
        # the ctypes mirrors must match the C structs byte for byte
        sizes = (C.c_int64 * 8)()
        _check(L.smile_struct_sizes(sizes, 8), "smile_struct_sizes")
        mine = [C.sizeof(t) for t in (Shape, Sizes, Route, Stats, LayerIO, WsView, GradIO, XOp)]
        if list(sizes) != mine:
            raise ImportError(f"libsmile struct sizes {list(sizes)} != binding {mine}: rebuild or fix smile.py")
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        raise SmileError(rc, what)


def _shape(n, m, e, d, d_ff, T, cf, dtype, mode, nprocs=1, proc=0, device=0, ffn_impl=FFN_AUTO, topk=1) -> Shape:
    dt = {"fp32": FP32, "bf16": BF16}[dtype] if isinstance(dtype, str) else dtype
    md = {"bilevel": BILEVEL, "flat": FLAT}[mode] if isinstance(mode, str) else mode
    fi = {"auto": FFN_AUTO, "simt": FFN_SIMT, "tcgen05": FFN_TCGEN05}[ffn_impl] if isinstance(ffn_impl, str) else ffn_impl
    return Shape(n, m, e, md, dt, d, d_ff, T, cf, nprocs, proc, device, fi, topk)


def plan(**kw) -> Sizes:
    """Host-only size plan (no GPU needed): smile_plan."""
    z = Sizes()
    _check(lib().smile_plan(C.byref(_shape(**kw)), C.byref(z)), "smile_plan")
    return z


def capacity(T: int, dests: int, cf: float) -> int:
    """Host-only: ceil(cf*T/dests) per (sending rank, destination) (smile_capacity; -1 if invalid)."""
    return int(lib().smile_capacity(T, dests, cf))


def group(n: int, m: int, level: int, r: int) -> list[int]:
    """Host-only: members of rank r's group at level (1 inter, 2 intra, 0 world)."""
    sh = _shape(n, m, 1, 8, 8, 1, 1.0, "fp32", "bilevel")
    buf = (C.c_int32 * (n * m))()
    cnt = C.c_int32()
    _check(lib().smile_group(C.byref(sh), level, r, buf, C.byref(cnt)), "smile_group")
    return list(buf[: cnt.value])


class XOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("peer_proc", C.c_int32), ("src", C.c_int32), ("dst", C.c_int32),
                ("chunk", C.c_int32)]


def exchange_plan(level: int, **kw) -> list[tuple]:
    """Host-only: the (kind, peer_proc, src, dst, chunk) transfers smile_all2all posts
    for the cross-process pairs of `level` (smile_exchange_plan)."""
    sh = _shape(**kw)
    cnt = C.c_int32()
    lib().smile_exchange_plan(C.byref(sh), level, None, 0, C.byref(cnt))
    ops = (XOp * max(1, cnt.value))()
    _check(lib().smile_exchange_plan(C.byref(sh), level, ops, cnt.value, C.byref(cnt)), "smile_exchange_plan")
    return [(o.kind, o.peer_proc, o.src, o.dst, o.chunk) for o in ops[: cnt.value]]


def launch_count() -> int:
    """Kernels libsmile has launched so far in this process (smile_launch_count)."""
    return int(lib().smile_launch_count())


def unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().smile_get_unique_id(buf), "smile_get_unique_id")
    return bytes(buf)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


class SmileLayer:
    """One SMILE (or flat Switch) layer: G = n*m ranks, V = G/nprocs of them resident here.

    Buffers are torch tensors owned by the caller / this object; calls are asynchronous on
    the current torch stream."""

    def __init__(self, n, m, e, d, d_ff, T, cf=2.0, dtype="bf16", mode="bilevel", nprocs=1, proc=0,
                 device=None, ffn_impl="auto", nccl_id: bytes | None = None, topk: int = 1):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.shape = _shape(n, m, e, d, d_ff, T, cf, dtype, mode, nprocs, proc, self.device.index, ffn_impl, topk)
        self.topk = max(1, topk)
        self.n, self.m, self.e, self.d, self.d_ff, self.T, self.cf = n, m, e, d, d_ff, T, cf
        self.dtype = torch.bfloat16 if self.shape.dtype == BF16 else torch.float32
        self.flat = self.shape.mode == FLAT
        self._ctx = C.c_void_p()
        idbuf = None if nccl_id is None else (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        _check(lib().smile_create(C.byref(self._ctx), C.byref(self.shape), idbuf), "smile_create")
        self.sizes = Sizes()
        _check(lib().smile_query(self._ctx, C.byref(self.sizes)), "smile_query")
        z = self.sizes
        self.G, self.V, self.K1, self.K2, self.KW = z.G, z.V, z.K1, z.K2, z.KW
        self.C1, self.C2, self.S, self.Cseg = z.C1, z.C2, z.S, z.Cseg
        self.ws = None

    def close(self):
        if self._ctx:
            lib().smile_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- workspace ------------------------------------------------------------------
    def alloc_workspace(self):
        self.ws = torch.empty(self.sizes.ws_bytes + 256, dtype=torch.uint8, device=self.device)
        off = (-self.ws.data_ptr()) % 256
        self.ws = self.ws[off: off + self.sizes.ws_bytes]
        self._view = WsView()
        _check(lib().smile_forward_ws(self._ctx, _ptr(self.ws), C.byref(self._view)), "smile_forward_ws")
        return self.ws

    def enable_peer_exchange(self, allgather_bytes=None):
        """Register the workspace and switch smile_forward to the fused permute -> peer-store
        exchange (smile_register_workspace).  With several processes, `allgather_bytes(b)`
        must return the concatenation of every process's `b` in process order (e.g. over
        torch.distributed); all processes must barrier after this call."""
        if self.ws is None:
            self.alloc_workspace()
        buf = None
        if self.shape.nprocs > 1:
            h = (C.c_uint8 * 72)()
            _check(lib().smile_ipc_handle(self._ctx, _ptr(self.ws), h), "smile_ipc_handle")
            allh = allgather_bytes(bytes(h))
            buf = (C.c_uint8 * len(allh)).from_buffer_copy(allh)
        _check(lib().smile_register_workspace(self._ctx, _ptr(self.ws), buf, XCHG_PEER), "smile_register_workspace")

    def disable_peer_exchange(self):
        _check(lib().smile_register_workspace(self._ctx, _ptr(self.ws), None, XCHG_COPY), "smile_register_workspace")

    def _slice(self, addr, shape, dtype):
        nel = 1
        for s in shape:
            nel *= s
        nbytes = nel * torch.empty((), dtype=dtype).element_size()
        off = addr - self.ws.data_ptr()
        return self.ws[off: off + nbytes].view(dtype).view(shape)

    def view(self) -> dict:
        """Workspace buffers of the last forward as tensors (for inspection / tests)."""
        w, V, T = self._view, self.V, self.T
        i32, f32, f64, dt = torch.int32, torch.float32, torch.float64, self.dtype
        out = {k: self._slice(getattr(w.route, k), (V, T), i32 if k in ("dest1", "dest2", "slot1") else f32)
               for k in ("dest1", "dest2", "slot1", "p", "q", "gate")}
        if self.topk > 1:                     # choice-major [k, V, T] (smile.h smile_route)
            for k in ("dest1", "slot1", "gate"):
                out[k] = self._slice(getattr(w.route, k), (self.topk, V, T), i32 if k != "gate" else f32)
        out["hist1"] = self._slice(w.stats.hist1, (V, self.K1), i32)
        out["hist2"] = self._slice(w.stats.hist2, (V, self.K2), i32)
        out["psum1"] = self._slice(w.stats.psum1, (V, self.K1), f64)
        out["psum2"] = self._slice(w.stats.psum2, (V, self.K2), f64)
        out["counts1"] = self._slice(w.counts1, (V, self.K1), i32)
        out["rcounts"] = self._slice(w.rcounts, (V, self.S, self.e), i32)
        out["logits"] = self._slice(w.logits, (V, T, self.KW), f32)
        out["dlogits"] = self._slice(w.dlogits, (V, T, self.KW), f32)
        if not self.flat:
            out["rmeta1"] = self._slice(w.rmeta1, (V, self.n * self.C1), i32)
            out["slot2"] = self._slice(w.slot2, (V, self.n * self.C1), i32)
            out["counts2"] = self._slice(w.counts2, (V, self.K2), i32)
        return out

    # ---- the steps (C ABI) ------------------------------------------------------------
    def route_struct(self):
        return self._view.route

    def forward(self, x, W1t, b1, W2t, b2, out, loss, logits=None, w_router=None, alpha=0.005, beta=0.005,
                stream=None, train=False):
        if self.ws is None:
            self.alloc_workspace()
        io = LayerIO(_ptr(x), _ptr(logits), _ptr(w_router), _ptr(W1t), _ptr(b1), _ptr(W2t), _ptr(b2), _ptr(out),
                     _ptr(loss), alpha, beta, _ptr(self.ws), int(train))
        self._io = io
        _check(lib().smile_forward(self._ctx, C.byref(io), _stream(stream)), "smile_forward")

    def backward(self, gout, dx, W1, W2, dW1, db1, dW2, db2, dW_router=None, lam=1.0, stream=None):
        """smile_backward after forward(..., train=True) with the same buffers."""
        g = GradIO(_ptr(gout), _ptr(dx), _ptr(dW_router), _ptr(W1), _ptr(W2), _ptr(dW1), _ptr(db1), _ptr(dW2),
                   _ptr(db2), lam)
        _check(lib().smile_backward(self._ctx, C.byref(self._io), C.byref(g), _stream(stream)), "smile_backward")

    def forward_host(self, x_dev, host_x, W1t, b1, W2t, b2, out, loss, host_out, host_loss, logits=None,
                     host_logits=None, w_router=None, alpha=0.005, beta=0.005, stream=None):
        if self.ws is None:
            self.alloc_workspace()
        io = LayerIO(_ptr(x_dev), _ptr(logits), _ptr(w_router), _ptr(W1t), _ptr(b1), _ptr(W2t), _ptr(b2),
                     _ptr(out), _ptr(loss), alpha, beta, _ptr(self.ws), 0)
        _check(lib().smile_forward_host(self._ctx, C.byref(io), _ptr(host_x), _ptr(host_logits), _ptr(host_out),
                                        _ptr(host_loss), _stream(stream)), "smile_forward_host")

    def forward_host_stream(self, x_dev2, out_dev2, host_xs, host_outs, host_loss, W1t, b1, W2t, b2, loss,
                            w_router=None, alpha=0.005, beta=0.005, stream=None):
        """smile_forward_host_stream: len(host_xs) batches from pinned host memory with the
        H2D / layer / D2H of consecutive batches overlapped.  x_dev2, out_dev2: two device
        buffers each; host_loss: pinned float64 [nb, V]."""
        if self.ws is None:
            self.alloc_workspace()
        io = LayerIO(0, 0, _ptr(w_router), _ptr(W1t), _ptr(b1), _ptr(W2t), _ptr(b2), 0, _ptr(loss), alpha, beta,
                     _ptr(self.ws), 0)
        nb = len(host_xs)
        P2 = C.c_void_p * 2
        PN = C.c_void_p * max(nb, 1)
        xd = P2(*[_ptr(t) for t in x_dev2])
        od = P2(*[_ptr(t) for t in out_dev2])
        hx = PN(*[_ptr(t) for t in host_xs])
        ho = PN(*[_ptr(t) for t in host_outs])
        _check(lib().smile_forward_host_stream(self._ctx, C.byref(io), xd, od, nb, hx, ho, _ptr(host_loss),
                                               _stream(stream)), "smile_forward_host_stream")

    def set_fabric(self, inter_gbps: float, inter_latency_us: float):
        """smile_set_fabric: the emulated inter-node fabric of the COPY exchange (SURVEY 8(f)
        row 1; an in-box emulation).  inter_gbps <= 0 disables it."""
        f = Fabric(float(inter_gbps), float(inter_latency_us))
        _check(lib().smile_set_fabric(self._ctx, C.byref(f)), "smile_set_fabric")

    def set_output(self, out):
        """smile_set_output: bind the layer output for the following step calls (None unbinds)."""
        _check(lib().smile_set_output(self._ctx, _ptr(out)), "smile_set_output")

    def get_error(self, stream=None) -> int:
        return lib().smile_get_error(self._ctx, _stream(stream))

    # individual steps, same names as the C ABI ------------------------------------------
    def gate_inter(self, x, route, stats, counts1, w_router=None, logits=None, logits_out=None, stream=None):
        _check(lib().smile_gate_inter(self._ctx, _ptr(x), _ptr(w_router), _ptr(logits), _ptr(logits_out),
                                      C.byref(route), C.byref(stats), _ptr(counts1), _stream(stream)),
               "smile_gate_inter")

    def gate_dispatch_inter(self, x, w_router, route, stats, counts1, send_rows, send_meta=None, logits_out=None,
                            stream=None):
        """smile_gate_dispatch_inter: a1-a4 fused (tensor-core gate + level-1 permute)."""
        _check(lib().smile_gate_dispatch_inter(self._ctx, _ptr(x), _ptr(w_router), _ptr(logits_out), C.byref(route),
                                               C.byref(stats), _ptr(counts1), _ptr(send_rows), _ptr(send_meta),
                                               _stream(stream)), "smile_gate_dispatch_inter")

    def dispatch(self, level, rows_in, send_rows, route=None, recv_meta=None, slot2=None, send_meta=None,
                 stream=None):
        _check(lib().smile_dispatch(self._ctx, level, _ptr(rows_in), None if route is None else C.byref(route),
                                    _ptr(recv_meta), _ptr(slot2), _ptr(send_rows), _ptr(send_meta),
                                    _stream(stream)), "smile_dispatch")

    def gate_intra(self, recv_meta, slot2, counts2, stream=None):
        _check(lib().smile_gate_intra(self._ctx, _ptr(recv_meta), _ptr(slot2), _ptr(counts2), _stream(stream)),
               "smile_gate_intra")

    def all2all(self, level, reverse, send_rows, recv_rows, send_ints=None, recv_ints=None, fwd_counts=None,
                stream=None):
        _check(lib().smile_all2all(self._ctx, level, int(reverse), _ptr(send_rows), _ptr(recv_rows),
                                   _ptr(send_ints), _ptr(recv_ints), _ptr(fwd_counts), _stream(stream)),
               "smile_all2all")

    def all2all_inter(self, reverse, send_rows, recv_rows, send_meta=None, recv_meta=None, fwd_counts=None,
                      stream=None):
        _check(lib().smile_all2all_inter(self._ctx, int(reverse), _ptr(send_rows), _ptr(recv_rows), _ptr(send_meta),
                                         _ptr(recv_meta), _ptr(fwd_counts), _stream(stream)), "smile_all2all_inter")

    def all2all_intra(self, reverse, send_rows, recv_rows, send_cnt=None, recv_cnt=None, fwd_counts=None,
                      stream=None):
        _check(lib().smile_all2all_intra(self._ctx, int(reverse), _ptr(send_rows), _ptr(recv_rows), _ptr(send_cnt),
                                         _ptr(recv_cnt), _ptr(fwd_counts), _stream(stream)), "smile_all2all_intra")

    def expert_ffn(self, X, counts, W1t, b1, W2t, b2, H, Y, stream=None):
        _check(lib().smile_expert_ffn(self._ctx, _ptr(X), _ptr(counts), _ptr(W1t), _ptr(b1), _ptr(W2t), _ptr(b2),
                                      _ptr(H), _ptr(Y), _stream(stream)), "smile_expert_ffn")

    def combine(self, level, ret_rows, out, route=None, recv_meta=None, slot2=None, stream=None):
        _check(lib().smile_combine(self._ctx, level, _ptr(ret_rows), None if route is None else C.byref(route),
                                   _ptr(recv_meta), _ptr(slot2), _ptr(out), _stream(stream)), "smile_combine")

    def aux_loss(self, stats, loss, alpha=0.005, beta=0.005, stream=None):
        _check(lib().smile_aux_loss(self._ctx, C.byref(stats), C.c_double(alpha), C.c_double(beta), _ptr(loss),
                                    _stream(stream)), "smile_aux_loss")


def forward_chunked(layers, xs, W1t, b1, W2t, b2, outs, losses, w_router=None, logits=None, alpha=0.005, beta=0.005,
                    stream=None, stream2=None):
    """smile_forward_chunked: the layer over len(layers) chunks pipelined on two streams.
    layers[k]: a SmileLayer per chunk (T = tokens per chunk, same shape otherwise), xs[k] /
    outs[k]: [V, T/c, d] chunk inputs / outputs, losses[k]: [V] float64; logits (supplied
    mode) a list of per-chunk logits or None."""
    n = len(layers)
    for L in layers:
        if L.ws is None:
            L.alloc_workspace()
    Ctxs = C.c_void_p * n
    IOs = LayerIO * n
    ctxs = Ctxs(*[L._ctx for L in layers])
    ios = IOs(*[LayerIO(_ptr(xs[k]), _ptr(None if logits is None else logits[k]), _ptr(w_router), _ptr(W1t), _ptr(b1),
                        _ptr(W2t), _ptr(b2), _ptr(outs[k]), _ptr(losses[k]), alpha, beta, _ptr(layers[k].ws), 0)
                for k in range(n)])
    if stream2 is None:
        raise ValueError("forward_chunked needs a second stream")
    _check(lib().smile_forward_chunked(ctxs, ios, n, _stream(stream), _stream(stream2)), "smile_forward_chunked")
