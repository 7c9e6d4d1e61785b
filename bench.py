#!/usr/bin/env python
"""Benchmark of the SMILE bi-level MoE layer (and the flat Switch layer beside it).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--mode both|bilevel|flat]
                    [--config c2|c1|c4|c5] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): one MoE layer forward, G = 8 ranks as a 2x4
hierarchy (n = 2 groups x m = 4 ranks), 1 expert per rank, T = 16384 tokens per rank,
d = 768, d_ff = 3072, bf16, capacity factor 2.0, fused router (a1) on synthetic
N(0,1) tokens with random-init weights.  The job always runs the 8-rank problem:
N processes each drive V = 8/N ranks (N = 1 emulates all 8 ranks on one B200, the
exchanges becoming device copies; N = 8 is one rank per GPU with NCCL all-to-alls on
the split inter/intra communicators), so total work is fixed: "scaling": "strong".

A step = one pass of the whole hot path over one batch.  value =
G*T / (max over ranks of the device time of the step), inputs resident in HBM; L2 is
flushed before every timed step, outside its events: a 256 MiB write, then a 256 MiB read of
another buffer (``--flush write+read``, the default), so the write-back of the flush's own
dirty lines is finished before the step starts instead of being charged to the step's
first kernel (``--flush write`` keeps the plain write).  e2e = the same
metric through smile_forward_host with pinned host buffers (H2D of x and D2H of the
output and loss inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # tag: n, m, e, T (per rank), d, d_ff, cf, dtype
    "c1": dict(n=2, m=4, e=1, T=1024, d=64, d_ff=256, cf=1.0, dtype="fp32"),
    "c2": dict(n=2, m=4, e=1, T=16384, d=768, d_ff=3072, cf=2.0, dtype="bf16"),
    "c3": dict(n=2, m=4, e=1, T=32768, d=768, d_ff=3072, cf=1.25, dtype="bf16", train=True),
    "c3_4x2": dict(n=4, m=2, e=1, T=32768, d=768, d_ff=3072, cf=1.25, dtype="bf16", train=True),
    "c4": dict(n=2, m=4, e=8, T=65536, d=1024, d_ff=4096, cf=2.0, dtype="bf16"),
    "c5": dict(n=2, m=4, e=16, T=8192, d=1600, d_ff=6400, cf=2.0, dtype="bf16"),
    # multi-node topologies emulated on one B200 for the emulated-fabric runs (--fabric; the
    # paper's nodes x GPUs, P:L287 -- 32 ranks, the most the flat layer's 1024 FFN segments
    # allow): C2's widths with 4K tokens per rank, and C1's
    "e4x8": dict(n=4, m=8, e=1, T=4096, d=768, d_ff=3072, cf=2.0, dtype="bf16"),
    "e8x4": dict(n=8, m=4, e=1, T=4096, d=768, d_ff=3072, cf=2.0, dtype="bf16"),
    "e4x8_c1": dict(n=4, m=8, e=1, T=1024, d=64, d_ff=256, cf=1.0, dtype="fp32"),
}
METRIC = "MoE-layer tokens/sec (bi-level vs flat All2All) at 1/2/4/8 B200; kernel HBM GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="both", choices=["both", "bilevel", "flat"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--ffn", default="auto", choices=["auto", "simt", "tcgen05"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--graph", action="store_true", help="replay each step as a CUDA graph")
    ap.add_argument("--fused-gate", action="store_true",
                    help="gate + level-1 permute as one call (smile_gate_dispatch_inter); default: two calls")
    ap.add_argument("--chunks", type=int, default=1,
                    help="> 1: the layer as c pipelined micro-batches on two streams (SURVEY 8(f) row 2)")
    ap.add_argument("--clock-ms", type=int, default=50, help="nvidia-smi sampling period (0 = off)")
    ap.add_argument("--fabric", default=None,
                    help="GBPS,LATENCY_US: emulated inter-node fabric (smile_set_fabric; SURVEY 8(f) row 1, an in-box "
                         "emulation) on the COPY exchange, N = 1 only")
    ap.add_argument("--topk", type=int, default=1,
                    help="experts per token of the FLAT layer (Eq. 2; SURVEY 8(f) row 4); the bi-level layer is top-1")
    ap.add_argument("--flush", default="write+read", choices=["write+read", "write"],
                    help="L2 flush between timed steps (write+read: drain the flush's dirty lines)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "copy"],
                    help="peer: fused permute -> peer-store exchange (CUDA IPC over NVLink); copy: device copies / NCCL")
    return ap.parse_args()


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi samples of SM clock and throttle reasons during the timed region."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 100):
        self.index, self.proc, self.lines, self.period = index, None, [], period_ms

    def start(self):
        """Start nvidia-smi (writing to a file, no reader thread here) and wait for its first
        sample: NVML initialisation stalls CUDA work of the process for up to ~1 s, so it
        must be done before the timed region, never inside it."""
        import tempfile
        try:
            self.path = tempfile.mktemp(prefix="smile_clocks_", suffix=".csv")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period), "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            t0 = time.time()
            while time.time() - t0 < 10:
                if os.path.exists(self.path) and os.path.getsize(self.path) > 0:
                    break
                time.sleep(0.05)
            time.sleep(2 * self.period / 1000.0)
        except Exception:
            self.proc = None

    def mark(self, which: str):
        setattr(self, which, time.time())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        try:
            with open(self.path) as f:
                self.lines = [ln.strip() for ln in f]
            os.remove(self.path)
        except Exception:
            self.lines = []
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        import datetime
        t_beg, t_end = getattr(self, "t_beg", 0.0), getattr(self, "t_end", 1e18)
        rows = []
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(p[1]), float(p[2]), p[3:7]))
            except ValueError:
                continue
        inside = [r for r in rows if t_beg - 0.05 <= r[0] <= t_end + 0.05]
        window = "timed region"
        if not inside and rows:           # region shorter than the sampling period: nearest samples
            inside = sorted(rows, key=lambda r: min(abs(r[0] - t_beg), abs(r[0] - t_end)))[:2]
            window = "nearest samples to a timed region shorter than the sampling period"
        for ts, a, b, rs in inside:
            sm.append(a)
            mx.append(b)
            for nm, v in zip(names, rs):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "window": window, "period_ms": self.period}


# --------------------------------------------------------------------------- reference arm
def _oracle_step_fn(cfgd, mode, Ts, seed=0):
    """One step of the CPU oracle (oracle/, as it stands: the serial fp64 functions, one
    thread) on a bounded sample of the workload: the whole layer -- router logits (Eq. 1),
    bi-level (or flat) routing with capacities (Eq. 3, R5-R8), the expert FFN of every
    kept token and the gate-weighted output (Eq. 3), the aux loss (Eq. 4) -- on a mini-batch
    of Ts tokens per rank with the configuration's n, m, e, d, d_ff and cf.  Inputs are
    generated outside the timed call.  Returns (fn, tokens per step)."""
    import numpy as np
    import oracle
    import synth
    n, m, e, d, d_ff, cf = (cfgd[k] for k in ("n", "m", "e", "d", "d_ff", "cf"))
    flat = mode == "flat"
    G = n * m
    cfg = oracle.Config(n, m, e, Ts, cf, flat=flat, alpha=0.01 if flat else 0.005)
    KW = cfg.logit_width
    x = synth.tokens(G, Ts, d, seed=seed, dtype=cfgd["dtype"])
    W = synth.router_weights(KW, d, seed=seed)
    W1, b1, W2, b2 = synth.expert_weights(G * e, d, d_ff, seed=seed, dtype=cfgd["dtype"], bias=False)

    def fn():
        lg = oracle.logits(x.reshape(-1, d), W).reshape(G, Ts, KW)
        r = oracle.route(cfg, lg)
        return oracle.out_rows(cfg, r, x, W1, b1, W2, b2)
    return fn, G * Ts


def _oracle_sample_size(cfgd, mode, per_step_s):
    """Tokens per rank of the oracle's mini-batch so that one step takes ~per_step_s: the
    per-token cost is calibrated on an 8-token-per-rank step (the cost is linear in the
    tokens: logits, routing and the FFN are per token)."""
    fn, tok = _oracle_step_fn(cfgd, mode, 8)
    t0 = time.perf_counter()
    fn()
    per_tok = (time.perf_counter() - t0) / tok
    G = cfgd["n"] * cfgd["m"]
    return max(1, min(cfgd["T"], int(per_step_s / (per_tok * G)))), per_tok


def cpu_oracle_sample(cfgd, mode, seconds_budget=15.0):
    """cpu_baseline of our arm (rank 0, N = 1): the oracle as it stands timed on the host
    cores over a bounded sample -- a few whole-layer steps on a mini-batch (see
    _oracle_step_fn), ~seconds_budget of CPU work; value = tokens per second measured, no
    extrapolation."""
    Ts, _ = _oracle_sample_size(cfgd, mode, seconds_budget / 3)
    fn, tok = _oracle_step_fn(cfgd, mode, Ts, seed=1)
    times = []
    t_all = time.perf_counter()
    while len(times) < 3 and time.perf_counter() - t_all < seconds_budget:
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": tok / t, "unit": "tokens/s", "cores": 1, "nproc": os.cpu_count(), "kind": "oracle",
            "sample": f"{len(times)} whole-layer oracle steps (logits + routing + FFN of every kept token + loss) "
                      f"on a mini-batch of {Ts} tokens/rank x {cfgd['n'] * cfgd['m']} ranks with the workload's "
                      f"n, m, e, d, d_ff, cf; median {t:.2f} s per step; single thread (serial fp64 oracle)"}


def run_reference(args):
    """The reference arm: for this tier the CPU oracle (oracle/, as it stands) on the box's
    host cores -- rank 0 only.  Each step = the whole oracle layer on a bounded mini-batch
    of the same workload (_oracle_step_fn), sized so --warmup + --steps steps take about
    90 s; the measured median step time gives the tokens/s (no extrapolation)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfgd = CONFIGS[args.config]
    mode = "bilevel" if args.mode in ("both", "bilevel") else "flat"
    n_steps = args.warmup + args.steps
    Ts, per_tok = _oracle_sample_size(cfgd, mode, 90.0 / max(1, n_steps))
    fn, tok = _oracle_step_fn(cfgd, mode, Ts)
    times = []
    t_wall = time.perf_counter()
    for it in range(n_steps):
        t0 = time.perf_counter()
        fn()
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    wall = time.perf_counter() - t_wall
    t = statistics.median(times)
    value = tok / t
    G = cfgd["n"] * cfgd["m"]
    q = statistics.quantiles(times, n=10) if len(times) >= 2 else [t] * 9
    sample = (f"per step: the whole oracle layer (router logits, routing with capacities, FFN of every kept token, "
              f"gate-weighted output, aux loss) on a mini-batch of {Ts} tokens/rank x {G} ranks with the workload's "
              f"n, m, e, d, d_ff, cf (the full layer has T={cfgd['T']}/rank); single thread")
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: one SMILE {mode} layer fwd, {G} ranks {cfgd['n']}x{cfgd['m']}, "
                                   f"e={cfgd['e']}, d={cfgd['d']}, d_ff={cfgd['d_ff']}, cf={cfgd['cf']}; CPU oracle "
                                   f"mini-batch of {Ts} tokens/rank per step", "l2": "n/a (CPU)"},
            "step_ms": {"median": t * 1e3, "p10": q[0] * 1e3, "p90": q[-1] * 1e3, "mean": statistics.mean(times) * 1e3},
            "wall_s": wall,
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "nproc": os.cpu_count(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
PHASES_BI = ["gate1", "dispatch1", "a2a_inter", "gate2", "dispatch2", "a2a_intra", "ffn", "a2a_intra_rev",
             "combine2", "a2a_inter_rev", "combine1", "aux"]
PHASES_FLAT = ["gate1", "dispatch1", "a2a_world", "ffn", "a2a_world_rev", "combine1", "aux"]


class Addr:
    def __init__(self, a):
        self.a = a

    def data_ptr(self):
        return self.a


class L2Flush:
    """Empties L2 between timed steps.  Writing 256 MiB (2x the 126 MB L2) evicts every line
    of the step's data but leaves L2 full of DIRTY lines of the flush buffer, whose write-back
    to DRAM would otherwise overlap (and be charged to) the next step's first kernel; a read
    of another 256 MiB buffer after the write drains them, so each step starts from an L2
    that holds neither its data nor pending write-backs."""

    def __init__(self, dev, how):
        import torch
        self.how = how
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        self.r = torch.ones(32 << 20, dtype=torch.int64, device=dev) if how == "write+read" else None
        self.sink = torch.empty(1, dtype=torch.int64, device=dev)

    def __call__(self):
        import torch
        self.w.zero_()
        if self.r is not None:
            torch.sum(self.r, dim=(0,), out=self.sink[0])

    def describe(self):
        return ("flushed (256 MiB write + 256 MiB read of another buffer) before every timed step, "
                "outside its events" if self.how == "write+read" else
                "flushed (256 MiB write) before every timed step, outside its events")


def make_layer(cfgd, mode, nprocs, proc, dev, ffn, nccl_id, topk=1):
    from paper_2212_05191_b200 import SmileLayer
    L = SmileLayer(cfgd["n"], cfgd["m"], cfgd["e"], cfgd["d"], cfgd["d_ff"], cfgd["T"], cfgd["cf"], cfgd["dtype"],
                   mode, nprocs=nprocs, proc=proc, device=dev, ffn_impl=ffn, nccl_id=nccl_id,
                   topk=topk if mode == "flat" else 1)
    L.alloc_workspace()
    return L


def step(L, inp, ev=None):
    """One forward through the C-ABI steps (the sequence of smile_forward), with an event
    recorded after each phase when `ev` is given."""
    import torch
    w = L._view
    A = lambda p: Addr(p)
    rec = (lambda i: ev[i].record()) if ev is not None else (lambda i: None)
    rec(0)
    if inp.get("fused_gate"):
        # a1-a4 in one tensor-core kernel (smile_gate_dispatch_inter); "dispatch1" is empty
        L.gate_dispatch_inter(inp["x"], inp["w_router"], w.route, w.stats, A(w.counts1), A(w.send1),
                              send_meta=A(w.meta1) if not L.flat else None)
        rec(1)
    else:
        L.gate_inter(inp["x"], w.route, w.stats, A(w.counts1), w_router=inp["w_router"])
        rec(1)
        L.dispatch(1, inp["x"], A(w.send1), route=w.route, send_meta=A(w.meta1) if not L.flat else None)
    rec(2)
    if not L.flat:
        L.all2all_inter(0, A(w.send1), A(w.recv1), A(w.meta1), A(w.rmeta1), A(w.counts1))
        rec(3)
        L.gate_intra(A(w.rmeta1), A(w.slot2), A(w.counts2))
        rec(4)
        L.dispatch(2, A(w.recv1), A(w.send2), recv_meta=A(w.rmeta1), slot2=A(w.slot2))
        rec(5)
        L.all2all_intra(0, A(w.send2), A(w.recv2), A(w.counts2), A(w.rcounts), A(w.counts2))
        rec(6)
        L.expert_ffn(A(w.recv2), A(w.rcounts), inp["W1t"], inp["b1"], inp["W2t"], inp["b2"], A(w.H), A(w.Y))
        rec(7)
        L.all2all_intra(1, A(w.Y), A(w.ret2), fwd_counts=A(w.counts2))
        rec(8)
        L.combine(2, A(w.ret2), A(w.ret1), recv_meta=A(w.rmeta1), slot2=A(w.slot2))
        rec(9)
        L.all2all_inter(1, A(w.ret1), A(w.back1), fwd_counts=A(w.counts1))
        rec(10)
        L.combine(1, A(w.back1), inp["out"], route=w.route)
        rec(11)
        L.aux_loss(w.stats, inp["loss"], 0.005, 0.005)
        rec(12)
    else:
        L.all2all(0, 0, A(w.send1), A(w.recv1), A(w.counts1), A(w.rcounts), A(w.counts1))
        rec(3)
        L.expert_ffn(A(w.recv1), A(w.rcounts), inp["W1t"], inp["b1"], inp["W2t"], inp["b2"], A(w.H), A(w.Y))
        rec(4)
        L.all2all(0, 1, A(w.Y), A(w.back1), fwd_counts=A(w.counts1))
        rec(5)
        L.combine(1, A(w.back1), inp["out"], route=w.route)
        rec(6)
        L.aux_loss(w.stats, inp["loss"], 0.01, 0.0)
        rec(7)


def run_pipelined(args):
    """SURVEY 8(f) row 2 / P:L391-405: smile_forward_chunked -- the layer over c chunks of
    T/c tokens per rank (each chunk its own capacities), the FFN of chunk k on a second
    stream overlapping the front of chunk k+1 and the back of chunk k-1 -- timed beside
    the unchunked layer (smile_forward) in the same run, same inputs."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2212_05191_b200 import smile as smb
    cfgd = dict(CONFIGS[args.config])
    G, c = cfgd["n"] * cfgd["m"], args.chunks
    V, T, d, d_ff, e = G // world, cfgd["T"], cfgd["d"], cfgd["d_ff"], cfgd["e"]
    if T % c:
        raise SystemExit(f"T={T} not divisible into {c} chunks")
    Tc = T // c
    tdt = torch.bfloat16 if cfgd["dtype"] == "bf16" else torch.float32
    modes = ["bilevel", "flat"] if args.mode == "both" else [args.mode]
    flush = L2Flush(dev, args.flush)

    def new_layer(ck, mode):
        nid = None
        if world > 1:
            buf = torch.zeros(128, dtype=torch.uint8, device=dev)
            if rank == 0:
                buf.copy_(torch.frombuffer(bytearray(smb.unique_id()), dtype=torch.uint8))
            dist.broadcast(buf, 0)
            nid = bytes(buf.cpu().numpy().tobytes())
        L = make_layer(ck, mode, world, rank, local, args.ffn, nid)

        def allgather(b):
            t = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(dev)
            outs = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(outs, t)
            return b"".join(bytes(o.cpu().numpy().tobytes()) for o in outs)
        L.enable_peer_exchange(allgather if world > 1 else None)
        if dist:
            dist.barrier()
        return L

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        t0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        t1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush()
            t0[k].record()
            fn()
            t1[k].record()
        torch.cuda.synchronize()
        ms = torch.tensor([statistics.median(t0[k].elapsed_time(t1[k]) for k in range(args.steps))],
                          dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return ms.item()

    out_modes, base_modes = {}, {}
    for mode in modes:
        Ls = [new_layer(dict(cfgd, T=Tc), mode) for _ in range(c)]
        Lfull = new_layer(cfgd, mode)
        KW = Ls[0].KW
        gen = torch.Generator(device=dev)
        gen.manual_seed(7)
        w_router = (torch.rand(KW, d, generator=gen, device=dev) * 2 - 1) / math.sqrt(d)
        gen.manual_seed(2000 + rank)
        W1t = ((torch.rand(V * e, d_ff, d, generator=gen, device=dev) * 2 - 1) / math.sqrt(d)).to(tdt)
        W2t = ((torch.rand(V * e, d, d_ff, generator=gen, device=dev) * 2 - 1) / math.sqrt(d_ff)).to(tdt)
        b1 = torch.zeros(V * e, d_ff, device=dev)
        b2 = torch.zeros(V * e, d, device=dev)
        gen.manual_seed(1000 + rank)
        x = torch.randn(V, T, d, generator=gen, device=dev, dtype=torch.float32).to(tdt)
        xs = [x[:, k * Tc:(k + 1) * Tc].contiguous() for k in range(c)]
        outs = [torch.empty_like(xk) for xk in xs]
        losses = [torch.empty(V, dtype=torch.float64, device=dev) for _ in range(c)]
        out_full = torch.empty_like(x)
        loss_full = torch.empty(V, dtype=torch.float64, device=dev)
        s2 = torch.cuda.Stream()
        a_, b_ = (0.005, 0.005) if mode == "bilevel" else (0.01, 0.0)
        out_modes[mode] = timed(lambda: smb.forward_chunked(Ls, xs, W1t, b1, W2t, b2, outs, losses, w_router=w_router,
                                                            alpha=a_, beta=b_, stream2=s2))
        base_modes[mode] = timed(lambda: Lfull.forward(x, W1t, b1, W2t, b2, out_full, loss_full, w_router=w_router,
                                                       alpha=a_, beta=b_))
        if any(L.get_error() for L in Ls + [Lfull]):
            raise SystemExit("device error")
        if dist:
            dist.barrier()
        for L in Ls + [Lfull]:
            L.close()
    if rank == 0:
        m0 = modes[0]
        line = {"metric": METRIC, "value": G * T / (out_modes[m0] / 1e3), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": out_modes[m0], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16" if cfgd["dtype"] == "bf16" else "f32",
                "data": "synthetic", "config": {"workload": f"{args.config}: {m0} layer fwd through smile_forward_chunked, "
                                                            f"{c} pipelined chunks of T={Tc}/rank on 2 streams (SURVEY 8(f) row 2)",
                                                 "chunks": c, "exchange": "peer", "timing": "median over steps",
                                                 "l2": flush.describe()},
                "chunked_ms": out_modes, "unchunked_ms": base_modes,
                "chunked_over_unchunked": {k: base_modes[k] / out_modes[k] for k in out_modes}}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


PHASES_TRAIN = ["fwd", "bwd"]


def step_train(L, inp, ev=None):
    """C3: one training step of the layer -- smile_forward(train) then smile_backward
    (a16-a19), the router gradient included."""
    rec = (lambda i: ev[i].record()) if ev is not None else (lambda i: None)
    rec(0)
    L.forward(inp["x"], inp["W1t"], inp["b1"], inp["W2t"], inp["b2"], inp["out"], inp["loss"],
              w_router=inp["w_router"], alpha=inp["alpha"], beta=inp["beta"], train=True)
    rec(1)
    L.backward(inp["gout"], inp["dx"], inp["W1"], inp["W2"], inp["dW1"], inp["db1"], inp["dW2"], inp["db2"],
               dW_router=inp["dWr"])
    rec(2)


def hbm_phases(res, peaks):
    """Achieved HBM GB/s of the HBM-bound phases (per process, max-over-ranks phase time):
    algorithmic bytes / phase time, against MEASURED_PEAKS.json hbm_gbs.  A phase's time
    includes its small side kernels (scan, meta fill), so the fraction is a lower bound
    for the row kernel itself."""
    peak = peaks.get("hbm_gbs")
    out = {}
    for ph, b in res["hbm_bytes"].items():
        t = res["phase_ms"].get(ph)
        if not t or not b:
            if ph in res["phase_ms"] and not b:
                out[ph] = {"bytes": 0, "ms": t, "note": "no rows to move (fused into the FFN's GEMM 2)"}
            continue
        gbs = b / (t / 1e3) / 1e9
        out[ph] = {"bytes": b, "ms": t, "GB/s": gbs, "frac": gbs / peak if peak else None}
    out["peak_GB/s"] = peak
    out["peak_source"] = "MEASURED_PEAKS.json hbm_gbs"
    return out


def nvlink_levels(res, world, mode, exchange):
    """Per exchange level: bytes this process sends to other GPUs in one direction
    (valid rows only; the reverse path moves the same bytes back) and the achieved
    NVLink GB/s over the phases that carry them.  PEER: the permute / combine kernels
    store / load remote rows, so a level's time is its mover phase plus its barrier;
    COPY: the NCCL all-to-all phase (which moves capacity-padded chunks)."""
    if world == 1:
        return None
    ph = res["phase_ms"]
    if mode == "bilevel":
        legs = {"inter": (("dispatch1", "a2a_inter"), ("combine1", "a2a_inter_rev")),
                "intra": (("dispatch2", "a2a_intra"), ("combine2", "a2a_intra_rev"))}
    else:
        legs = {"world": (("dispatch1", "a2a_world"), ("combine1", "a2a_world_rev"))}
    out = {}
    for lvl, (fwd, rev) in legs.items():
        b = res["nvl_bytes"].get(lvl, 0)
        tf = sum(ph[p] for p in fwd) if exchange == "peer" else ph[fwd[1]]
        tr = sum(ph[p] for p in rev) if exchange == "peer" else ph[rev[1]]
        out[lvl] = {"bytes_per_direction": b, "fwd_ms": tf, "rev_ms": tr,
                    "fwd_GB/s": b / (tf / 1e3) / 1e9 if tf else None, "rev_GB/s": b / (tr / 1e3) / 1e9 if tr else None}
    out["note"] = ("rank-0 process, valid rows only; peer: mover + barrier phases, copy: NCCL phase; "
                   "measured NVLink reference 770 GB/s per direction (B200_PROFILING.md)")
    return out


def layer_roofline(res, cfgd, peaks, world, flops):
    """layer time bound = HBM bytes / HBM peak + NVLink bytes / 770 GB/s +
    FFN flops / bf16 peak (serial) or max(HBM + NVLink, FFN) (perfect overlap), per
    process; tokens/s of the whole job = G*T / that time."""
    hbm_b = sum(res["hbm_bytes"].values())
    nvl_b = 2 * sum(res["nvl_bytes"].values()) if world > 1 else 0
    t_h = hbm_b / (peaks.get("hbm_gbs", 6449.1) * 1e9)
    t_n = nvl_b / 770e9
    t_f = flops / (peaks.get("bf16_tflops", 1620.5) * 1e12)
    ser, ovl = t_h + t_n + t_f, max(t_h + t_n, t_f)
    tok = res["tokens"]
    return {"t_hbm_ms": t_h * 1e3, "t_nvlink_ms": t_n * 1e3, "t_ffn_ms": t_f * 1e3,
            "serial_tokens_per_s": tok / ser, "overlap_tokens_per_s": tok / ovl,
            "frac_serial": (tok / (res["ms"] / 1e3)) / (tok / ser), "frac_overlap": (tok / (res["ms"] / 1e3)) / (tok / ovl),
            "note": "per process (max over ranks of the measured step); HBM bytes as hbm_phases, FFN flops as roofline"}


def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world if world > 1 else args.gpus
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfgd = CONFIGS[args.config]
    G = cfgd["n"] * cfgd["m"]
    if G % world:
        raise SystemExit(f"{world} processes do not divide {G} ranks")
    from paper_2212_05191_b200 import smile as smb
    nccl_id = None
    if world > 1:
        buf = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(smb.unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())

    modes = ["bilevel", "flat"] if args.mode == "both" else [args.mode]
    fabric = None
    if args.fabric:
        if world != 1:
            raise SystemExit("--fabric emulates every rank's NIC on one GPU: N = 1 only")
        bw, lat = (float(v) for v in args.fabric.split(","))
        fabric = {"inter_gbps_per_rank": bw, "inter_latency_us_per_message": lat, "emulated": True}
        args.exchange = "copy"
    if args.fused_gate:
        # smile_gate_dispatch_inter is the 128-token tensor-core gate (it refuses the
        # default swapped 256-token tile with SMILE_ENOTSUP): select that tile
        os.environ["SMILE_GATE_SWAP"] = "0"
    V = G // world
    T, d, d_ff, e = cfgd["T"], cfgd["d"], cfgd["d_ff"], cfgd["e"]
    tdt = torch.bfloat16 if cfgd["dtype"] == "bf16" else torch.float32
    gen = torch.Generator(device=dev)
    results = {}
    flush = L2Flush(dev, args.flush)
    sampler = ClockSampler(local, args.clock_ms) if rank == 0 and args.clock_ms > 0 else None
    if sampler:
        sampler.start()
    for mode in modes:
        # the two layers are measured one after the other; the second gets its own id
        if mode != modes[0] and world > 1:
            buf = torch.zeros(128, dtype=torch.uint8, device=dev)
            if rank == 0:
                buf.copy_(torch.frombuffer(bytearray(smb.unique_id()), dtype=torch.uint8))
            dist.broadcast(buf, 0)
            nccl_id = bytes(buf.cpu().numpy().tobytes())
        L = make_layer(cfgd, mode, world, rank, local, args.ffn, nccl_id, topk=args.topk)
        if fabric:
            L.set_fabric(fabric["inter_gbps_per_rank"], fabric["inter_latency_us_per_message"])
        if args.exchange == "peer":
            def allgather(b):
                t = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(dev)
                outs = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(outs, t)
                return b"".join(bytes(o.cpu().numpy().tobytes()) for o in outs)
            L.enable_peer_exchange(allgather if world > 1 else None)
            if dist:
                dist.barrier()
        KW = L.KW
        gen.manual_seed(1000 + rank)
        x = torch.randn(V, T, d, generator=gen, device=dev, dtype=torch.float32).to(tdt)
        gen.manual_seed(7)                                     # tied router: same on every rank
        bw = 1.0 / math.sqrt(d)
        w_router = (torch.rand(KW, d, generator=gen, device=dev) * 2 - 1) * bw
        gen.manual_seed(2000 + rank)
        W1t = ((torch.rand(V * e, d_ff, d, generator=gen, device=dev) * 2 - 1) / math.sqrt(d)).to(tdt)
        W2t = ((torch.rand(V * e, d, d_ff, generator=gen, device=dev) * 2 - 1) / math.sqrt(d_ff)).to(tdt)
        b1 = torch.zeros(V * e, d_ff, device=dev)
        b2 = torch.zeros(V * e, d, device=dev)
        out = torch.empty_like(x)
        loss = torch.empty(V, dtype=torch.float64, device=dev)
        inp = dict(x=x, w_router=w_router, W1t=W1t, W2t=W2t, b1=b1, b2=b2, out=out, loss=loss,
                   fused_gate=args.fused_gate)
        train = bool(cfgd.get("train"))
        if args.exchange == "peer" and not train:
            # the step calls then fuse the level-1 return for in-process tokens into GEMM 2
            # (smile_set_output; smile_forward does the same for its io->out)
            L.set_output(out)
        if train:
            f32 = dict(dtype=torch.float32, device=dev)
            inp.update(alpha=0.005 if mode == "bilevel" else 0.01, beta=0.005 if mode == "bilevel" else 0.0,
                       gout=torch.randn(V, T, d, generator=gen, device=dev, dtype=torch.float32).to(tdt),
                       dx=torch.empty_like(x), W1=W1t.transpose(1, 2).contiguous(), W2=W2t.transpose(1, 2).contiguous(),
                       dW1=torch.empty(V * e, d, d_ff, **f32), db1=torch.empty(V * e, d_ff, **f32),
                       dW2=torch.empty(V * e, d_ff, d, **f32), db2=torch.empty(V * e, d, **f32),
                       dWr=torch.empty(KW, d, **f32))
            step_fn = step_train
        else:
            step_fn = step
        phases = PHASES_TRAIN if train else (PHASES_BI if mode == "bilevel" else PHASES_FLAT)
        nph = len(phases)
        for _ in range(args.warmup):
            step_fn(L, inp)
        torch.cuda.synchronize()
        err = L.get_error()
        if err:
            raise SystemExit(f"device error {err} in {mode}")
        # (1) the phase breakdown: an event after every phase (the events serialise the
        # kernels around them, so these steps are not the headline)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nph + 1)] for _ in range(args.steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush()                       # L2 flush outside the step's events
            step_fn(L, inp, evs[k])
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ph = [[evs[k][i].elapsed_time(evs[k][i + 1]) for i in range(nph)] for k in range(args.steps)]
        phased_ms = statistics.median([sum(p) for p in ph])
        # (2) the headline: events only around each step (the libsmile kernels of a step run
        # back to back, with programmatic dependent launch between them)
        e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        lc0 = smb.launch_count()
        t_beg = time.time()
        for k in range(args.steps):
            flush()                       # L2 flush outside the step's events
            e0[k].record()
            step_fn(L, inp)
            e1[k].record()
        torch.cuda.synchronize()
        t_end = time.time()
        launched = smb.launch_count() - lc0           # libsmile kernels enqueued in the timed region
        if dist:
            dist.barrier()
        step_ms = [e0[k].elapsed_time(e1[k]) for k in range(args.steps)]
        eager_ms = statistics.median(step_ms)            # median, with p10 / p90 reported
        q = statistics.quantiles(step_ms, n=10) if len(step_ms) >= 2 else [eager_ms] * 9
        step_stats = {"median": eager_ms, "p10": q[0], "p90": q[-1], "mean": statistics.mean(step_ms),
                      "min": min(step_ms), "max": max(step_ms)}
        graph_ms = None
        if args.graph and world == 1:
            # the same step captured once as a CUDA graph and replayed (the libsmile calls
            # are stream-ordered with no host syncs); timed with events around each replay
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                step_fn(L, inp)
            torch.cuda.current_stream().wait_stream(cs)
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg):
                step_fn(L, inp)
            for _ in range(max(3, args.warmup)):
                cg.replay()
            g0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            g1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            torch.cuda.synchronize()
            for k in range(args.steps):
                flush()
                g0[k].record()
                cg.replay()
                g1[k].record()
            torch.cuda.synchronize()
            graph_ms = statistics.median(g0[k].elapsed_time(g1[k]) for k in range(args.steps))
            if L.get_error():
                raise SystemExit("device error in graph replay")
            del cg
        mine = torch.tensor([graph_ms if graph_ms is not None else eager_ms] +
                            [statistics.mean(p[i] for p in ph) for i in range(nph)],
                            dtype=torch.float64, device=dev)
        allr = [torch.empty_like(mine) for _ in range(world)] if dist else [mine]
        if dist:
            dist.all_gather(allr, mine)
        allr = torch.stack(allr).cpu()
        ms = allr[:, 0].max().item()                         # max over ranks
        rank_ms = allr[:, 0].tolist()
        phase_ms = {phases[i]: allr[:, 1 + i].max().item() for i in range(nph)}
        # algorithmic work of the dominant kernel (expert FFN): 4 * rows * d * d_ff flops
        w = L.view()
        rows = int(w["rcounts"].sum().item())
        kept = rows
        # algorithmic HBM bytes of the routing / data-movement phases:
        # gate reads x and writes the 24 B route record per token; every row mover reads
        # and writes each row it moves; combine1 also writes the zero rows of drops.
        rb = d * (2 if cfgd["dtype"] == "bf16" else 4)
        kept1 = int(w["counts1"].sum().item())
        if inp.get("fused_gate") and not train:
            # fused gate + permute: x read once, kept rows written, 24 B route record per token
            hbm = {"gate1": V * T * (rb + 24) + kept1 * rb, "combine1": (kept1 + V * T) * rb}
        else:
            hbm = {"gate1": V * T * (rb + 24), "dispatch1": 2 * kept1 * rb, "combine1": (kept1 + V * T) * rb}
        if mode == "bilevel":
            recv2 = int(w["counts2"].sum().item())
            hbm.update({"dispatch2": 2 * recv2 * rb, "combine2": 2 * recv2 * rb})
        # rows this process sends to ranks of OTHER processes (NVLink), per level
        c1 = w["counts1"].cpu().numpy()
        r0 = rank * V
        nvl = {}
        if mode == "bilevel":
            m_ = cfgd["m"]
            rem1 = sum(int(c1[v, i]) for v in range(V) for i in range(cfgd["n"])
                       if (i * m_ + (r0 + v) % m_) // V != rank)
            c2 = w["counts2"].cpu().numpy()
            rem2 = sum(int(c2[v, k]) for v in range(V) for k in range(c2.shape[1])
                       if (((r0 + v) // m_) * m_ + k // e) // V != rank)
            nvl = {"inter": rem1 * rb, "intra": rem2 * rb}
        else:
            nvl = {"world": sum(int(c1[v, E]) for v in range(V) for E in range(c1.shape[1]) if (E // e) // V != rank) * rb}
        ffn_ms = phase_ms["ffn"] if not train else None
        ffn_tc = cfgd["dtype"] == "bf16" and args.ffn != "simt" and smb.TCGEN05_DEFAULT
        if (mode == "flat" and args.exchange == "peer" and ffn_tc and not train and args.topk == 1
                and os.environ.get("SMILE_OUT_DIRECT", "1") != "0" and not inp.get("fused_gate")):
            # FLAT gets the same GEMM 2 -> out fusion: out[t] for tokens whose expert is in this
            # process; combine1 moves the other kept tokens and zeroes drops
            import numpy as np
            d1 = w["dest1"].cpu().numpy()
            s1 = w["slot1"].cpu().numpy()
            kept_l1 = s1 < L.C1
            remote = kept_l1 & ((d1 // e) // V != rank)
            if L.V == L.G:
                hbm["dispatch1"] = hbm.get("dispatch1", 0) + int((~kept_l1).sum()) * rb
                hbm["combine1"] = 0
            else:
                hbm["combine1"] = (2 * int(remote.sum()) + int((~kept_l1).sum())) * rb
        if (mode == "bilevel" and args.exchange == "peer" and ffn_tc
                and os.environ.get("SMILE_RET_DIRECT", "1") != "0"):
            # GEMM 2 wrote the rows of this process's intermediates straight into ret1
            # (a11 fused into the FFN, no extra bytes); combine2 moves only rows of experts
            # in other processes -- the level-2 rows this process sent away
            hbm["combine2"] = 2 * nvl.get("intra", 0)
            if not train and os.environ.get("SMILE_OUT_DIRECT", "1") != "0" and not inp.get("fused_gate"):
                # ... and out[t] for tokens whose intermediate and expert are in this process
                # too (a12 + a13 fused): combine1 moves the other kept tokens and zeroes drops
                import numpy as np
                d1 = w["dest1"].cpu().numpy()
                d2 = w["dest2"].cpu().numpy()
                s1 = w["slot1"].cpu().numpy()
                m_ = cfgd["m"]
                rk = rank * V + np.arange(V)[:, None]
                u = d1 * m_ + rk % m_
                q = d1 * m_ + d2 // e
                kept_l1 = s1 < L.C1
                remote = kept_l1 & ((u // V != rank) | (q // V != rank))
                if L.V == L.G:
                    # every rank in this process: the level-1 permute writes the dropped tokens'
                    # zero rows and combine1 is not launched
                    hbm["dispatch1"] = hbm.get("dispatch1", 0) + int((~kept_l1).sum()) * rb
                    hbm["combine1"] = 0
                else:
                    hbm["combine1"] = (2 * int(remote.sum()) + int((~kept_l1).sum())) * rb
        fabric_model = None
        if fabric:
            # the emulation's own cost model for one cross-node exchange (forward; the reverse
            # moves the same rows back): per sending rank, sum over its cross-node messages of
            # latency + bytes / bandwidth; max over ranks (the NICs run concurrently)
            import numpy as np
            c1 = w["counts1"].cpu().numpy().astype(np.int64)
            m_, L_us, bw = cfgd["m"], fabric["inter_latency_us_per_message"], fabric["inter_gbps_per_rank"]
            per_rank = []
            for v in range(V):
                s_ = (rank * V + v) // m_
                dests = range(c1.shape[1])
                node = (lambda i: i) if mode == "bilevel" else (lambda E: (E // e) // m_)
                msgs = [i for i in dests if node(i) != s_]
                # flat: one message per destination RANK (its e experts travel together)
                if mode == "flat":
                    ranks = sorted({E // e for E in msgs})
                    per_rank.append(sum(L_us + sum(int(c1[v, q * e + k]) for k in range(e)) * rb / bw / 1e3
                                        for q in ranks))
                else:
                    per_rank.append(sum(L_us + int(c1[v, i]) * rb / bw / 1e3 for i in msgs))
            fabric_model = {"cross_node_exchange_model_ms": max(per_rank) / 1e3,
                            "measured_ms": phase_ms["a2a_inter" if mode == "bilevel" else "a2a_world"]}
        res = dict(L=L, inp=inp, ms=ms, ffn_tc=ffn_tc, fabric_model=fabric_model, rank_ms=rank_ms, phase_ms=phase_ms, rows=rows, kept=kept, ffn_ms=ffn_ms,
                   t_beg=t_beg, t_end=t_end,
                   tokens=G * T, launches=launched, hbm_bytes=hbm, train=train, eager_ms=eager_ms, graph_ms=graph_ms,
                   step_stats=step_stats, phased_ms=phased_ms,
                   nvl_bytes=nvl)
        if train:
            res["hbm_bytes"] = {}
        # e2e through smile_forward_host_stream: every step's x comes from pinned host memory
        # and its output + loss go back to pinned host memory, inside the timed region; the
        # H2D of step k+1 and the D2H of step k-1 overlap step k (two copy engines)
        if not args.no_e2e and not train:
            hx = [x.cpu().pin_memory() for _ in range(2)]
            ho = [torch.empty_like(hx[0]).pin_memory() for _ in range(2)]
            xd2 = [torch.empty_like(x) for _ in range(2)]
            od2 = [torch.empty_like(x) for _ in range(2)]
            e2e_steps = max(4, min(args.steps, 20))
            hl = torch.empty(e2e_steps, V, dtype=torch.float64).pin_memory()
            L.forward_host_stream(xd2, od2, hx, ho, hl[:2], W1t, b1, W2t, b2, loss, w_router=w_router)
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            L.forward_host_stream(xd2, od2, [hx[k % 2] for k in range(e2e_steps)], [ho[k % 2] for k in range(e2e_steps)],
                                  hl, W1t, b1, W2t, b2, loss, w_router=w_router)
            t1.record()
            torch.cuda.synchronize()
            et = torch.tensor([t0.elapsed_time(t1) / e2e_steps], dtype=torch.float64, device=dev)
            if dist:
                dist.all_reduce(et, op=dist.ReduceOp.MAX)
            res["e2e"] = {"value": G * T / (et.item() / 1e3), "unit": "tokens/s",
                          "h2d_bytes_per_step": x.numel() * x.element_size(),
                          "d2h_bytes_per_step": x.numel() * x.element_size() + V * 8,
                          "ms_per_step": et.item(), "steps": e2e_steps,
                          "api": "smile_forward_host_stream (pinned host in/out, copies overlapped across steps)"}
        results[mode] = res
        del evs
    if sampler:
        main_mode = results[modes[0]]
        sampler.t_beg, sampler.t_end = main_mode["t_beg"], main_mode["t_end"]
        results[modes[0]]["clocks"] = sampler.stop()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    main = results[modes[0]]
    ms = main["ms"]
    flops = 4.0 * main["rows"] * d * d_ff
    timed_s = ms * args.steps / 1e3
    bf16_peak = peaks.get("bf16_tflops_sustained" if timed_s > 1.0 else "bf16_tflops")
    ffn_is_tensor = main["ffn_tc"]
    traffic = load_json(os.path.join(ROOT, "profiles", "traffic.json")) or {}
    if main.get("train"):
        flops = 12.0 * main["rows"] * d * d_ff        # expert FFN fwd (2 GEMMs) + bwd (4 GEMMs)
        achieved = flops / (ms / 1e3) / 1e12
    else:
        achieved = flops / (main["ffn_ms"] / 1e3) / 1e12
    if cfgd["dtype"] == "bf16" and ffn_is_tensor:
        roof = {"bound": "tensor", "achieved": achieved, "peak": bf16_peak, "unit": "TFLOP/s",
                "frac": achieved / bf16_peak if bf16_peak else None,
                "peak_source": "MEASURED_PEAKS.json " + ("bf16_tflops_sustained" if timed_s > 1.0 else "bf16_tflops")}
    else:
        # SIMT FFMA: 148 SMs x 128 lanes x 2 flop x sm clock
        clk = (main.get("clocks") or {}).get("sm_mhz") or 1965.0
        alu_peak = 148 * 128 * 2 * clk * 1e6 / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "TFLOP/s",
                "frac": achieved / alu_peak, "peak_source": f"148 SM x 128 FP32 lanes x 2 x {clk:.0f} MHz"}
    roof["kernel"] = ("whole training step (expert FFN fwd + bwd flops / step time; all six GEMMs on tcgen05)" if main.get("train")
                      else "smile_expert_ffn (2 grouped GEMM launches)")
    tr = traffic.get(f"{args.config}_{modes[0]}_ffn")
    roof["traffic"] = tr["bytes_per_step"] if tr else None
    if tr:
        roof["traffic_note"] = (f"DRAM read+write bytes of the FFN's {tr['launches']} GEMM launches of one step, "
                                f"ncu --set full ({tr['source']})")
    roof["algorithmic_flops_per_step"] = flops
    if not main.get("train") and ffn_is_tensor:
        # the FFN's bound is max(flops / tensor peak, bytes / HBM peak): the
        # weights of every resident expert are streamed once per step besides X, H, Y
        eb = 2
        kept = main["rows"]
        ffn_bytes = kept * d * eb + 2 * kept * d_ff * eb + kept * d * eb + (G // world) * e * 2 * d * d_ff * eb
        t_fl = flops / (bf16_peak * 1e12)
        t_by = ffn_bytes / (peaks.get("hbm_gbs", 6542.7) * 1e9)
        t_me = main["ffn_ms"] / 1e3
        roof["max_bound"] = {"bound": "tensor" if t_fl >= t_by else "hbm", "t_flops_ms": t_fl * 1e3,
                             "t_bytes_ms": t_by * 1e3, "algorithmic_bytes": ffn_bytes,
                             "frac": max(t_fl, t_by) / t_me,
                             "note": "FFN bytes = X + H write + H read + Y + all resident experts' W1, W2 once"}
    line = {
        "metric": METRIC, "value": main["tokens"] / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16" if cfgd["dtype"] == "bf16" else "f32",
        "data": "synthetic (N(0,1) tokens, U(+-1/sqrt(fan_in)) random-init router and experts)",
        "config": {"workload": f"{args.config}: one {modes[0]} MoE layer {'fwd+bwd' if main.get('train') else 'fwd'}, "
                               f"{G} ranks as {cfgd['n']}x{cfgd['m']} (n x m), "
                               f"e={e}/rank, T={T}/rank, d={d}, d_ff={d_ff}, cf={cfgd['cf']}, fused router; "
                               f"{V} ranks per GPU; exchange={args.exchange}", "ranks_per_gpu": V, "mode": modes[0],
                   "exchange": args.exchange, "flat_topk": args.topk,
                   "fabric": fabric and dict(fabric, note="IN-BOX EMULATION (smile_set_fabric): cross-node transfers "
                                             "of the COPY exchange go through per-rank emulated NICs -- "
                                             "latency per message + bytes / bandwidth of wall time each; not a "
                                             "real network"),
                   "l2": flush.describe(),
                   "timing": "CUDA events per phase on the launching stream; value from the median step"},
        "phase_ms": main["phase_ms"], "phase_ms_note": "per phase: max over ranks of the mean over steps (events on the launching stream)",
        "rank_ms_per_step": main["rank_ms"], "kept_tokens": main["kept"],
        "cuda_graph": main["graph_ms"] is not None, "eager_ms_per_step": main["eager_ms"],
        "step_ms_stats": main["step_stats"], "phase_instrumented_ms_per_step": main["phased_ms"],
        "step_ms_note": "rank-0 process, eager steps; ms_per_step = max over ranks of each rank's median",
        "roofline": roof,
        "hbm_phases": hbm_phases(main, peaks),
        "nvlink": None if main.get("train") else nvlink_levels(main, world, modes[0], args.exchange),
        "layer_roofline": None if main.get("train") else layer_roofline(main, cfgd, peaks, world, flops),
        "gpu_launches": main["launches"],
        "gpu_launches_note": "libsmile kernels launched in the timed region (smile_launch_count delta; NCCL not counted)",
        "clocks": main.get("clocks"),
    }
    if "e2e" in main:
        line["e2e"] = main["e2e"]
    if "flat" in results and modes[0] != "flat":
        f = results["flat"]
        line["flat"] = {"value": f["tokens"] / (f["ms"] / 1e3), "ms_per_step": f["ms"], "eager_ms_per_step": f["eager_ms"],
                        "phase_ms": f["phase_ms"],
                        "e2e": f.get("e2e"), "kept_tokens": f["kept"]}
        line["bilevel_over_flat"] = line["value"] / line["flat"]["value"]
        if fabric:
            line["flat"]["fabric_model"] = f.get("fabric_model")
    if fabric:
        line["fabric_model"] = main.get("fabric_model")
    if not args.no_cpu and world == 1:           # rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_oracle_sample(cfgd, modes[0])
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.chunks > 1:
        return run_pipelined(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
