#!/usr/bin/env python
"""Per-CTA timeline of one tensor-core kernel (measurement only).

    SMILE_TRACE=gate|ffn1|ffn2 python tools/gpu/trace_kernels.py --config c2 --mode bilevel

Runs a few bench steps (bench.run_ours), then reads the stamps the named kernel wrote in its
LAST launch (smile_debug_trace; slot layout in smile_internal.h and the kernels) and prints,
over CTAs (mean / median / min / max, in kilo-cycles of each CTA's own clock64): the MMA
thread's per-tile issue span (accumulator acquired -> last commit issued) and its waits for a
free accumulator, the epilogue's wait for the tile's accumulator, its duration and (gate) the
phases of gate_finish.  The globaltimer start / end stamps are reported as well but tick too
coarsely for spans of tens of microseconds.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

SLOTS = 1024


def main():
    name = os.environ.get("SMILE_TRACE")
    if not name:
        raise SystemExit("set SMILE_TRACE=gate|ffn1|ffn2")
    import bench
    from paper_2212_05191_b200 import smile as smb
    sys.argv = [sys.argv[0]] + sys.argv[1:] + ["--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu",
                                               "--clock-ms", "0"]
    args = bench.parse()
    bench.run_ours(args)
    import torch
    torch.cuda.synchronize()
    L = smb.lib()
    L.smile_debug_trace.restype = C.c_int64
    L.smile_debug_trace.argtypes = [C.c_void_p, C.c_int64]
    buf = np.zeros((256, SLOTS), np.uint64)
    rows = L.smile_debug_trace(buf.ctypes.data, buf.nbytes)
    if rows <= 0:
        raise SystemExit("no trace recorded")
    tr = buf[:rows].astype(np.int64)
    live = tr[:, 0] > 0
    tr = tr[live]
    gt0 = tr[:, 0].min()
    out = {"kernel": name, "ctas": int(len(tr))}
    rate = (tr[:, 3] - tr[:, 2]) / np.maximum(tr[:, 1] - tr[:, 0], 1)     # cycles per ns (GHz)
    out["sm_ghz_median"] = float(np.median(rate))
    start = (tr[:, 0] - gt0) / 1e3
    end = (tr[:, 1] - gt0) / 1e3
    out["cta_start_us"] = [float(start.min()), float(np.median(start)), float(start.max())]
    out["cta_end_us"] = [float(end.min()), float(np.median(end)), float(end.max())]

    # %globaltimer ticks too coarsely for these spans (its per-CTA rates come out above the
    # SM clock), so every duration below is in kilo-cycles of the CTA's own clock64, from
    # the CTA's start stamp
    out["cta_span_kcyc"] = [float(x) for x in np.percentile((tr[:, 3] - tr[:, 2]) / 1e3, [0, 50, 100])]

    def us(c, slot):                  # slot's clock64 -> kilo-cycles since the CTA's start
        v = tr[c, slot]
        if v == 0:
            return None
        return float((v - tr[c, 2]) / 1e3)

    mma_base, epi_base, epi_stride = (8, 256, 4) if name == "gate" else (8, 520, 2)
    per = {"mma_span": [], "mma_wait_acc": [], "epi_wait": [], "epi_release": [], "epi_done": [],
           "tail_after_last_mma": [], "first_mma": [], "tiles": []}
    for c in range(len(tr)):
        ntile = 0
        prev_end = None
        while ntile < 240 and tr[c, mma_base + 2 * ntile] != 0:
            s0, s1 = us(c, mma_base + 2 * ntile), us(c, mma_base + 2 * ntile + 1)
            if s1 is None:
                break
            if ntile == 0:
                per["first_mma"].append(s0)
            per["mma_span"].append(s1 - s0)
            if prev_end is not None:
                per["mma_wait_acc"].append(s0 - prev_end)
            prev_end = s1
            ntile += 1
        if ntile:
            per["tiles"].append(ntile)
            per["tail_after_last_mma"].append((tr[c, 3] - tr[c, 2]) / 1e3 - prev_end)
        it = 0
        while it < 240:
            g = us(c, epi_base + epi_stride * it)
            r = us(c, epi_base + epi_stride * it + 1)
            if g is None or r is None:
                it += 1
                if it > 2 * max(ntile, 1):
                    break
                continue
            m1 = us(c, mma_base + 2 * it + 1)
            if m1 is not None:
                per["epi_wait"].append(g - m1)          # MMA commit issued -> accumulator ready
            per["epi_release"].append(r - g)
            if epi_stride == 4:
                d = us(c, epi_base + epi_stride * it + 2)
                if d is not None:
                    per["epi_done"].append(d - g)
                f0, f1, f2 = us(c, 600 + 4 * it), us(c, 601 + 4 * it), us(c, 602 + 4 * it)
                if None not in (f0, f1, f2) and d is not None:
                    per.setdefault("fin_phaseB", []).append(f0 - r)
                    per.setdefault("fin_rank", []).append(f1 - f0)
                    per.setdefault("fin_stats", []).append(f2 - f1)
                    per.setdefault("fin_after", []).append(d - f2)
            it += 1
    for k, v in per.items():
        if v:
            out[k] = {"mean": statistics.mean(v), "median": statistics.median(v), "min": min(v), "max": max(v),
                      "n": len(v)}
    pslot = {4: "producer_ready", 5: "producer_last_load", 6: "split_built"}
    for sl, nm in pslot.items():
        vals = [us(c, sl) for c in range(len(tr)) if tr[c, sl] != 0]
        if vals:
            out[nm + "_kcyc"] = [min(vals), statistics.median(vals), max(vals)]
    print("TRACE " + json.dumps(out))


if __name__ == "__main__":
    main()
