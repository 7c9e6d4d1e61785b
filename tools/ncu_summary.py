#!/usr/bin/env python
"""Summarise an `ncu --set full` report of one bench step into profiles/:

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_c2.md [--config c2 --mode bilevel]

Writes a markdown table (duration, DRAM bytes read/written, DRAM and tensor-pipe
utilisation, registers per kernel launch) and merges the per-step DRAM traffic of the
expert FFN (its two GEMM launches) into profiles/traffic.json under "<config>_<mode>_ffn",
which bench.py reports as roofline.traffic.  Reads the report with `ncu -i` only."""
import csv
import io
import json
import os
import subprocess
import sys

COLS = {
    "dur_us": "gpu__time_duration.sum",
    "rd_MB": "dram__bytes_read.sum",
    "wr_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm_ghz": "sm__cycles_elapsed.avg.per_second",
    "regs": "launch__registers_per_thread",
}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c2"
    mode = sys.argv[sys.argv.index("--mode") + 1] if "--mode" in sys.argv else "bilevel"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {k: hdr.index(v) for k, v in COLS.items() if v in hdr}
    iname = hdr.index("Kernel Name")
    unit = {k: units[i] for k, i in idx.items()}
    lines = ["| kernel | duration (us) | DRAM read (MB) | DRAM write (MB) | DRAM % | tensor % | SM GHz | regs |",
             "|---|---|---|---|---|---|---|---|"]
    ffn = []
    for r in data:
        def g(k, scale=1.0):
            if k not in idx or not r[idx[k]]:
                return None
            v = float(r[idx[k]].replace(",", ""))
            u = unit[k]
            if k == "dur_us":
                v = v / 1000.0 if u in ("nsecond", "ns") else (v * 1000.0 if u in ("msecond", "ms") else v)
            if k in ("rd_MB", "wr_MB"):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}.get(u, 1.0)
            if k == "sm_ghz":
                v = v * {"hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}.get(u.lower().capitalize() if u else "", 1.0)
            return v
        name = r[iname].split("(")[0].replace("smile::<unnamed>::", "").replace("void ", "")
        vals = [g(k) for k in COLS]
        lines.append("| " + name + " | " + " | ".join("" if v is None else f"{v:.3g}" for v in vals) + " |")
        if "ffn_gemm" in name:
            ffn.append((g("rd_MB") or 0) + (g("wr_MB") or 0))
    md = f"# ncu --set full: one {cfg} {mode} step ({os.path.basename(rep)})\n\n" + "\n".join(lines) + "\n"
    open(out, "w").write(md)
    tj = os.path.join(os.path.dirname(out), "traffic.json")
    t = json.load(open(tj)) if os.path.exists(tj) else {}
    if len(ffn) >= 2:
        t[f"{cfg}_{mode}_ffn"] = {"bytes_per_step": sum(ffn[:2]) * 1e6, "launches": 2, "source": os.path.basename(out)}
    json.dump(t, open(tj, "w"), indent=1)
    print(md)


if __name__ == "__main__":
    main()
