#!/usr/bin/env python
"""Launch list of one bench step from `ncu --metrics gpu__time_duration.sum --csv`:

    python tools/launch_summary.py gpurun_out/launches.csv profiles/r01_launches_c2_bilevel.md [--skip N] [--count M]

Keeps the launches of one step (default: the first router split through the next aux-loss
kernel; or --skip N launches, then --count M), writes a
markdown table with each kernel's share of the step and the expert FFN's total share."""
import csv
import sys


def main():
    src, out = sys.argv[1], sys.argv[2]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    count = int(sys.argv[sys.argv.index("--count") + 1]) if "--count" in sys.argv else None
    rows = list(csv.reader(open(src)))
    hdr = None
    ks = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            u = d.get("Metric Unit", "ns")
            us = v / 1000.0 if u in ("ns", "nsecond") else (v * 1000.0 if u in ("ms", "msecond") else v)
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("smile::<unnamed>::", "")
            name = name.replace("<unnamed>::", "").replace("(int)", "").replace("(bool)", "")
            ks.append((name, us))
    ks = ks[skip:]
    if count:
        ks = ks[:count]
    else:
        # one layer step: from the first router split through the next aux-loss kernel
        b = next(i for i, (n, _) in enumerate(ks) if n.startswith("router_split"))
        e = next(i for i in range(b, len(ks)) if ks[i][0].startswith("aux_kernel"))
        ks = ks[b:e + 1]
    tot = sum(us for _, us in ks)
    ffn = sum(us for n, us in ks if "ffn_gemm" in n)
    lines = ["| kernel | us | share |", "|---|---|---|"]
    lines += [f"| {n} | {us:.1f} | {100 * us / tot:.1f}% |" for n, us in ks]
    md = ("# Launch list of one C2 bi-level step (ncu --metrics gpu__time_duration.sum --clock-control none; "
          "cold, serialised)\n\n" + "\n".join(lines) +
          f"\n\nTotal {tot:.0f} us; the expert FFN ({sum('ffn_gemm' in n for n, _ in ks)} ffn_gemm_tcgen05 launches) "
          f"is {100 * ffn / tot:.1f}% of it.\n")
    open(out, "w").write(md)
    print(md)


if __name__ == "__main__":
    main()
