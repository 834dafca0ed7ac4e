#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, no GPU needed).

    python profiles/summarize_ncu.py launches.csv [full.ncu-rep] > profiles/rNN_summary.md

* launch list (``--metrics gpu__time_duration.sum --clock-control none`` CSV): per-kernel
  mean device time and share of one scan (cold-cache, serialised: compare SHARES).
* full capture (``--set full``): duration, DRAM bytes, throughput, occupancy, issue
  activity and the top stall reasons of every captured kernel.
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("::")[-1]
        v = float(r[vi].replace(",", ""))
        v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3,
             "ms": v * 1e3}.get(r[ui], v)
        agg.setdefault(name, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {sum(v) / tot:.3f} |")
    return "\n".join(out)


METRICS = [("gpu__time_duration.sum", "us", 1), ("dram__bytes_read.sum", "MB", 1e-6),
           ("dram__bytes_write.sum", "MB", 1e-6), ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "% dram", 1),
           ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "% sm", 1),
           ("sm__warps_active.avg.pct_of_peak_sustained_active", "% occ", 1),
           ("smsp__issue_active.avg.pct_of_peak_sustained_active", "% issue", 1),
           ("smsp__inst_executed.sum", "Minstr", 1e-6), ("launch__registers_per_thread", "regs", 1),
           ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "% fma", 1)]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].split("::")[-1]
        vals = []
        for m, u, sc in METRICS:
            if m in h:
                x = r[h.index(m)].replace(",", "")
                try:
                    xv = float(x)
                    # ncu raw units vary (ns / us / bytes / Kbyte ...): normalise the common ones
                    unit = units[h.index(m)]
                    if m == "gpu__time_duration.sum":
                        xv = xv * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                                   "ms": 1e3}.get(unit, 1.0)
                    if m.startswith("dram__bytes"):
                        xv = xv * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
                    vals.append(f"{xv * sc:.4g} {u}")
                except ValueError:
                    pass
        stall = [(m.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                  float(r[h.index(m)] or 0)) for m in h
                 if "smsp__average_warps_issue_stalled" in m and m.endswith("per_issue_active.ratio")]
        stall.sort(key=lambda x: -x[1])
        out.append(f"* `{name}`: " + ", ".join(vals) + "; stalls/issue: " +
                   ", ".join(f"{a} {b:.2f}" for a, b in stall[:5]))
    return "\n".join(out)


if __name__ == "__main__":
    print("## Launch list\n")
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print("\n## Full capture\n")
        print(full(sys.argv[2]))
