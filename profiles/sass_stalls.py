#!/usr/bin/env python
"""Per-SASS-instruction stall breakdown of one ncu report (source page, --print-source sass).

    python profiles/sass_stalls.py report.ncu-rep [top]
Prints the stall-reason totals and the top instructions by stall samples with their reasons.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = [i for i, r in enumerate(rows) if "Instructions Executed" in r][0]
h = rows[hi]
iI, iS, iW = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
sc = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
data, tot = [], {}
for idx, r in enumerate(rows[hi + 1:]):
    try:
        w, ins = float(r[iW]), float(r[iI])
    except (ValueError, IndexError):
        continue
    st = {c: float(r[i] or 0) for i, c in sc}
    for c, v in st.items():
        tot[c] = tot.get(c, 0) + v
    data.append((w, ins, idx, r[iS].strip(), st))
allw = sum(d[0] for d in data)
insn = sum(d[1] for d in data)
print(f"warp-instructions {insn:.0f}, stall samples {allw:.0f}")
print("by reason:", ", ".join(f"{c[6:]} {100 * v / allw:.1f}%" for c, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v > 0.005 * allw))
for w, ins, idx, s, st in sorted(data, reverse=True)[:top]:
    rs = ", ".join(f"{c[6:]} {v:.0f}" for c, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v > 0)
    print(f"{idx:5d} {100 * w / allw:5.1f}% {ins:9.0f}  {s:60s} [{rs}]")
