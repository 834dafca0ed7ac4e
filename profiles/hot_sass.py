#!/usr/bin/env python
"""Top SASS lines by warp-stall samples of one kernel in an ncu report (run here, no GPU).

    python profiles/hot_sass.py report.ncu-rep kernel_substring [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for line in txt.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line]
        blocks.append(cur)
    elif cur is not None:
        cur.append(line)
blk = [b for b in blocks if kern in b[0]][0]
print(blk[0][:160])
rows = list(csv.reader(io.StringIO("\n".join(blk[1:]))))
h = rows[0]
si, src, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
tot = sum(int(r[si]) for r in rows[1:] if r[si].isdigit())
ranked = sorted(rows[1:], key=lambda r: -int(r[si]) if r[si].isdigit() else 0)
print(f"total samples {tot}")
for r in ranked[:top]:
    print(f"{int(r[si]) / tot:6.3f} {r[ie]:>9} {r[0][-5:]}  {r[src].strip()}")
