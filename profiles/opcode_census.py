#!/usr/bin/env python
"""Executed warp-instructions of one kernel by SASS opcode, from an ncu report's source page
(run here, no GPU).   python profiles/opcode_census.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout.splitlines()
hdr, agg, samp, tot, tsamp = None, collections.Counter(), collections.Counter(), 0, 0
for row in csv.reader(txt):
    if row and row[0] == "Address":
        hdr = row
        ie, ws = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(row) < len(hdr) or not row[0].startswith("0x"):
        continue
    ins = row[1].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1]
    op = ins.split()[0].split(".")[0] if ins else "?"
    n = int(row[ie] or 0)
    s = int(row[ws] or 0)
    agg[op] += n
    samp[op] += s
    tot += n
    tsamp += s
print(f"{kern}: {tot} warp-instr executed, {tsamp} stall samples")
for op, n in agg.most_common(top):
    print(f"{op:10s} {n:12d} {n / tot:6.3f}  samples {samp[op] / max(tsamp, 1):6.3f}")
