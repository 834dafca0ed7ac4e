#!/usr/bin/env python
"""Warp-level instructions executed and stall samples per CUDA source line of one kernel
(ncu report captured with -lineinfo and --import-source on).

    python profiles/hot_lines.py report.ncu-rep kernel_substring [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
# blocks: "Kernel Name" / "File Path" headers followed by csv rows
agg = collections.defaultdict(lambda: [0, 0, ""])
cur_kernel, cur_file, hdr = None, None, None
for line in txt:
    if line.startswith('"Kernel Name"') or line.startswith('"Function Name"'):
        cur_kernel = line
        continue
    if line.startswith('"File Path"') or line.startswith('"File Name"'):
        cur_file = line.split('","')[-1].strip('",').split("/")[-1]
        continue
    if line.startswith('"Line No"'):
        hdr = next(csv.reader([line]))
        continue
    if hdr is None or cur_kernel is None or kern not in cur_kernel:
        continue
    r = next(csv.reader([line]))
    if len(r) != len(hdr):
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        si = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    key = (cur_file, r[0])
    agg[key][0] += ie
    agg[key][1] += si
    agg[key][2] = r[1].strip()[:100]
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"{kern}: {tot_i} warp-instr, {tot_s} samples")
for (f, ln), (i, s_, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{i / tot_i:6.3f} {s_ / tot_s:6.3f}  {f}:{ln}  {src}")
