#!/usr/bin/env python
"""Write profiles/rNN_summary.md, rNN_launches.csv and ncu_traffic.json from a GPU check
(scripts/gpu_check.sh <tag>) and a one-scan full capture (scripts/ncu_scan.sh <tag>_scan).

    python profiles/make_summary.py <round> <check tag> <scan tag>
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
rnd, tag, scan = sys.argv[1], sys.argv[2], sys.argv[3]
out_dir = os.path.join(ROOT, "gpurun_out")
launches = os.path.join(out_dir, tag, "launches.csv")
rep = os.path.join(out_dir, scan, "full.ncu-rep")
bench = json.load(open(os.path.join(out_dir, tag, "bench.json")))
summ = subprocess.run([sys.executable, os.path.join(HERE, "summarize_ncu.py"), launches, rep], capture_output=True,
                      text=True).stdout
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
traffic = collections.defaultdict(float)
for r in rows[2:]:
    b = sum(float(r[h.index(m)].replace(",", "")) * scale.get(units[h.index(m)], 1)
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    name = r[ki]
    traffic["project" if "k_project" in name else "render" if "k_render" in name else "bin_sort"] += b
json.dump({**{k: int(v) for k, v in traffic.items()},
           "note": f"dram__bytes_read.sum + dram__bytes_write.sum per scan (all launches of the stage), ncu --set full "
                   f"of one steady-state config-B scan, round {rnd} (profiles/r{rnd}_summary.md)"},
          open(os.path.join(HERE, "ncu_traffic.json"), "w"), indent=1)
shutil.copy(launches, os.path.join(HERE, f"r{rnd}_launches.csv"))
st = bench["stages"]
head = [f"# Round {rnd} ncu evidence (config B, bench.py launch configuration)", "",
        f"bench.py (N=1): {bench['value'] / 1e6:.1f} M rays/s, {bench['ms_per_step']:.3f} ms/scan "
        f"(project {st['project']['ms']:.3f}, bin_sort {st['bin_sort']['ms']:.3f}, render {st['render']['ms']:.3f} ms); "
        f"e2e {bench['e2e']['value'] / 1e6:.1f} M rays/s; SM clock {bench['clocks']['sm_mhz']} MHz "
        f"(max {bench['clocks']['sm_max_mhz']}), reasons {bench['clocks']['reasons']}.", "",
        "Per-stage DRAM traffic of one scan (ncu): " +
        ", ".join(f"{k} {v / 1e6:.0f} MB" for k, v in traffic.items()) + ".", "",
        "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` of `bench.py --steps 2 --warmup 3` "
        "(cold-cache, serialised: compare SHARES). Full capture: `ncu --set full` of one steady-state scan "
        "(scripts/ncu_scan.sh).", ""]
# SM clock ncu observed per kernel (--clock-control none) and the issue peak at that clock
txt2 = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                       "sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum,smsp__inst_executed.sum"],
                      capture_output=True, text=True).stdout
r2 = list(csv.reader(io.StringIO(txt2)))
h2 = r2[0]
clk = ["", "## SM clock ncu observed (--clock-control none) and issue utilisation at that clock", "",
       "| kernel | us | SM GHz | warp-instr | issue util at observed clock | FP32 issue peak at that clock (T lane-instr/s) |",
       "|---|---|---|---|---|---|"]
for r in r2[2:]:
    f = float(r[h2.index("sm__cycles_elapsed.avg.per_second")].replace(",", ""))
    us = float(r[h2.index("gpu__time_duration.sum")].replace(",", ""))
    wi = float(r[h2.index("smsp__inst_executed.sum")].replace(",", ""))
    util = wi / (148 * 4 * f * 1e9 * us * 1e-6)
    clk.append(f"| `{r[h2.index('Kernel Name')].split('(')[0].split('::')[-1]}` | {us:.1f} | {f:.3f} | {wi / 1e6:.1f} M | "
               f"{100 * util:.1f} % | {148 * 128 * f / 1e3:.1f} |")
open(os.path.join(HERE, f"r{rnd}_summary.md"), "w").write("\n".join(head) + summ + "\n".join(clk) + "\n")
print("\n".join(head))
