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
open(os.path.join(HERE, f"r{rnd}_summary.md"), "w").write("\n".join(head) + summ)
print("\n".join(head))
