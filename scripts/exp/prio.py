"""Experiment: stream priorities for the stages of in-flight scans (config B headline regime).

Modes (S renderers / scans in flight, scan i on slot i mod S):
  base        one default-priority stream per slot (bench.py's headline)
  split_hi    projection on a low-priority stream, bin_sort + render on a high-priority
              stream of the same slot (event join)
  split_lo    the reverse (projection high, sort + render low)
  render_hi   projection + bin_sort low, render high
Prints rays/s per mode (device time between events on the main stream)."""
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_12901_b200 import simuli as SM, synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    SM.load()
    cfg = synth.lidar_config("B")
    scene = SM.to_device_scene(synth.scene_for("B"), dev)
    S = int(os.environ.get("S", "6"))
    n = int(os.environ.get("N", "300"))
    rs = [SM.LidarRenderer(cfg, scene, device=dev) for _ in range(S)]
    for x in rs:
        x.keep_keys = False
    my = bench.shard_poses(n + 40, 1, 0)
    r = rs[0]
    need = 0
    for p0, p1 in my[::40]:
        r.scan(p0, p1, sync_capacity=True)
        torch.cuda.synchronize()
        need = max(need, int(r.n_pairs.item()))
    for x in rs:
        x.set_capacity(int(need * 1.3) + 4096)
    lo, hi = torch.cuda.Stream.priority_range()  # (lowest, highest) numerically (0, -k)
    main_s = torch.cuda.current_stream()
    base = [torch.cuda.Stream(device=dev) for _ in range(S)]
    slo = [torch.cuda.Stream(device=dev, priority=lo) for _ in range(S)]
    shi = [torch.cuda.Stream(device=dev, priority=hi) for _ in range(S)]

    def one(mode, i, p):
        x = rs[i % S]
        x.set_poses(*p)
        if mode == "base":
            x.project(base[i % S]); x.bin_sort(base[i % S]); x.render(base[i % S])
            return
        a, b = {"split_hi": (slo, shi), "split_lo": (shi, slo), "render_hi": (slo, shi)}[mode]
        sa, sb = a[i % S], b[i % S]
        # sb must not start slot i's next scan before sa's previous one finished with the buffers:
        # stream order within each stream + the join below keep slot buffers ordered
        sa.wait_stream(sb)
        x.project(sa)
        if mode == "render_hi":
            x.bin_sort(sa)
        sb.wait_stream(sa)
        if mode != "render_hi":
            x.bin_sort(sb)
        x.render(sb)

    res = {}
    for rep in range(2):
        for mode in os.environ.get("MODES", "base,split_hi,split_lo,render_hi").split(","):
            for i in range(20):
                one(mode, i, my[i])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            for st in base + slo + shi:
                st.wait_event(e0)
            h0 = time.perf_counter()
            for i in range(n):
                one(mode, i, my[20 + i])
            host_us = (time.perf_counter() - h0) / n * 1e6
            for st in base + slo + shi:
                ej = torch.cuda.Event()
                ej.record(st)
                main_s.wait_event(ej)
            e1.record(main_s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            res.setdefault(mode + "_host_us_per_scan", []).append(round(host_us, 1))
            res.setdefault(mode, []).append(round(n * cfg.n_rays_total / (ms * 1e-3) / 1e6, 1)
                                            if hasattr(cfg, "n_rays_total") else round(n * 115200 / (ms * 1e-3) / 1e6, 1))
            for x in rs:
                x.check_capacity()
    print("S", S, "priority range", (lo, hi))
    for k, v in res.items():
        print(f"{k:10s} M rays/s {v}")


if __name__ == "__main__":
    main()
