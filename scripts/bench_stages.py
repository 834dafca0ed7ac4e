"""Per-stage device time (project / bin_sort / render) over 10 poses of the B-batch
trajectory, L2 flushed before every stage launch.  Usage: python scripts/bench_stages.py [config]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM, synth

name = sys.argv[1] if len(sys.argv) > 1 else "B"
cfg, scene = synth.lidar_config(name), synth.scene_for(name)
r = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
r.keep_keys = False
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
poses = synth.batch_poses(210)[::21] if name == "B" else [(cfg.pose_start, cfg.pose_end)]
res = {"project": [], "bin_sort": [], "render": []}
for p0, p1 in poses:
    r.scan(p0, p1, sync_capacity=True)
    torch.cuda.synchronize()
    for stage in res:
        t = []
        for i in range(6):
            flush.zero_()
            if stage == "render":
                pass
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); getattr(r, stage)(); e1.record()
            torch.cuda.synchronize()
            t.append(e0.elapsed_time(e1) * 1e3)
        res[stage].append(np.median(t[1:]))
tag = os.environ.get("TAG", "")
print(f"{name} {tag} " + "  ".join(f"{k} {np.mean(v):.1f} us (min {np.min(v):.1f} max {np.max(v):.1f})"
                                    for k, v in res.items()), flush=True)
