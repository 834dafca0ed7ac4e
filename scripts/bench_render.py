"""Render-only timing of config B (and a saved output for cross-kernel comparison).
Usage: SIMULI_LIDAR_KERNEL=<kind> [SIMULI_PER_RAY_SH=1] python scripts/bench_render.py [config] [out.npz]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM, synth

name = sys.argv[1] if len(sys.argv) > 1 else "B"
cfg, scene = synth.lidar_config(name), synth.scene_for(name)
per_ray = os.environ.get("SIMULI_PER_RAY_SH") == "1"
r = SM.LidarRenderer(cfg, SM.to_device_scene(scene), per_ray_sh=per_ray)
r.keep_keys = False
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
poses = synth.batch_poses(210)[::21] if name in ("B", "C") else [(cfg.pose_start, cfg.pose_end)]
per_pose = []
for p0, p1 in poses:  # the B-batch trajectory (bench.py's workload), 10 poses across it
    r.scan(p0, p1, sync_capacity=True)
    torch.cuda.synchronize()
    times = []
    for i in range(8):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r.render(); e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    per_pose.append(np.median(times[2:]))
kind = os.environ.get("SIMULI_LIDAR_RENDER", "split") + ":" + os.environ.get("SIMULI_LIDAR_VARIANT", "0") + (" per-ray SH" if per_ray else "")
print(f"{name} render[{kind}]: mean over {len(poses)} poses {np.mean(per_pose):.1f} us  "
      f"(min {np.min(per_pose):.1f}, max {np.max(per_pose):.1f})", flush=True)
if len(sys.argv) > 2:
    np.savez(sys.argv[2], **{k: v.cpu().numpy() for k, v in r.out.items() if v is not None})
