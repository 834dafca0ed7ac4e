"""Small driver for ncu captures of one stage kernel on config B (default: the LiDAR render).
Usage: ncu ... python scripts/ncu_render.py [config] [stage]   (stage: render | project | bin_sort)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_12901_b200 import simuli as SM, synth

name = sys.argv[1] if len(sys.argv) > 1 else "B"
stage = sys.argv[2] if len(sys.argv) > 2 else "render"
cfg, scene = synth.lidar_config(name), synth.scene_for(name)
r = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
r.keep_keys = False
p0, p1 = synth.batch_poses(210)[105]
r.scan(p0, p1, sync_capacity=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(4):
    flush.zero_()
    getattr(r, stage)()
torch.cuda.synchronize()
print("ok", stage)
