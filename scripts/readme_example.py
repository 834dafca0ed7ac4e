"""The README usage example, runnable from the repo root: python scripts/readme_example.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_12901_b200 import simuli as SM, synth

cfg, scene = synth.lidar_config("B"), synth.scene_for("B")      # Pandar64-like, 2M particles
lidar = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
out = lidar.scan(cfg.pose_start, cfg.pose_end, sync_capacity=True)  # project -> bin_sort -> render
depth, intensity, raydrop = out["depth"], out["intensity"], out["raydrop"]

lidar.requires_grad(True)                                        # keep the view vectors
lidar.scan(sync_capacity=True)
grads = lidar.backward({"depth": torch.randn_like(out["depth"])})  # d/d(means, quats, scales, opacity, sh)
torch.cuda.synchronize()
print({k: float(v.abs().max()) for k, v in grads.items()}, float(depth.max()))
