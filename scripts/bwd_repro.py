"""Small LiDAR backward repro (debugging aid): config B sensor, n particles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_12901_b200 import simuli as SM, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
cfg, scene = synth.lidar_config("B"), synth.scene_for("B", n=n)
f = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
f.requires_grad(True)
f.scan(sync_capacity=True)
torch.cuda.synchronize()
g = {"opacity": torch.randn(f.n_rays, device="cuda")}
out = f.backward(g)
torch.cuda.synchronize()
print("ok", out["means"].abs().max().item())
