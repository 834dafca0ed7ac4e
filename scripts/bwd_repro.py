"""Backward repro (debugging aid): python scripts/bwd_repro.py <config> <n> [use_forward_totals]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_12901_b200 import simuli as SM, synth
name = sys.argv[1]
n = int(sys.argv[2])
uft = len(sys.argv) < 4 or sys.argv[3] == "1"
if name in ("B", "C"):
    cfg, scene = synth.lidar_config(name), synth.scene_for(name, n=n)
    f = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
    f.requires_grad(True)
    f.scan(sync_capacity=True)
    g = {"opacity": torch.randn(f.n_rays, device="cuda")}
else:
    cam, scene = synth.camera_config(name), synth.scene_for("D", n=n)
    f = SM.CameraRenderer(cam, SM.to_device_scene(scene))
    f.requires_grad(True)
    f.frame(sync_capacity=True)
    R = cam.width * cam.height
    g = {"rgb": torch.randn(R, 3, device="cuda"), "opacity": torch.randn(R, device="cuda")}
torch.cuda.synchronize()
P = int(f.n_pairs.item())
rg = f.tile_ranges.cpu()
ids = f.sorted_ids[:P].cpu()
print("forward ok: pairs", P, "capacity", f.capacity, "ranges max", int(rg.max()), "min", int(rg.min()),
      "bad ranges", int((rg[:, 0] > rg[:, 1]).sum()), "ids max", int(ids.max()) if P else -1, "n", f.n, flush=True)
reps = int(os.environ.get("REPS", "1"))
for k in range(reps):
    out = f.backward(g, use_forward_totals=uft)
    torch.cuda.synchronize()
print("ok", name, n, uft, out["means"].abs().max().item(), flush=True)
