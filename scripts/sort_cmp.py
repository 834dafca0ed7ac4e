"""Device time of simuli_bin_sort on one config-B projection (L2 warm, back to back)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_12901_b200 import simuli as SM, synth
cfg = synth.lidar_config("B")
r = SM.LidarRenderer(cfg, SM.to_device_scene(synth.scene_for("B")))
r.keep_keys = False
r.scan(sync_capacity=True)
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", "30"))
for _ in range(3):
    r.bin_sort()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    r.bin_sort()
e1.record()
torch.cuda.synchronize()
print(f"simuli_bin_sort config B P={int(r.n_pairs.item())}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us (L2 warm)")
