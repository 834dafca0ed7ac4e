"""Camera render-only timing of config D (CUDA events, L2 flushed, median)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM, synth
cam = synth.camera_config("D")
c = SM.CameraRenderer(cam, SM.to_device_scene(synth.scene_for("D")), per_ray_sh=os.environ.get("SIMULI_PER_RAY_SH") == "1")
c.frame(sync_capacity=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c.render(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"D render: median {np.median(ts[2:]):.1f} us")
