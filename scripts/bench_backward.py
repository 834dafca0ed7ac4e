"""Backward (A31) timing at full size: config B (LiDAR, 2M) and D (camera 1920x1080, 2M).
Forward once, then the backward timed alone with CUDA events (L2 flushed before each)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM, synth

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts[2:])


for name in sys.argv[1:] or ["B", "D"]:
    if name in ("B", "C"):
        cfg, scene = synth.lidar_config(name), synth.scene_for(name)
        f = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
        f.requires_grad(True)
        f.scan(sync_capacity=True)
        R = f.n_rays
        g = {k: torch.randn(R, device="cuda") for k in ("opacity", "depth", "intensity", "raydrop")}
        g["zeta"] = torch.randn(R, 3, device="cuda")
        fwd = timed(lambda: f.scan())
    else:
        cam, scene = synth.camera_config(name), synth.scene_for(name)
        f = SM.CameraRenderer(cam, SM.to_device_scene(scene))
        f.requires_grad(True)
        f.frame(sync_capacity=True)
        R = cam.width * cam.height
        g = {"rgb": torch.randn(R, 3, device="cuda"), "opacity": torch.randn(R, device="cuda")}
        fwd = timed(lambda: f.frame())
    torch.cuda.synchronize()
    bwd = timed(lambda: f.backward(g))
    bwd1 = timed(lambda: f.backward(g, use_forward_totals=False))
    print(f"{name}: forward {fwd:.1f} us, backward {bwd:.1f} us ({bwd / fwd:.2f}x forward; {bwd1:.1f} us with its own totals pass)", flush=True)
