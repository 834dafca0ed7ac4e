"""Eq. 2 composition timing on config D (CUDA events, L2 flushed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM, synth
cam = synth.camera_config("D")
c = SM.CameraRenderer(cam, SM.to_device_scene(synth.scene_for("D", n=200_000)))
c.frame(sync_capacity=True)
rng = np.random.default_rng(3)
env = torch.from_numpy(rng.uniform(0, 1, (512, 1024, 3)).astype(np.float32)).cuda()
grid = torch.from_numpy((np.eye(3, 4).reshape(1, 1, 1, 12) + 0.05 * rng.normal(size=(8, 16, 16, 12))).astype(np.float32)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for args in ((env, grid), (env, None), (None, grid)):
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c.compose(*args); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print("env" if args[0] is not None else "-", "grid" if args[1] is not None else "-", f"{np.median(ts[2:]):.1f} us")
