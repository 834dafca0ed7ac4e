"""Config D camera frame: per-stage device time (L2 flushed) and counters; used for tuning / ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM, synth
cam = synth.camera_config("D")
c = SM.CameraRenderer(cam, SM.to_device_scene(synth.scene_for("D")))
c.keep_keys = False
c.frame(sync_capacity=True)
c.want_counters(True)
c.frame()
torch.cuda.synchronize()
nv, ni, nc = (c.out[k].cpu().numpy().astype(np.int64) for k in ("n_visited", "n_inbox", "n_contrib"))
print(f"pairs {int(c.n_pairs.item())} tiles {c.n_tiles}; per pixel visited mean {nv.mean():.0f} max {nv.max()}, "
      f"in-box mean {ni.mean():.0f}, composited mean {nc.mean():.1f}; T<Tmin {(c.out['final_T'].cpu().numpy() < 1e-4).mean():.3f}")
c.want_counters(False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {"project": [], "bin_sort": [], "render": []}
for _ in range(int(os.environ.get("REPS", "8"))):
    for st in res:
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); getattr(c, st)(); e1.record(); torch.cuda.synchronize()
        res[st].append(e0.elapsed_time(e1) * 1e3)
print("D " + "  ".join(f"{k} {np.median(v):.1f} us" for k, v in res.items()))
