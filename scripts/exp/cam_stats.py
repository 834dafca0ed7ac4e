"""Config D: per-pixel member counts (in-box) and tile list lengths -- the camera render's tail."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM, synth
cam = synth.camera_config("D")
c = SM.CameraRenderer(cam, SM.to_device_scene(synth.scene_for("D")))
c.want_counters(True)
c.frame(sync_capacity=True)
torch.cuda.synchronize()
ni = c.out["n_inbox"].cpu().numpy().astype(np.int64).reshape(cam.height, cam.width)
nv = c.out["n_visited"].cpu().numpy().astype(np.int64).reshape(cam.height, cam.width)
rg = c.tile_ranges.cpu().numpy().reshape(-1, 2)
ln = rg[:, 1] - rg[:, 0]
print("inbox per pixel: mean %.1f p99 %d max %d" % (ni.mean(), np.percentile(ni, 99), ni.max()))
print("visited per pixel: mean %.1f p99 %d max %d" % (nv.mean(), np.percentile(nv, 99), nv.max()))
print("list len: mean %.1f p99 %d max %d; tiles > 5000: %d" % (ln.mean(), np.percentile(ln, 99), ln.max(), (ln > 5000).sum()))
# per 2x16 strip: max member count over its 32 pixels (the warp's critical path)
H, W = cam.height // 2 * 2, cam.width // 16 * 16
s = ni[:H, :W].reshape(H // 2, 2, W // 16, 16).max(axis=(1, 3))
tot = ni[:H, :W].reshape(H // 2, 2, W // 16, 16).sum(axis=(1, 3))
print("strip max-member: mean %.1f p99 %d max %d; strip total members mean %.0f max %d" % (s.mean(), np.percentile(s, 99), s.max(), tot.mean(), tot.max()))
print("sum of members %d; the busiest strip's max-member / mean strip total: %.1f" % (ni.sum(), s.max() / tot.mean()))
