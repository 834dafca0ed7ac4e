"""Projection cost split (config B, L2 flushed): SH degree 3 vs 0, and culling modes --
bounds what the record / SH part and the culling cost inside k_project."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM, synth
cfg = synth.lidar_config("B")
sc = synth.scene_for("B")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
def t_proj(scene, **kw):
    r = SM.LidarRenderer(cfg, SM.to_device_scene(scene), **kw)
    r.scan(sync_capacity=True)
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r.project(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return np.median(ts) * 1e3
print("deg3 cull2", t_proj(sc))
sc0 = dict(sc); sc0["sh"] = np.ascontiguousarray(sc["sh"][:, :1, :])
print("deg0 cull2", t_proj(sc0))
print("deg3 cull0", t_proj(sc, enable_culling=0))
print("deg3 cull1", t_proj(sc, enable_culling=1))
print("deg3 write_all", t_proj(sc, write_all_records=True))
