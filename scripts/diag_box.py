"""Diagnostic: GPU vs oracle LiDAR box edges (absolute and in float32 ulps)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import synth as S, simuli as SM
from oracle import oracle as O

for name, n in (("A", None), ("B", 300_000), ("C", 300_000)):
    cfg = S.lidar_config(name)
    scene = S.scene_for(name, n=n) if n else S.scene_for(name)
    r = SM.LidarRenderer(cfg, SM.to_device_scene(scene), write_all_records=True)
    r.scan(sync_capacity=True); torch.cuda.synchronize()
    rec = r.record.cpu().numpy()
    proj = O.project_lidar(scene, cfg)
    gv = np.isfinite(rec[:, 16]); ov = proj["valid"] != 0; amb = proj["ambiguous"] != 0
    both = gv & ov & ~amb
    g = rec[both, 16:20]; o = proj["box"][both]
    dab = np.abs(g.astype(np.float64) - o)
    ulp = np.abs(g.view(np.int32).astype(np.int64) - o.view(np.int32).astype(np.int64))
    print(name, "valid mismatch", int((gv[~amb] != ov[~amb]).sum()), "n", int(both.sum()))
    for c in range(4):
        print(f"  edge {c}: abs max {dab[:, c].max():.3e}  ulps max {ulp[:, c].max()}  frac!=0 {(ulp[:, c] > 0).mean():.4f}"
              f"  frac>1 {(ulp[:, c] > 1).mean():.6f}")
