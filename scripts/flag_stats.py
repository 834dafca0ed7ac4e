"""A23 flag accounting on the full-size configs (GPU box: the GPU's projection + the CPU
oracle on the host cores).  For B and C (LiDAR) and D (camera):
  * how far the GPU's float32 boxes are from the oracle's for the non-ambiguous and for the
    validity-ambiguous particles (the evidence the listing margin of ambiguous particles
    needs), and how many particles' validity differs;
  * tier-2 flags by kind (bit 1 box edge, 2 alpha_min, 4 T_min, 8 validity-ambiguous,
    16 near plane) on a sample of tiles, at the test margins and with the ambiguous-particle
    listing margin shrunk to a multiple of the measured box error.
Usage: python scripts/flag_stats.py > profiles/r02_flag_stats.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2510_12901_b200 import simuli as SM, synth  # noqa: E402

LIDAR_EPS = {"a": 3e-7, "b": 3e-7, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4, "impact": 5e-6}
CAMERA_EPS = {"a": 5e-4, "b": 5e-4, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4, "impact": 5e-6}
BITS = {1: "box_edge", 2: "alpha_min", 4: "T_min", 8: "validity_ambiguous", 16: "near_plane"}
O.build()
O.set_threads(os.cpu_count() or 1)


def kinds(flag):
    return {name: int(((flag & b) != 0).sum()) for b, name in BITS.items()} | {
        "any": int((flag != 0).sum()), "rays": int(flag.shape[0]), "share": float((flag != 0).mean())}


def box_err(gpu_box, gpu_valid, proj):
    ov, amb = proj["valid"] != 0, proj["ambiguous"] != 0
    both = gpu_valid & ov & np.isfinite(proj["box"]).all(1)
    d = np.abs(gpu_box.astype(np.float64) - proj["box"].astype(np.float64))
    d[:, :2] = np.minimum(d[:, :2], 2 * np.pi - d[:, :2]) if gpu_box.shape[1] == 4 else d[:, :2]
    out = {"n": int(gpu_box.shape[0]), "n_ambiguous": int(amb.sum()),
           "validity_differs": int((gpu_valid != ov).sum()),
           "validity_differs_non_ambiguous": int(((gpu_valid != ov) & ~amb).sum()),
           "max_box_err_non_ambiguous": float(d[both & ~amb].max(initial=0)),
           "max_box_err_ambiguous_both_valid": float(d[both & amb].max(initial=0))}
    return out


def lidar(name, n_tiles_sample=64):
    cfg, scene = synth.lidar_config(name), synth.scene_for(name)
    r = SM.LidarRenderer(cfg, SM.to_device_scene(scene), write_all_records=True)
    r.want_ray_od(True)
    r.scan(sync_capacity=True)
    torch.cuda.synchronize()
    rec = r.record.cpu().numpy()
    proj = O.project_lidar(scene, cfg)
    res = {"projection": box_err(rec[:, 16:20], np.isfinite(rec[:, 16]), proj)}
    t = O.Tiling(cfg)
    rng = np.random.default_rng(3)
    tiles = rng.choice(t.n_tiles, n_tiles_sample, replace=False)
    rays = np.concatenate([t.tile_rays[t.tile_ray_offsets[x]:t.tile_ray_offsets[x + 1]] for x in tiles])
    rec2 = O.records_from_projection(proj, scene)
    od2 = O.lidar_rays(t, cfg.pose_start, cfg.pose_end)[rays]
    amb = proj["ambiguous"] != 0
    listed = ((proj["valid"] != 0) | amb) & np.isfinite(proj["box"]).all(1)
    gamb = np.where(amb, np.where(proj["valid"] != 0, 1, 2), 0).astype(np.int32)
    res["tier2"] = {}
    margins = {"test (0.1, 0.02) rad": O.AMBIGUOUS_MARGIN}
    m = max(res["projection"]["max_box_err_ambiguous_both_valid"], 3e-7)
    margins[f"10 x measured ({10 * m:.2e} rad)"] = (10 * m, 10 * m)
    for label, (ma, mb) in margins.items():
        lbox = O.expand_box(proj["box"], LIDAR_EPS["a"], LIDAR_EPS["b"])
        lbox[amb] = O.expand_box(proj["box"][amb], ma, mb)
        count, rect = O.cull_lidar(listed.astype(np.int32), lbox, t, False)
        _, ids2, ranges2 = O.bin_pairs(count, rect, proj["key"], t.n_tiles, t.n_theta)
        ref2 = O.composite(rec2, ids2, ranges2, t.ray_tile[rays], t.ray_az[rays], t.ray_el[rays], od2, wrap=1,
                           near=cfg.min_range, gamb=gamb, flag_eps=dict(LIDAR_EPS, amb_a=ma, amb_b=mb),
                           pi_f=t.pi_f, two_pi_f=t.two_pi_f)
        res["tier2"][label] = kinds(ref2["flag"])
    res["sample"] = f"{n_tiles_sample} random tiles of {t.n_tiles}, {len(rays)} rays"
    return res


def camera(n_tiles_sample=48):
    cam, scene = synth.camera_config("D"), synth.scene_for("D")
    c = SM.CameraRenderer(cam, SM.to_device_scene(scene), write_all_records=True)
    c.frame(sync_capacity=True)
    torch.cuda.synchronize()
    rec = c.record.cpu().numpy()
    proj = O.project_camera(scene, cam)
    res = {"projection": box_err(rec[:, 16:20], np.isfinite(rec[:, 16]), proj)}
    Wt, Ht = O.camera_tiles(cam)
    rays = O.camera_rays(cam)
    rng = np.random.default_rng(4)
    tiles = rng.choice(Wt * Ht, n_tiles_sample, replace=False)
    sel = np.nonzero(np.isin(rays["tile"], tiles))[0]
    rs = {k: (v[sel] if isinstance(v, np.ndarray) and v.shape[:1] == (cam.width * cam.height,) else v)
          for k, v in rays.items()}
    rec2 = O.records_from_projection(proj, scene)
    amb = proj["ambiguous"] != 0
    listed = ((proj["valid"] != 0) | amb) & np.isfinite(proj["box"]).all(1)
    gamb = np.where(amb, np.where(proj["valid"] != 0, 1, 2), 0).astype(np.int32)
    res["tier2"] = {}
    m = max(res["projection"]["max_box_err_ambiguous_both_valid"], 5e-4)
    for label, mm in (("test 20 px", 20.0), (f"10 x measured ({10 * m:.2e} px)", 10 * m)):
        lbox = O.expand_box(proj["box"], CAMERA_EPS["a"], CAMERA_EPS["b"])
        lbox[amb] = O.expand_box(proj["box"][amb], mm, mm)
        count, rect = O.cull_camera(listed.astype(np.int32), lbox, cam)
        _, ids2, ranges2 = O.bin_pairs(count, rect, proj["key"], Wt * Ht, Wt)
        ref2 = O.composite(rec2, ids2, ranges2, rs["tile"], rs["u"], rs["v"], rs["od"], wrap=0, near=cam.near,
                           ray_valid=rs["valid"], gamb=gamb, flag_eps=dict(CAMERA_EPS, amb_a=mm, amb_b=mm))
        res["tier2"][label] = kinds(ref2["flag"])
    res["sample"] = f"{n_tiles_sample} random 16x16 tiles, {len(sel)} pixels"
    return res


out = {"what": "A23 flag accounting (scripts/flag_stats.py)", "cores": os.cpu_count()}
for name in ("B", "C"):
    t0 = time.perf_counter()
    out[name] = lidar(name)
    out[name]["seconds"] = time.perf_counter() - t0
    print(name, json.dumps(out[name]), file=sys.stderr, flush=True)
t0 = time.perf_counter()
out["D"] = camera()
out["D"]["seconds"] = time.perf_counter() - t0
print(json.dumps(out, indent=1))
