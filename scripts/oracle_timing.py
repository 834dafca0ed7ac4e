"""SURVEY §8(d) oracle timing beside the GPU numbers: the CPU oracle (oracle/, double
precision, OpenMP) as it stands, on this machine's host cores and on one core.
  A: tiled + brute force, 3 runs each; B and C: one full tiled scan; D: the 480x270 centre
  crop (all particles projected / binned, the crop's pixels composited), extrapolated per
  pixel to 1920x1080 (the survey's crop rule).
Usage: python scripts/oracle_timing.py > profiles/r02_oracle_timing.json"""
import json
import os
import platform
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2510_12901_b200 import synth  # noqa: E402

O.build()
cores = len(os.sched_getaffinity(0))


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        return {k.strip(): v.strip() for k, v in (ln.split(":", 1) for ln in out.splitlines() if ":" in ln)
                if k.strip() in ("Model name", "CPU(s)", "Thread(s) per core", "Core(s) per socket", "Socket(s)")}
    except Exception:
        return {"platform": platform.processor()}


def timed(fn, runs=1):
    ts = []
    for _ in range(runs):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return ts


res = {"what": "CPU oracle timings (scripts/oracle_timing.py)", "nproc": os.cpu_count(), "affinity_cores": cores,
       "lscpu": cpu_model()}
for threads in (cores, 1):
    O.set_threads(threads)
    key = f"{threads}_threads"
    r = {}
    cfg, scene = synth.lidar_config("A"), synth.scene_for("A")
    t = O.Tiling(cfg)
    for mode in ("tiled", "brute"):
        ts = timed(lambda: O.render_lidar(scene, cfg, tiling=t, mode=mode), 3)
        r[f"A_{mode}"] = {"seconds": ts, "rays_per_s": cfg.n_rays / float(np.median(ts))}
    for name in ("B", "C"):
        if threads == 1 and name == "C":
            continue  # ~1 min on one core; B gives the one-core rate
        cfg, scene = synth.lidar_config(name), synth.scene_for(name)
        t = O.Tiling(cfg)
        ts = timed(lambda: O.render_lidar(scene, cfg, tiling=t))
        r[name] = {"seconds": ts, "rays_per_s": cfg.n_rays / ts[0]}
    if threads == cores:
        cam, scene = synth.camera_config("D"), synth.scene_for("D")
        rays = O.camera_rays(cam)
        W, H, cw, ch = cam.width, cam.height, 480, 270
        x0, y0 = (W - cw) // 2, (H - ch) // 2
        pix = (np.arange(y0, y0 + ch)[:, None] * W + np.arange(x0, x0 + cw)[None, :]).ravel()

        def crop():
            proj = O.project_camera(scene, cam)
            rec = O.records_from_projection(proj, scene)
            Wt, Ht = O.camera_tiles(cam)
            count, rect = O.cull_camera(proj["valid"], proj["box"], cam)
            _, ids, ranges = O.bin_pairs(count, rect, proj["key"], Wt * Ht, Wt)
            O.composite(rec, ids, ranges, rays["tile"][pix], rays["u"][pix], rays["v"][pix], rays["od"][pix], wrap=0,
                        near=cam.near, ray_valid=rays["valid"][pix])
        ts = timed(crop)
        r["D_crop_480x270"] = {"seconds": ts, "pixels_per_s": len(pix) / ts[0],
                               "extrapolated_full_frame_s": ts[0] * (W * H) / len(pix),
                               "note": "projection + binning of all 2M particles included in the crop time, so the "
                                       "per-pixel extrapolation overestimates the full frame slightly"}
    res[key] = r
    print(key, json.dumps(r), file=sys.stderr, flush=True)
print(json.dumps(res, indent=1))
