"""A3 (rolling-shutter firing-time fixed point, P:129 / P:139): how far the default K = 1
iteration is from the converged K = 8 on the B-batch trajectory (oracle, double precision).
Reports per pose the max difference of the UT mean azimuth / elevation and of the 3-sigma
box edges, the implied firing-time difference of the particle mean (|d view vector| / |t1 -
t0|: the sensor moves 1 m per sweep), and how many particles change tiles / validity.
Usage: python scripts/a3_bound.py [n_poses] > profiles/r02_a3_bound.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2510_12901_b200 import synth  # noqa: E402

n_poses = int(sys.argv[1]) if len(sys.argv) > 1 else 3
O.build()
O.set_threads(os.cpu_count() or 1)
cfg, scene = synth.lidar_config("B"), synth.scene_for("B")
t = O.Tiling(cfg)
poses = synth.batch_poses(512)
rows = []
for i in np.linspace(0, 511, n_poses).astype(int):
    p0, p1 = poses[i]
    t0 = time.perf_counter()
    a = O.project_lidar(scene, cfg, p0, p1, K=1)
    b = O.project_lidar(scene, cfg, p0, p1, K=8)
    both = (a["valid"] != 0) & (b["valid"] != 0)
    dm = np.abs(a["mean2d"][both] - b["mean2d"][both])
    dm[:, 0] = np.minimum(dm[:, 0], 2 * np.pi - dm[:, 0])
    db = np.abs(a["box"][both].astype(np.float64) - b["box"][both].astype(np.float64))
    db[:, :2] = np.minimum(db[:, :2], 2 * np.pi - db[:, :2])
    motion = float(np.linalg.norm(np.asarray(p1["t"], np.float64) - np.asarray(p0["t"], np.float64)))
    ds = np.linalg.norm(a["viewdir"][both] - b["viewdir"][both], axis=1) / motion
    ca, ra = O.cull_lidar(a["valid"], a["box"], t, 2)
    cb, rb = O.cull_lidar(b["valid"], b["box"], t, 2)
    rows.append({"pose": int(i), "x": float(p0["t"][0]), "n_valid_K1": int((a["valid"] != 0).sum()),
                 "validity_changed": int(((a["valid"] != 0) != (b["valid"] != 0)).sum()),
                 "max_dmean_az_rad": float(dm[:, 0].max()), "max_dmean_el_rad": float(dm[:, 1].max()),
                 "p99_dmean_az_rad": float(np.percentile(dm[:, 0], 99)),
                 "max_dbox_rad": float(db.max()), "max_ds_firing_time": float(ds.max()),
                 "p99_ds_firing_time": float(np.percentile(ds, 99)),
                 "tile_rect_changed": int((np.any(ra != rb, axis=1) | (ca != cb)).sum()),
                 "seconds": time.perf_counter() - t0})
    print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
out = {"what": "A3: K=1 (default) vs K=8 firing-time fixed-point iterations, oracle (double), config-B scene on "
               "B-batch poses (1 m / 0.03 rad per sweep)",
       "poses": rows,
       "bound": {k: max(r[k] for r in rows) for k in ("max_dmean_az_rad", "max_dmean_el_rad", "max_dbox_rad",
                                                     "max_ds_firing_time", "validity_changed", "tile_rect_changed")}}
print(json.dumps(out, indent=1))
