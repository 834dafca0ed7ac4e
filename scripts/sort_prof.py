"""Per-partition timeline of the onesweep passes on config B (profiling build:
SIMULI_EXTRA_NVCC=-DSIMULI_SORT_PROFILE)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import build as B
B.build(force=True)
from paper_2510_12901_b200 import simuli as SM, synth
cfg = synth.lidar_config("B")
r = SM.LidarRenderer(cfg, SM.to_device_scene(synth.scene_for("B")))
r.keep_keys = False
r.scan(sync_capacity=True)
for _ in range(3):
    r.bin_sort()
torch.cuda.synchronize()
L = SM.load()
buf = np.zeros(6 * 4096 * 8, np.int64)
L.simuli_debug_sort_prof(buf.ctypes.data_as(C.c_void_p))
p = buf.reshape(6, 4096, 8)
names = ["load", "rank", "publish", "lookback", "scatter"]
for ps in range(6):
    q = p[ps][p[ps][:, 7] == 1]
    if len(q) == 0:
        continue
    t0 = q[:, 0].min()
    span = (q[:, 5].max() - t0) / 1e3
    ph = np.diff(q[:, :6], axis=1) / 1e3
    print(f"pass {ps}: partitions {len(q)}, span {span:.1f} us, last start {(q[:, 0].max() - t0) / 1e3:.1f} us; "
          + ", ".join(f"{n} mean {ph[:, i].mean():.2f} max {ph[:, i].max():.2f}" for i, n in enumerate(names))
          + f"; rank clock64 cycles mean {q[:, 6].mean():.0f} p50 {np.median(q[:, 6]):.0f} max {q[:, 6].max():.0f}")
    order = np.argsort(q[:, 0])
    lb_end = (q[:, 4] - t0) / 1e3
    idx = np.arange(len(q))
    for f in (0.1, 0.25, 0.5, 0.75, 0.9, 1.0):
        k = min(len(q) - 1, int(f * (len(q) - 1)))
        print(f"   partition {k:5d}: start {(q[k, 0] - t0) / 1e3:6.2f} ranked {(q[k, 2] - t0) / 1e3:6.2f} "
              f"lookback done {lb_end[k]:6.2f} end {(q[k, 5] - t0) / 1e3:6.2f} us")
