"""Per-item timeline of the LiDAR render kernel (chunks = 32-entry chunks run) (profiling build: SIMULI_EXTRA_NVCC=-DSIMULI_RENDER_PROFILE)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import build as B
B.build(force=True)
from paper_2510_12901_b200 import simuli as SM, synth
name = sys.argv[1] if len(sys.argv) > 1 else "B"
cfg, scene = synth.lidar_config(name), synth.scene_for(name)
r = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
r.scan(sync_capacity=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_(); r.render()
torch.cuda.synchronize()
L = SM.load()
n = 1 << 18
buf = np.zeros(4 * n, np.int64)
L.simuli_debug_render_prof(buf.ctypes.data_as(C.c_void_p), C.c_int64(n))
p = buf.reshape(n, 4)
used = p[:, 1] > 0
p = p[used]
t0 = p[:, 0].min()
st, en, chunks = (p[:, 0] - t0) / 1e3, (p[:, 1] - t0) / 1e3, p[:, 2]
ln, sm = p[:, 3] & 0xffffffff, p[:, 3] >> 32
dur = en - st
print(f"items {used.sum()}, kernel span {en.max():.1f} us, last start {st.max():.1f} us")
print(f"item duration: mean {dur.mean():.2f} p50 {np.median(dur):.2f} p99 {np.percentile(dur, 99):.2f} max {dur.max():.2f} us")
print(f"chunks: total {chunks.sum()} mean {chunks.mean():.2f} max {chunks.max()}")
ok = chunks > 0
print(f"us per chunk (items with chunks): median {np.median(dur[ok] / chunks[ok]):.3f}, "
      f"weighted {dur[ok].sum() / chunks[ok].sum():.3f}")
for q in (0.5, 0.9, 0.99, 1.0):
    print(f"  items ending by {q:.2f} of span: {(en <= q * en.max()).mean():.3f}")
top = np.argsort(-dur)[:8]
print("longest items: dur", dur[top].round(1), "chunks", chunks[top], "len", ln[top], "start", st[top].round(1))
busy = np.zeros(200)
for s_, e_, m in zip(st, en, sm):
    busy[m] += e_ - s_
print(f"per-SM busy (sum of item durations): mean {busy[:148].mean():.1f} max {busy[:148].max():.1f} us")

ph = np.zeros(8, np.uint64)
if hasattr(L, "simuli_debug_render_phase"):
    L.simuli_debug_render_phase(ph.ctypes.data_as(C.c_void_p))
    names = ["cons wait full", "cons chain", "prod wait cp.async", "prod [A]", "prod wait empty", "prod [B]"]
    runs = 4  # renders since the kernel start (scan + 3 timed)
    print("phase cycles per render (summed over warps):", ", ".join(f"{n} {ph[i] / runs / 1e6:.1f} M" for i, n in enumerate(names)))
