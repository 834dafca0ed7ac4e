"""Throughput with S scans in flight (S renderers, S streams) vs one at a time, config B."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM, synth

cfg = synth.lidar_config("B")
scene = SM.to_device_scene(synth.scene_for("B"))
poses = synth.batch_poses(512)
K = 120
for S in (1, 2, 3, 4):
    rs = [SM.LidarRenderer(cfg, scene) for _ in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    for r in rs:
        r.keep_keys = False
        r.scan(*poses[0], sync_capacity=True)
    torch.cuda.synchronize()
    cap = max(int(r.n_pairs.item()) for r in rs)
    for r in rs:
        r.set_capacity(int(cap * 1.4) + 4096)
    for i in range(6):
        rs[i % S].scan(*poses[i], stream=streams[i % S])
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for st in streams:
        st.wait_event(e0)
    for i in range(K):
        rs[i % S].scan(*poses[(10 + i) % 512], stream=streams[i % S])
    for st in streams:
        ev = torch.cuda.Event()
        ev.record(st)
        main.wait_event(ev)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"S={S}: {ms:.3f} ms/scan  {cfg.n_azimuth * len(cfg.beams) / ms / 1e3:.1f} M rays/s", flush=True)
    del rs
    torch.cuda.empty_cache()
