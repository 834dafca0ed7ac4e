#!/usr/bin/env python
"""Config E: 64 Waymo-top-like LiDAR scans (C-type) + 64 KB-fisheye
rolling-shutter frames (D-type) of one 4M G_l + 4M G_c corridor scene, data-parallel.

    python scripts/batch_e.py                       # 1 GPU
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/batch_e.py

One process per GPU, scene replicated (same seed on every rank), scan / frame i on rank
i mod N; no collective on the data path.  Timed on the device (CUDA events around every
scan and frame, max over ranks).  Then a spot check: scans / frames 0, 17, 34, 51 (one per
rank up to 4 ranks) are all_gather-ed to rank 0 (NCCL) and must be bit-identical to rank 0
rendering them itself.
Prints one JSON line on rank 0."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2510_12901_b200 import batch, simuli as SM, synth  # noqa: E402

N = int(os.environ.get("E_FRAMES", "64"))
ws, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if ws > 1:
    dist.init_process_group("nccl", init_method="env://")
scans, frames = synth.e_poses(N)
lid = SM.LidarRenderer(synth.lidar_config("C"), SM.to_device_scene(synth.scene_for("E-lidar"), dev), device=dev)
cam = SM.CameraRenderer(synth.camera_config("D"), SM.to_device_scene(synth.scene_for("E-camera"), dev), device=dev)
lid.keep_keys = cam.keep_keys = False
mine = batch.shard_indices(N, ws, rank)
SPOT = [i for i in range(0, N, 17)]  # spot j = frame 17 j lives on rank j mod ws
# size the pair buffers (one synchronising call per renderer and a few poses), then warm up
for i in mine[:: max(1, len(mine) // 4)]:
    lid.scan(*scans[i], sync_capacity=True)
    cam.frame(*frames[i], sync_capacity=True)
torch.cuda.synchronize()
lid.set_capacity(int(lid.n_pairs.item() * 1.5) + 4096)
cam.set_capacity(int(cam.n_pairs.item() * 1.5) + 4096)
for i in mine[:2]:
    lid.scan(*scans[i]); cam.frame(*frames[i])
torch.cuda.synchronize()


def timed(fn, poses, keep):
    ev, outs = [], {}
    for i in mine:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); out = fn(*poses[i]); e1.record()
        ev.append((e0, e1))
        if i in SPOT:
            outs[SPOT.index(i)] = out[keep].clone()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev), outs


if ws > 1:
    dist.barrier()
t_scan, scan_out = timed(lid.scan, scans, "opacity")
t_frame, frame_out = timed(cam.frame, frames, "rgb")
t_scan_max = batch.reduce_max(t_scan, dev)
t_frame_max = batch.reduce_max(t_frame, dev)
over = batch.reduce_max(max(int(lid.n_pairs.item()) > lid.capacity, int(cam.n_pairs.item()) > cam.capacity), dev)
# spot check: gather the SPOT scans / frames to rank 0 and compare with rank 0's own render
g0 = time.perf_counter()
gs = batch.gather_frames(scan_out, len(SPOT), dev)
gf = batch.gather_frames(frame_out, len(SPOT), dev)
g_ms = 1e3 * (time.perf_counter() - g0)
if rank == 0:
    ok = True
    for j, i in enumerate(SPOT):
        ok &= torch.equal(lid.scan(*scans[i])["opacity"], gs[j].to(dev))
        ok &= torch.equal(cam.frame(*frames[i])["rgb"], gf[j].to(dev))
    line = {"workload": "E: 64 C-type LiDAR scans (64x2650) + 64 D-type fisheye frames (1920x1080) of one 4M G_l + "
                        "4M G_c corridor scene, round-robin over ranks",
            "n_gpus": ws, "scans_per_s": N / (t_scan_max * 1e-3), "frames_per_s": N / (t_frame_max * 1e-3),
            "rays_per_s": N * lid.n_rays / (t_scan_max * 1e-3),
            "pixels_per_s": N * cam.cam_cfg.width * cam.cam_cfg.height / (t_frame_max * 1e-3),
            "ms_per_scan_per_rank": t_scan_max / len(mine), "ms_per_frame_per_rank": t_frame_max / len(mine),
            "capacity_exceeded": bool(over), "spot_check_gather_ms": g_ms, "spot_check_identical": bool(ok),
            "timing": "device time (CUDA events around each scan / frame), max over ranks; inputs > L2"}
    print(json.dumps(line), flush=True)
if ws > 1:
    dist.destroy_process_group()
