#!/usr/bin/env python
"""Config E: 64 Waymo-top-like LiDAR scans (C-type) + 64 KB-fisheye
rolling-shutter frames (D-type) of one 4M G_l + 4M G_c corridor scene, data-parallel.

    python scripts/batch_e.py                       # 1 GPU
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/batch_e.py

One process per GPU, scene replicated (same seed on every rank), scan / frame i on rank
i mod N; no collective on the data path.  Two timings, device time (CUDA events), max over
ranks:
  * render only: every scan / frame rendered back to back;
  * render + gather: each rank's outputs (LiDAR depth / intensity / ray drop / opacity,
    camera rgb / opacity / depth) gathered to rank 0 (NCCL all_gather_into_tensor; a device
    copy at N = 1) on a second stream, unit k's gather overlapping unit k + 1's render (two
    renderers per sensor alternate so a unit's buffers stay intact until its gather ends).
Every gathered unit is compared bit for bit with rank 0 rendering the same pose itself
(G = 1).  Prints one JSON line on rank 0; NCCL's communicator init is logged to stderr
(NCCL_DEBUG=INFO) so the rank count can be checked."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2510_12901_b200 import batch, simuli as SM, synth  # noqa: E402

N = int(os.environ.get("E_FRAMES", "64"))
ws, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if ws > 1:
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dist.init_process_group("nccl", init_method="env://")
scans, frames = synth.e_poses(N)
lscene = SM.to_device_scene(synth.scene_for("E-lidar"), dev)
cscene = SM.to_device_scene(synth.scene_for("E-camera"), dev)
lids = [SM.LidarRenderer(synth.lidar_config("C"), lscene, device=dev) for _ in range(2)]
cams = [SM.CameraRenderer(synth.camera_config("D"), cscene, device=dev) for _ in range(2)]
for x in lids + cams:
    x.keep_keys = False
mine = batch.shard_indices(N, ws, rank)
LKEYS, CKEYS = ("depth", "intensity", "raydrop", "opacity"), ("rgb", "opacity", "depth")
# size the pair buffers (one synchronising call per renderer and a few poses), then warm up
need_l = need_c = 0
for i in mine[:: max(1, len(mine) // 4)]:
    lids[0].scan(*scans[i], sync_capacity=True)
    cams[0].frame(*frames[i], sync_capacity=True)
    torch.cuda.synchronize()
    need_l, need_c = max(need_l, int(lids[0].n_pairs.item())), max(need_c, int(cams[0].n_pairs.item()))
for x in lids:
    x.set_capacity(int(need_l * 1.5) + 4096)
for x in cams:
    x.set_capacity(int(need_c * 1.5) + 4096)
for i in mine[:2]:
    lids[0].scan(*scans[i]); cams[0].frame(*frames[i])
torch.cuda.synchronize()


def pack(out, keys, dst=None):
    return torch.cat([out[k].reshape(-1) for k in keys], out=dst)


# gather buffers allocated up front (an allocation inside the timed loop would synchronise)
UNITS = max(len(batch.shard_indices(N, ws, r)) for r in range(ws))
SIZES = {"s": pack(lids[0].out, LKEYS).numel(), "f": pack(cams[0].out, CKEYS).numel()}
STAGE = {k: [torch.zeros(n, device=dev) for _ in range(2)] for k, n in SIZES.items()}
GBUF = {k: torch.zeros((UNITS, ws, n), device=dev) for k, n in SIZES.items()}


def run(gather: bool):
    """Render this rank's units (scans then frames); with gather, unit k's packed outputs go
    to rank 0 on a side stream while unit k + 1 renders.  Returns (ms scans, ms frames,
    gathered {('s'|'f', i): tensor} on rank 0)."""
    main, side = torch.cuda.current_stream(), torch.cuda.Stream(device=dev)
    got = {}
    res = []
    for kind, objs, poses, keys in (("s", lids, scans, LKEYS), ("f", cams, frames, CKEYS)):
        done = [None, None]  # per renderer: event after its last gather
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        slot = 0
        for k in range(max(len(batch.shard_indices(N, ws, r)) for r in range(ws))):
            have = k < len(mine)
            obj = objs[slot]
            if done[slot] is not None:
                main.wait_event(done[slot])  # its previous unit has been gathered
            if have:
                i = mine[k]
                (obj.scan if kind == "s" else obj.frame)(*poses[i])
            if gather:
                ev = torch.cuda.Event()
                ev.record(main)
                with torch.cuda.stream(side):
                    side.wait_event(ev)
                    buf = STAGE[kind][slot]
                    if have:
                        pack(obj.out, keys, buf)
                    if ws > 1:
                        dist.all_gather_into_tensor(GBUF[kind][k], buf)
                    else:
                        GBUF[kind][k][0].copy_(buf)
                    de = torch.cuda.Event()
                    de.record(side)
                    done[slot] = de
            slot ^= 1
        ej = torch.cuda.Event()
        ej.record(side)
        main.wait_event(ej)
        e1.record(main)
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1))
        if gather and rank == 0:
            for r in range(ws):
                for k, i in enumerate(batch.shard_indices(N, ws, r)):
                    got[(kind, i)] = GBUF[kind][k][r]
    return res[0], res[1], got


if ws > 1:
    dist.barrier()
t_s, t_f, _ = run(False)
t_sg, t_fg, got = run(True)
mx = [batch.reduce_max(v, dev) for v in (t_s, t_f, t_sg, t_fg)]
over = batch.reduce_max(max(max(x.check_capacity() > x.capacity for x in lids + cams), 0), dev)
if rank == 0:
    ok = True
    for (kind, i), v in sorted(got.items()):
        obj = lids[0] if kind == "s" else cams[0]
        out = obj.scan(*scans[i]) if kind == "s" else obj.frame(*frames[i])
        ok &= torch.equal(pack(out, LKEYS if kind == "s" else CKEYS), v)
    line = {"workload": "E: 64 C-type LiDAR scans (64x2650) + 64 D-type fisheye frames (1920x1080) of one 4M G_l + "
                        "4M G_c corridor scene, round-robin over ranks",
            "n_gpus": ws,
            "render_only": {"scans_per_s": N / (mx[0] * 1e-3), "frames_per_s": N / (mx[1] * 1e-3),
                            "rays_per_s": N * lids[0].n_rays / (mx[0] * 1e-3),
                            "pixels_per_s": N * cams[0].cam_cfg.width * cams[0].cam_cfg.height / (mx[1] * 1e-3)},
            "render_plus_gather": {"scans_per_s": N / (mx[2] * 1e-3), "frames_per_s": N / (mx[3] * 1e-3)},
            "gathered_units": len(got), "gather_identical": bool(ok), "capacity_exceeded": bool(over),
            "gather": "NCCL all_gather_into_tensor per unit on a side stream (device copy at N = 1), overlapped with "
                      "the next unit's render; LiDAR depth/intensity/raydrop/opacity, camera rgb/opacity/depth",
            "timing": "device time (CUDA events on the launching stream), max over ranks; inputs > L2"}
    print(json.dumps(line), flush=True)
if ws > 1:
    dist.destroy_process_group()
