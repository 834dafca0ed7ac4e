#!/usr/bin/env python
"""Benchmark of the SimULi forward LiDAR hot path on B200 (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W [--impl reference]

A step = one full LiDAR scan of BASELINE.json configs[1] ("B": Pandar64-like 64 x 1800
rays, rolling-shutter spin pose interpolation, 2M Gaussians): simuli_project ->
simuli_bin_sort -> simuli_render_lidar through the C ABI, scene resident in HBM.  Scans
of the B-batch trajectory (512 poses 0.2 m apart) are sharded round-robin
over ranks (weak scaling: K scans per rank); there is no collective on the data path, NCCL
only reduces the timers / counters.

Prints ONE JSON line on rank 0.  value = whole-job LiDAR rays/s (scans/s in
``scans_per_s``): the K timed scans run six in flight per GPU (six renderers with their
own buffers on six streams, shared resident scene -- one scan's latency-bound stages
overlap the others'; with the default kernels 5 / 6 / 8 in flight measured 301 / 305 /
301 M rays/s), timed between two CUDA events on the launching stream,
bracketed by barrier + synchronize, max over ranks; inputs exceed the L2, so no flush.  A
second pass runs scans one at a time with the L2 flushed and per-stage CUDA events: the
stage breakdown and roofline, and ``latency_ms_per_scan``; a third the same with the
latency-optimised render shape (``latency_mode``).
``--impl reference`` times the CPU oracle (oracle/, test infrastructure) on a bounded
sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2510_12901_b200 import batch, synth  # noqa: E402

METRIC = "LiDAR rays/sec and scans/sec (64-beam, 2M Gaussians) at 1/2/4/8 B200; % roofline"
UNIT = "rays/s"
WORKLOAD = ("B: PandaSet-like Pandar64 scan, 64x1800 rays, 2M Gaussians (driving corridor), rolling-shutter "
            "spin pose interpolation (1 m, 0.03 rad per sweep), K=1 fixed-point iteration, N_phi=16, M=32")

# Algorithmic lane-instruction costs per compositing event; the counts
# come from the kernel's own workload counters (entries visited / in box / composited).
C_BOX, C_RESP, C_ACC, C_RAY = 8, 45, 8, 80
# SURVEY §8(d) projection instruction model (lane-instructions): per sigma point C_PROJ
# (transform + atan2 + asin + sqrt) and, per rolling-shutter iteration, C_PROJ + C_POSE;
# per particle C_UT + C_MISC; per visible particle C_SH
C_PROJ, C_POSE, C_UT, C_MISC, C_SH = 75, 60, 60, 240, 90


def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return {"hbm_gbs": float(p["hbm_gbs"]), "sm_max_mhz": float(p.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region by a separate process (an
    NVML poll every 0.5 ms, monotonic timestamps, written to a temp file; a thread of this
    process would need the GIL the launch loop holds) and kept for the window
    [mark_begin, mark_end]; falls back to ``nvidia-smi -lms 100`` if NVML is unavailable."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))
    POLL = (
        "import sys, time\n"
        "import pynvml as n\n"
        "n.nvmlInit(); h = n.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))\n"
        "smax = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)\n"
        "out = open(sys.argv[2], 'w', buffering=1)\n"
        "out.write('ready\\n')\n"
        "while True:\n"
        "    out.write('%.6f %d %d %d\\n' % (time.monotonic(), n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM), smax,\n"
        "              n.nvmlDeviceGetCurrentClocksEventReasons(h)))\n"
        "    time.sleep(0.0005)\n")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []  # (t, sm_mhz, max_mhz, reasons bitmask)
        self.proc = None
        self.path = None
        self.window = [None, None]
        self.source = "nvml 0.5 ms (poller process)"

    def start(self):
        import tempfile
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
        fd, self.path = tempfile.mkstemp(prefix="bench_clk_", suffix=".txt")
        os.close(fd)
        try:
            import pynvml  # noqa: F401  (the poller imports it too)
            self.err_path = self.path + ".err"
            self.proc = subprocess.Popen([sys.executable, "-c", self.POLL, str(idx), self.path],
                                         stdout=subprocess.DEVNULL, stderr=open(self.err_path, "w"))
        except Exception:
            self.source = "nvidia-smi 100 ms"
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(idx), "--query-gpu=timestamp,clocks.sm,clocks.max.sm,"
                                          "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms",
                                          "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        t0 = time.monotonic()
        while time.monotonic() - t0 < 20.0:  # wait for the poller's first line
            if os.path.getsize(self.path) > 0 or self.proc.poll() is not None:
                break
            time.sleep(0.01)

    def mark_begin(self):
        self.window[0] = time.monotonic()

    def mark_end(self):
        self.window[1] = time.monotonic()

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        t_lo = self.window[0] if self.window[0] is not None else -1e30
        t_hi = self.window[1] if self.window[1] is not None else 1e30
        try:
            lines = open(self.path).read().splitlines()
            os.unlink(self.path)
        except OSError:
            lines = []
        for ln in lines:
            try:
                if self.source.startswith("nvml"):
                    t, a, b, c = ln.split()
                    t, a, b, c = float(t), float(a), float(b), int(c)
                else:  # nvidia-smi: no monotonic stamp -- every sample of the run
                    _, a, b, c = [x.strip() for x in ln.split(",")]
                    t, a, b, c = 0.0, float(a), float(b), int(c, 16)
                    t_lo, t_hi = -1e30, 1e30
            except ValueError:
                continue
            if t_lo <= t <= t_hi:
                self.samples.append((t, a, b, c))
        if not self.samples:
            why = {"lines": len(lines), "window": [t_lo, t_hi], "poller_rc": self.proc.returncode if self.proc else None}
            try:
                why["first"] = lines[:2]
                why["err"] = open(self.err_path).read()[-300:]
            except (OSError, AttributeError):
                pass
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "samples": 0, "debug": why}
        sm = [s[1] for s in self.samples]
        reasons = sorted({name for _, _, _, m in self.samples for name, bit in self.REASONS if m & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[2] for s in self.samples),
                "sm_mhz_min": min(sm), "reasons": reasons, "samples": len(sm), "source": self.source,
                "window": "the headline timed region"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


N_STAGE = 60  # scans of the per-stage timing pass (>= 50 timed iterations)
# k_project; k_count_reduce, k_count_top, k_duplicate, 6 x k_onesweep (passes beyond the
# device-side pass count exit at once), k_ranges, k_tile_order; k_render_lidar
LAUNCHES_PER_SCAN = 1 + (3 + 6 + 2) + 1
B_BATCH = 512  # scans in the B-batch trajectory (poses 0.2 m apart, x in [-51, +51] m)


def shard_poses(n_total: int, world: int, rank: int):
    """Round-robin shard of the B-batch trajectory: scan i -> rank i mod world,
    scan i at pose i mod 512 (the trajectory repeats, so every rank count sees the same mix
    of poses however many scans a run takes)."""
    poses = synth.batch_poses(B_BATCH)
    return [poses[i % B_BATCH] for i in batch.shard_indices(n_total, world, rank)]


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------------------ oracle (CPU) leg
def oracle_scan_sample(scene, cfg, tiling, pose0, pose1, n_tiles_sample, rng):
    """One bounded sample of the workload on the CPU oracle: the full projection + culling +
    binning of every particle (needed to know any tile's list), compositing of the rays of
    `n_tiles_sample` random tiles.  Returns (seconds, rays rendered)."""
    from oracle import oracle as O
    t0 = time.perf_counter()
    proj = O.project_lidar(scene, cfg, pose0, pose1)
    count, rect = O.cull_lidar(proj["valid"], proj["box"], tiling, True)
    _, ids, ranges = O.bin_pairs(count, rect, proj["key"], tiling.n_tiles, tiling.n_theta)
    tiles = rng.choice(tiling.n_tiles, min(n_tiles_sample, tiling.n_tiles), replace=False)
    rays = np.concatenate([tiling.tile_rays[tiling.tile_ray_offsets[x]:tiling.tile_ray_offsets[x + 1]]
                           for x in tiles])
    od = O.lidar_rays(tiling, pose0, pose1)[rays]
    rec = O.records_from_projection(proj, scene)
    O.composite(rec, ids, ranges, tiling.ray_tile[rays], tiling.ray_az[rays], tiling.ray_el[rays], od, wrap=1,
                near=cfg.min_range, pi_f=tiling.pi_f, two_pi_f=tiling.two_pi_f)
    return time.perf_counter() - t0, len(rays)


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, timed on the host cores.  A step is a
    bounded, proportional sample of one config-B scan: a random 1/S of the particles is
    projected, culled and binned, and the rays of a random 1/S of the render tiles are
    composited over the scan's full tile lists (built outside the timed region for a few
    poses).  S = 1 (the whole scan) for short runs; S grows with --steps so that a run costs
    about 24 full scans of oracle work.  value = rays composited / timed seconds."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    cores = cpu_count()
    O.set_threads(cores)
    cfg = synth.lidar_config("B")
    scene = synth.scene_for("B")
    tiling = O.Tiling(cfg)
    n = scene["means"].shape[0]
    S = max(1, math.ceil((args.steps + args.warmup) / 24))
    poses = synth.batch_poses(max(args.steps + args.warmup, 1))
    rng = np.random.default_rng(0)
    full = {}  # per pose index: records, lists, rays of the full scan (untimed when S > 1)

    def full_scan(pi, p0, p1):
        if pi not in full:
            proj = O.project_lidar(scene, cfg, p0, p1)
            count, rect = O.cull_lidar(proj["valid"], proj["box"], tiling, True)
            _, ids, ranges = O.bin_pairs(count, rect, proj["key"], tiling.n_tiles, tiling.n_theta)
            full[pi] = (O.records_from_projection(proj, scene), ids, ranges, O.lidar_rays(tiling, p0, p1))
        return full[pi]

    def step(i):
        p0, p1 = poses[i]
        if S == 1:  # the whole scan, every stage timed
            t0 = time.perf_counter()
            rec, ids, ranges, od = full_scan(-1 - i, p0, p1)
            rays = np.arange(tiling.n_rays)
            full.pop(-1 - i)
        else:
            pi = i % 4
            rec, ids, ranges, od = full_scan(pi, *poses[pi])
            sub_idx = np.sort(rng.choice(n, n // S, replace=False))
            sub = {k: v[sub_idx] for k, v in scene.items()}
            tiles = rng.choice(tiling.n_tiles, max(1, tiling.n_tiles // S), replace=False)
            rays = np.concatenate([tiling.tile_rays[tiling.tile_ray_offsets[x]:tiling.tile_ray_offsets[x + 1]]
                                   for x in tiles])
            t0 = time.perf_counter()
            proj = O.project_lidar(sub, cfg, p0, p1)
            count, rect = O.cull_lidar(proj["valid"], proj["box"], tiling, True)
            O.bin_pairs(count, rect, proj["key"], tiling.n_tiles, tiling.n_theta)
        O.composite(rec, ids, ranges, tiling.ray_tile[rays], tiling.ray_az[rays], tiling.ray_el[rays], od[rays],
                    wrap=1, near=cfg.min_range, pi_f=tiling.pi_f, two_pi_f=tiling.two_pi_f)
        return time.perf_counter() - t0, len(rays)

    for i in range(args.warmup):
        step(i)
    secs, rays = 0.0, 0
    for i in range(args.steps):
        s, n_r = step(args.warmup + i)
        secs += s
        rays += n_r
    value = rays / secs
    sample = (f"1/{S} of a config-B scan per step: a random 1/{S} of the 2M particles projected, culled and binned, "
              f"the rays of a random 1/{S} of the 3600 tiles composited over the full lists, {args.steps} steps"
              if S > 1 else f"full config-B scan per step (2M particles projected, all {tiling.n_rays} rays "
                            f"composited), {args.steps} steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU leg
def roofline_entries(stage_ms, counters, peaks, clocks_mhz):
    """Roofline of every stage per launch.  Each stage reports (a) its binding bound under
    SURVEY §8(d) -- projection: max(bytes N 48 + N_vis (192 + 96) over HBM, the §8(d)
    instruction model over the FP32 issue peak) = issue-bound at K = 1; bin_sort: the
    duplication bytes 8N + 16 N_vis + 12P plus the radix passes P (8 + passes 24) + 8P over
    HBM; render: the counted lane-instructions over the issue peak -- and (b) a strict
    variant beside it (algorithmic bytes only: inputs read once, outputs written once)."""
    hbm = peaks["hbm_gbs"]
    n, n_vis, P, R, n_tiles = (counters[k] for k in ("n", "n_vis", "P", "R", "n_tiles"))
    alu_peak = 148 * 128 * peaks["sm_max_mhz"] * 1e6 / 1e12  # T lane-instr/s at max clock
    K = counters["K"]
    # strict algorithmic bytes: inputs the method must read + outputs it must write
    b_project = n * (12 + 16 + 12 + 4) + n * (4 + 16 + 4) + n_vis * (192 + 80)
    b_sort = n * (4 + 16 + 4) + 4 * P + 12 * n_tiles
    lane_instr = (C_BOX * counters["visited"] + C_RESP * counters["inbox"] + C_ACC * counters["contrib"] +
                  C_RAY * R)
    b_render = n_vis * 80 + P * 4 + R * (40 + 12)
    # SURVEY §8(d) model
    i_proj = n * (7 * (C_PROJ + K * (C_PROJ + C_POSE)) + C_UT + C_MISC) + n_vis * C_SH
    b_proj8 = n * 48 + n_vis * (192 + 96)
    b_sort8 = (8 * n + 16 * n_vis + 12 * P) + P * (8 + counters["passes"] * 24) + 8 * P
    out = {}
    t = stage_ms["project"] * 1e-3
    hb, ib = b_proj8 / (hbm * 1e9), i_proj / (alu_peak * 1e12)
    out["project"] = ({"bound": "alu", "achieved": i_proj / t / 1e12, "peak": alu_peak, "unit": "T lane-instr/s",
                       "frac": ib / t} if ib >= hb else
                      {"bound": "hbm", "achieved": b_proj8 / t / 1e9, "peak": hbm, "unit": "GB/s", "frac": hb / t})
    out["project"].update({"model_lane_instr": int(i_proj), "survey_8d_bytes": int(b_proj8),
                           "hbm_frac_survey_8d": hb / t, "strict_bytes": int(b_project),
                           "strict_hbm_frac": b_project / t / 1e9 / hbm, "ms": stage_ms["project"]})
    t = stage_ms["bin_sort"] * 1e-3
    out["bin_sort"] = {"bound": "hbm", "achieved": b_sort8 / t / 1e9, "peak": hbm, "unit": "GB/s",
                       "frac": b_sort8 / t / 1e9 / hbm, "survey_8d_bytes": int(b_sort8), "strict_bytes": int(b_sort),
                       "strict_hbm_frac": b_sort / t / 1e9 / hbm, "ms": stage_ms["bin_sort"]}
    t = stage_ms["render"] * 1e-3
    ach = lane_instr / t / 1e12
    out["render"] = {"bound": "alu", "achieved": ach, "peak": alu_peak, "unit": "T lane-instr/s",
                     "frac": ach / alu_peak, "algorithmic_lane_instr": int(lane_instr),
                     "algorithmic_bytes": int(b_render), "hbm_frac": b_render / t / 1e9 / hbm,
                     "ms": stage_ms["render"]}
    t_roof = (b_project / (hbm * 1e9) + b_sort / (hbm * 1e9) +
              max(b_render / (hbm * 1e9), lane_instr / (alu_peak * 1e12)))
    parts = {"project": max(hb, ib), "duplicate": (8 * n + 16 * n_vis + 12 * P) / (hbm * 1e9),
             "sort": (P * (8 + counters["passes"] * 24) + 8 * P) / (hbm * 1e9),
             "render": max(b_render / (hbm * 1e9), lane_instr / (alu_peak * 1e12))}
    out["_scan"] = {"t_roof_ms": t_roof * 1e3, "t_roof_ms_survey_8d": sum(parts.values()) * 1e3,
                    "survey_8d_parts_ms": {k: v * 1e3 for k, v in parts.items()},
                    "survey_8d_inputs": {"projection_lane_instr": int(i_proj), "key_bits": counters["key_bits"],
                                         "passes": counters["passes"]}}
    return out


def pct(v, q):
    return float(np.percentile(np.asarray(v, np.float64), q))


def workload_counters(r, cfg):
    """SURVEY §8(d) workload counters of one config-B scan (outside every timed region):
    the Gaussian funnel, tile expansion, tile-list lengths, per-ray work and the
    warp-granularity ratio.  Needs r.want_counters(True) and write_all_records for N_valid."""
    import torch
    rec_box = r.record[:, 16]
    cnt = r.tile_count
    n = r.n
    n_valid = int(torch.isfinite(rec_box).sum().item())
    n_vis = int((cnt > 0).sum().item())
    P = int(r.n_pairs.item())
    rg = r.tile_ranges.cpu().numpy().astype(np.int64)
    L = rg[:, 1] - rg[:, 0]
    kb = r.depth_key[cnt > 0].view(torch.int32)
    kspan = int(kb.max().item()) - int(kb.min().item()) if n_vis else 0
    b = kspan.bit_length()
    tbits = max(1, (r.n_tiles - 1).bit_length())
    th = r.tiling_host
    ray_tile = th["ray_tile"].reshape(-1)
    nv = r.out["n_visited"].cpu().numpy().astype(np.int64)
    ni = r.out["n_inbox"].cpu().numpy().astype(np.int64)
    nc = r.out["n_contrib"].cpu().numpy().astype(np.int64)
    list_len = L[ray_tile]
    term = nv < list_len
    # warp granularity: a warp-per-tile kernel issues max over the tile's rays of the
    # entries scanned, for every ray of the tile
    off = th["tile_ray_offsets"].reshape(-1)
    rays = th["tile_rays"].reshape(-1)
    per_tile_max = np.maximum.reduceat(nv[rays], off[:-1]) if len(rays) else np.zeros(0)
    rays_in_tile = np.diff(off)
    nonempty = rays_in_tile > 0
    warp_gran = int((per_tile_max[nonempty] * rays_in_tile[nonempty]).sum())
    return {"n": n, "n_valid": n_valid, "n_culled": n_valid - n_vis, "n_vis": n_vis, "P": P,
            "tiles_per_visible_mean": P / max(n_vis, 1), "tiles_per_visible_max": int(cnt.max().item()),
            "list_len_mean": float(L.mean()), "list_len_p99": pct(L, 99), "list_len_max": int(L.max()),
            "R": r.n_rays, "n_tiles": r.n_tiles,
            "visited": int(nv.sum()), "inbox": int(ni.sum()), "contrib": int(nc.sum()),
            "visited_per_ray_mean": float(nv.mean()), "inbox_per_ray_mean": float(ni.mean()),
            "contrib_per_ray_mean": float(nc.mean()),
            "rays_terminated": int(term.sum()), "rays_exhausted": int((~term).sum()),
            "warp_granularity_entries": warp_gran, "warp_granularity_ratio": warp_gran / max(int(nv.sum()), 1),
            "key_bits": b + tbits, "depth_key_bits": b, "tile_bits": tbits, "passes": max(1, -(-(b + tbits) // 8)),
            "K": int(cfg.rs_iterations),
            "note": "terminated = the ray stopped before the end of its tile's list (T' < T_min, A14); a ray "
                    "terminated by its list's last entry counts as exhausted"}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2510_12901_b200 import simuli as SM

    ws, rank, local = dist_env()
    comm = None
    if ws > 1:
        # NCCL communicator init logged (stderr) so the rank count is verifiable
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
        comm = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    # clock poller started now, seconds before the timed region (its window is marked there)
    clocks = ClockSampler(dev.index if ws == 1 else local)
    clocks.start()
    SM.load()
    cfg = synth.lidar_config("B")
    scene_np = synth.scene_for("B")  # same seed on every rank: replicated scene
    scene = SM.to_device_scene(scene_np, dev)
    # S scans in flight: S renderers (own buffers, shared resident scene), S streams; scan i
    # runs on stream i mod S, so one scan's latency-bound stages overlap another's
    S = max(1, args.inflight)
    rs = [SM.LidarRenderer(cfg, scene, device=dev) for _ in range(S)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(S)]
    r = rs[0]
    for x in rs:
        x.keep_keys = False  # the renderer reads only the sorted ids
    n_total = (args.steps + args.warmup) * ws
    my = shard_poses(n_total, ws, rank)
    # size the pair buffers once (one sync) from a few poses of the shard, with head room;
    # every timed scan's pair count is tracked on the device (sticky max) and checked after
    # each timed region (a scan over capacity would have rendered truncated lists)
    need = 0
    for p0, p1 in my[:: max(1, len(my) // 4)]:
        r.scan(p0, p1, sync_capacity=True)
        torch.cuda.synchronize()
        need = max(need, int(r.n_pairs.item()))
    for x in rs:
        x.set_capacity(int(need * 1.3) + 4096)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def check_capacity(where):
        mx = max(x.check_capacity() for x in rs)  # raises on overflow
        return {"where": where, "max_pairs": mx, "capacity": min(x.capacity for x in rs)}

    for i in range(args.warmup):
        rs[i % S].scan(*my[i], stream=streams[i % S])
    torch.cuda.synchronize()
    # workload counters of one scan (outside the timed regions)
    r.want_counters(True)
    r.params.write_all_records = 1
    r.scan(*my[args.warmup])
    torch.cuda.synchronize()
    counters = workload_counters(r, cfg)
    r.params.write_all_records = 0
    r.want_counters(False)
    cap_checks = [check_capacity("warm-up + counters")]

    # ---- timed region (headline): K scans, S in flight; device time between two events on
    # the launching (main) stream, the S scan streams forked from / joined into it; no L2
    # flush needed: the resident scene (472 MB) and records (160 MB) exceed the 126 MB L2
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_begin()
    wall0 = time.perf_counter()
    e_beg, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_beg.record(stream)
    for st in streams:
        st.wait_event(e_beg)
    torch.cuda.nvtx.range_push(f"headline: {args.steps} scans, {S} in flight")
    for i in range(args.steps):
        rs[i % S].scan(*my[args.warmup + i], stream=streams[i % S])
    torch.cuda.nvtx.range_pop()
    for st in streams:
        ej = torch.cuda.Event()
        ej.record(st)
        stream.wait_event(ej)
    e_end.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clocks.mark_end()
    total_ms = e_beg.elapsed_time(e_end)
    max_ms = batch.reduce_max(total_ms, dev)  # slowest rank (device time)
    cap_checks.append(check_capacity("headline timed region"))

    # ---- stage breakdown (roofline evidence): N_STAGE scans one at a time on the main
    # stream, L2 flushed (256 MB write) before every scan outside the events, per-stage
    # CUDA events; median / p10 / p90 (SURVEY §8(d) timing protocol)
    n_stage = N_STAGE
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_stage)]
    nvtx = torch.cuda.nvtx
    for i in range(n_stage):
        flush.zero_()
        p0, p1 = my[(args.warmup + i) % len(my)]
        r.set_poses(p0, p1)
        e = ev[i]
        e[0].record(stream)
        nvtx.range_push("project")
        r.project()
        nvtx.range_pop()
        e[1].record(stream)
        nvtx.range_push("bin_sort")
        r.bin_sort()
        nvtx.range_pop()
        e[2].record(stream)
        nvtx.range_push("render")
        r.render()
        nvtx.range_pop()
        e[3].record(stream)
    torch.cuda.synchronize()
    # per-stage throughput: each stage alone, N_STAGE launches spread over the S renderers /
    # streams (lists and records from their last scan), device time / launches -- the cost of
    # one launch when S run concurrently, as in the headline
    stage_tp = {}
    for name in ("project", "bin_sort", "render"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for st in streams:
            st.wait_event(e0)
        for i in range(n_stage):
            getattr(rs[i % S], name)(stream=streams[i % S])
        for st in streams:
            ej = torch.cuda.Event()
            ej.record(st)
            stream.wait_event(ej)
        e1.record(stream)
        torch.cuda.synchronize()
        stage_tp[name] = e0.elapsed_time(e1) / n_stage
    # latency mode: the same stage pass with the latency-optimised render shape
    # (simuli_render_params.lidar_producers = 3); outputs identical, reported beside
    r.rparams.lidar_producers = 3
    lat = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(n_stage)]
    lat_scan = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(n_stage)]
    for i in range(n_stage):
        flush.zero_()
        p0, p1 = my[(args.warmup + i) % len(my)]
        r.set_poses(p0, p1)
        lat_scan[i][0].record(stream)
        r.project()
        r.bin_sort()
        lat[i][0].record(stream)
        r.render()
        lat[i][1].record(stream)
        lat_scan[i][1].record(stream)
    torch.cuda.synchronize()
    r.rparams.lidar_producers = 0
    latency_mode = {"render_producers": 3,
                    "render_ms_median": statistics.median(e[0].elapsed_time(e[1]) for e in lat),
                    "scan_ms_median": statistics.median(e[0].elapsed_time(e[1]) for e in lat_scan),
                    "note": "one scan at a time, L2 flushed, the latency-optimised render pipeline (3 producer "
                            "warps + 1 consumer warp per item); the headline uses the default hybrid (the longest "
                            "items by that pipeline, the rest one warp per item)"}
    clk = clocks.stop()
    cap_checks.append(check_capacity("stage pass"))
    samples = {"project": [e[0].elapsed_time(e[1]) for e in ev], "bin_sort": [e[1].elapsed_time(e[2]) for e in ev],
               "render": [e[2].elapsed_time(e[3]) for e in ev], "scan": [e[0].elapsed_time(e[3]) for e in ev]}
    dist_ms = {k: {"median": statistics.median(v), "p10": pct(v, 10), "p90": pct(v, 90), "mean": statistics.fmean(v)}
               for k, v in samples.items()}
    stage_ms = {k: dist_ms[k]["median"] for k in ("project", "bin_sort", "render")}
    latency_ms = batch.reduce_max(dist_ms["scan"]["median"], dev)
    job_counters = batch.reduce_sum({"pairs": counters["P"], "scans": args.steps}, dev)

    # ---- e2e through the public API with host buffers: every scan takes its pose pair in
    # (kernel parameters) and copies every per-ray output to pinned host memory on its own
    # stream, S scans in flight as in the headline (scan i+1 computes while scan i's outputs
    # travel); timed on the host wall clock from the first launch to the last host byte
    # (launch overhead included), max over ranks.
    hosts = [{k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in x.out.items() if v is not None}
             for x in rs]
    d2h = sum(v.numel() * v.element_size() for v in hosts[0].values())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.steps):
        p0, p1 = my[args.warmup + i]
        x, st, host = rs[i % S], streams[i % S], hosts[i % S]
        x.scan(p0, p1, stream=st)
        with torch.cuda.stream(st):
            for k, v in host.items():
                v.copy_(x.out[k], non_blocking=True)
    for st in streams:
        st.synchronize()
    tt = time.perf_counter() - t0
    e2e_s = batch.reduce_max(tt, dev)
    cap_checks.append(check_capacity("e2e timed region"))
    e2e = {"value": ws * args.steps * r.n_rays / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": 2 * 28, "d2h_bytes_per_step": int(d2h),
           "note": f"per scan: start/end pose (2 x 28 B) in as kernel parameters, all per-ray outputs "
                   f"(zeta, omega, D, depth, gamma, beta, T, n) copied to pinned host memory on the scan's "
                   f"stream; {S} scans in flight; host wall clock from first launch to last byte; "
                   f"scene resident in HBM"}

    # ---- B-batch spot check: every 64th scan of the batch (the ones this
    # rank rendered in the timed region) re-rendered, gathered to rank 0 (NCCL all_gather
    # for N > 1) and compared bit for bit with rank 0 rendering the same poses itself (G=1)
    spot = [i for i in range(args.warmup, n_total, 64)]
    mine_idx = set(batch.shard_indices(n_total, ws, rank))
    local = {}
    for j, i in enumerate(spot):
        if i in mine_idx:
            k = batch.shard_indices(n_total, ws, rank).index(i)
            out = r.scan(*my[k])
            local[j] = torch.stack([out["depth"], out["intensity"], out["raydrop"], out["opacity"]]).clone()
    torch.cuda.synchronize()
    g0 = time.perf_counter()
    like = torch.empty((4, r.n_rays), dtype=torch.float32, device=dev)
    full = batch.gather_frames(local, len(spot), dev, owner=lambda j: spot[j] % ws, like=like)
    gather_ms = 1e3 * (time.perf_counter() - g0)
    identical = None
    if rank == 0:
        all_poses = shard_poses(n_total, 1, 0)
        identical = True
        for j, i in enumerate(spot):
            out = r.scan(*all_poses[i])
            ref = torch.stack([out["depth"], out["intensity"], out["raydrop"], out["opacity"]])
            identical &= bool(torch.equal(full[j].to(dev), ref))
    spot_check = {"scans": len(spot), "gather_ms": gather_ms, "gather_identical": identical,
                  "note": "every 64th B-batch scan, rendered by its owner rank, gathered to rank 0 and compared "
                          "bit for bit with rank 0's own render of the same pose (depth, intensity, ray drop, "
                          "opacity)"}

    peaks = read_peaks()
    roof = roofline_entries(stage_ms, counters, peaks, clk.get("sm_mhz"))
    roof_tp = roofline_entries(stage_tp, counters, peaks, clk.get("sm_mhz"))
    roof_tp.pop("_scan")
    stages_inflight = {k: {"ms_per_launch": stage_tp[k], "bound": v["bound"], "achieved": v["achieved"],
                           "peak": v["peak"], "unit": v["unit"], "frac": v["frac"]} for k, v in roof_tp.items()}
    stages_inflight["note"] = (f"each stage alone, {n_stage} launches over {S} streams (S in flight, as the headline): "
                               "device time per launch and the stage's roofline fraction at that throughput")
    dom_tp = max(roof_tp, key=lambda k: roof_tp[k]["ms"])
    roofline_inflight = {k: stages_inflight[dom_tp][k] for k in ("bound", "achieved", "peak", "unit", "frac")}
    roofline_inflight.update({"kernel": dom_tp, "ms_per_launch": stage_tp[dom_tp],
                              "note": "the stage with the largest per-launch cost in flight (S concurrent launches, "
                                      "the headline's regime); `roofline` is the same for launches one at a time"})
    scan_roof = roof.pop("_scan")
    thr = max_ms / args.steps
    scan_roof.update({"latency_ms": latency_ms, "frac_of_latency": scan_roof["t_roof_ms"] / latency_ms,
                      "throughput_ms_per_scan": thr, "frac_of_throughput": scan_roof["t_roof_ms"] / thr,
                      "frac_of_throughput_survey_8d": scan_roof["t_roof_ms_survey_8d"] / thr,
                      "frac_of_latency_survey_8d": scan_roof["t_roof_ms_survey_8d"] / latency_ms,
                      "note": "t_roof = sum_s max(B_s / HBM, I_s / issue peak). strict: the stages' algorithmic "
                              "bytes (project, sort: bytes only) and render lane-instructions; survey_8d: "
                              "SURVEY §8(d) as written (projection instruction model, duplication bytes, radix "
                              "passes counted)"})
    # the dominant kernel: the largest per-launch cost in the headline's regime (S scans in
    # flight, stages_inflight); its roofline from the one-at-a-time stage pass, whose
    # per-launch times are comparable with ncu's serialised launch list
    dom = max(stage_tp, key=lambda k: stage_tp[k])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(dom)
    d = roof[dom]
    roofline = {"bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"], "unit": d["unit"],
                "frac": d["frac"], "traffic": traffic, "kernel": dom, "peak_source": peaks["source"],
                "note": "the stage with the largest per-launch cost in flight (the headline's regime), measured one "
                        "launch at a time; its binding bound under SURVEY §8(d) (projection: its instruction model "
                        "over the FP32 issue peak 148 SM x 128 lanes x max clock; bytes in stages[...]); traffic = "
                        "ncu dram read + write bytes of that stage's launches in one scan (profiles/ncu_traffic.json); "
                        "every stage one at a time in `stages`, in flight in `stages_inflight`"}
    if rank != 0:
        dist.destroy_process_group()
        return 0
    value = ws * args.steps * r.n_rays / (max_ms * 1e-3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": thr, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_gaussians": r.n, "rays_per_scan": r.n_rays,
                       "scans_per_rank": args.steps, "scans_in_flight": S,
                       "l2": "timed pass: inputs larger than L2 (scene 472 MB + records 160 MB > 126 MB), no "
                             "flush; stage pass: L2 flushed before every scan (256 MB write)",
                       "parallelism": f"dp{ws}"},
            "scans_per_s": value / r.n_rays,
            "latency_ms_per_scan": latency_ms, "latency_mode": latency_mode,
            "e2e": e2e, "gpu_launches": LAUNCHES_PER_SCAN * args.steps,
            "roofline": roofline, "roofline_inflight": roofline_inflight, "stages": roof,
            "stages_inflight": stages_inflight,
            "stage_ms_distribution": dict(dist_ms, n=n_stage),
            "scan_roofline": scan_roof, "counters": counters, "job_counters": job_counters,
            "capacity_checks": cap_checks, "spot_check": spot_check, "comm": comm,
            "clocks": clk,
            "wall_s_timed_region": wall}
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(scene_np, cfg)
    if ws == 1 and not args.no_secondary:
        del r, rs
        torch.cuda.empty_cache()
        line["secondary"] = secondary_configs(dev)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def secondary_configs(dev, steps=20, warmup=3):
    """The other full-size BASELINE.json configs, device time per scan / frame with the L2
    flushed between scans (not the headline): C = Waymo-top-like LiDAR, 64 x 2650 rays,
    4M particles; D = KB fisheye rolling-shutter camera 1920 x 1080, 2M particles."""
    import torch

    from paper_2510_12901_b200 import simuli as SM
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    out = {}

    def timed(obj, n_units, unit):
        obj.keep_keys = False
        for _ in range(warmup):
            obj.project(); obj.bin_sort(sync_capacity=True); obj.render()
        torch.cuda.synchronize()
        st = {"project": [], "bin_sort": [], "render": []}
        for _ in range(steps):
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(); obj.project(); ev[1].record(); obj.bin_sort(); ev[2].record(); obj.render(); ev[3].record()
            torch.cuda.synchronize()
            for k, (a, b) in zip(st, ((0, 1), (1, 2), (2, 3))):
                st[k].append(ev[a].elapsed_time(ev[b]))
        ms = sum(statistics.median(v) for v in st.values())
        return {"value": n_units / (ms * 1e-3), "unit": unit, "ms_per_step": ms,
                "stages_ms": {k: statistics.median(v) for k, v in st.items()}, "pairs": int(obj.n_pairs.item()),
                "steps": steps}

    cfg = synth.lidar_config("C")
    r = SM.LidarRenderer(cfg, SM.to_device_scene(synth.scene_for("C"), dev), device=dev)
    out["C"] = dict(timed(r, r.n_rays, "rays/s"), workload="C: Waymo-top-like 64x2650 rays (non-uniform beams), "
                    "4M particles, rolling shutter (1.5 m, 0.02 rad)")
    del r
    torch.cuda.empty_cache()
    cam = synth.camera_config("D")
    c = SM.CameraRenderer(cam, SM.to_device_scene(synth.scene_for("D"), dev), device=dev)
    out["D"] = dict(timed(c, cam.width * cam.height, "pixels/s"), workload="D: KB fisheye 1920x1080, rolling "
                    "shutter (30 ms, 0.3 m, 0.009 rad), 2M camera particles, 16x16 px tiles")
    del c
    torch.cuda.empty_cache()
    return out


def cpu_baseline(scene_np, cfg):
    """The oracle as it stands on the host cores, one bounded sample of the workload."""
    from oracle import oracle as O
    cores = cpu_count()
    O.set_threads(cores)
    tiling = O.Tiling(cfg)
    rng = np.random.default_rng(1)
    secs, rays = oracle_scan_sample(scene_np, cfg, tiling, cfg.pose_start, cfg.pose_end, tiling.n_tiles, rng)
    out = {"value": rays / secs, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"one full config-B scan: all {scene_np['means'].shape[0]} particles projected/culled/binned "
                     f"and all {rays} rays composited in double precision; {secs:.2f} s wall"}
    if cores > 1 and secs * cores < 40.0:  # the oracle on one core too (same scan)
        O.set_threads(1)
        s1, r1 = oracle_scan_sample(scene_np, cfg, tiling, cfg.pose_start, cfg.pose_end, tiling.n_tiles, rng)
        O.set_threads(cores)
        out["one_core"] = {"value": r1 / s1, "unit": UNIT, "cores": 1, "wall_s": s1}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the configs C and D lines")
    ap.add_argument("--inflight", type=int, default=6, help="scans in flight (renderers / streams) per GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
