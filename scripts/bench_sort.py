"""Micro-benchmark of simuli_bin_sort on synthetic tile lists (device time per call)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_12901_b200 import simuli as SM

def run(name, n_tiles, ncols, tiles_of, keys, reps=20):
    n = len(tiles_of)
    dev = "cuda"
    rows = n_tiles // ncols
    rect = np.stack([tiles_of // ncols, tiles_of // ncols, tiles_of % ncols, np.ones(n, np.int64)], 1).astype(np.int32)
    count = np.ones(n, np.int32)
    t = {k: torch.from_numpy(v).to(dev) for k, v in (("count", count), ("rect", rect), ("key", keys.astype(np.float32)))}
    proj = SM.Projected(0, t["rect"].data_ptr(), t["key"].data_ptr(), t["count"].data_ptr())
    cap = n + 16
    ws = torch.empty(SM.simuli_bin_sort_workspace_size(n, cap, n_tiles), dtype=torch.uint8, device=dev)
    ids = torch.empty(cap, dtype=torch.int32, device=dev)
    ranges = torch.empty((n_tiles, 2), dtype=torch.int32, device=dev)
    npairs = torch.zeros(1, dtype=torch.int64, device=dev)
    torder = torch.empty(n_tiles, dtype=torch.int32, device=dev)
    for _ in range(3):
        SM.simuli_bin_sort(proj, n, n_tiles, ncols, ws, cap, None, ids, ranges, npairs, tile_order=torder)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        SM.simuli_bin_sort(proj, n, n_tiles, ncols, ws, cap, None, ids, ranges, npairs, tile_order=torder)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:40s} n={n:9d} tiles={n_tiles:5d}: {e0.elapsed_time(e1) / reps * 1e3:8.1f} us", flush=True)

rng = np.random.default_rng(0)
only = sys.argv[1] if len(sys.argv) > 1 else None
for size in (256, 1024, 4096, 16384, 18000):
    if only and only != f"u{size}":
        continue
    n_tiles = max(1, 3_000_000 // size)
    n_tiles = min(n_tiles, 16384)
    ncols = 16 if n_tiles >= 16 else 1
    n_tiles = (n_tiles // ncols) * ncols
    tiles = np.repeat(np.arange(n_tiles), size)
    rng.shuffle(tiles)
    run(f"uniform lists of {size}", n_tiles, ncols, tiles, rng.uniform(3, 140, len(tiles)))
for size in (1024, 4096, 8192, 16384, 18000, 40000):
    if only and only != f"o{size}":
        continue
    tiles = np.zeros(size, np.int64)
    run(f"one list of {size}", 16, 16, tiles, rng.uniform(3, 140, size))
