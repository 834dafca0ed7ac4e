"""Multi-rank host logic on CPU (gloo, world sizes 2 and 3 with uneven shards; -m "not gpu").

The GPU path shards independent scans round-robin with no data-path collective
(SURVEY §8(e)); here each rank renders its shard of tiny scans with the CPU oracle as the
stand-in per-frame renderer, and the gathered batch must be bit-identical to a single-rank
run; timers reduce by MAX, counters by SUM.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_12901_b200 import batch, synth

N_SCANS = 7


def _render(i):
    from oracle import oracle as O
    cfg = synth.lidar_config("tiny")
    scene = synth.scene_for("tiny", seed=3)
    poses = synth.batch_poses(N_SCANS, x_lo=-1.0, step=0.3, motion=0.2)
    out = O.render_lidar(scene, cfg, pose0=poses[i][0], pose1=poses[i][1])
    return torch.from_numpy(np.stack([out["opacity"], out["depth"], out["T_final"]], 1))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = batch.shard_indices(N_SCANS, world, rank)
        local = {i: _render(i) for i in mine}
        full = batch.gather_frames(local, N_SCANS)
        tmax = batch.reduce_max(10.0 + rank)
        csum = batch.reduce_sum({"scans": len(mine), "rank1": rank})
        # bench.py's spot-check gather: frame j owned by rank spot[j] mod world, ranks that
        # own none contribute an empty (zero-padded) buffer shaped like `like`
        spot = [1, 5]
        own = lambda j: spot[j] % world  # noqa: E731
        sl = {j: torch.full((3,), float(spot[j]) + 0.5) for j in range(len(spot)) if own(j) == rank}
        sfull = batch.gather_frames(sl, len(spot), owner=own, like=torch.empty(3))
        if rank == 0:
            q.put(({i: v.numpy() for i, v in full.items()}, tmax, csum, {j: v.numpy() for j, v in sfull.items()}))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_indices_partition():
    for world in (1, 2, 3, 8):
        seen = sorted(i for r in range(world) for i in batch.shard_indices(37, world, r))
        assert seen == list(range(37))
    with pytest.raises(ValueError):
        batch.shard_indices(4, 2, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_gather_equals_single_rank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, tmax, csum, sfull = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 10.0 + world - 1
    assert csum == {"scans": N_SCANS, "rank1": sum(range(world))}
    assert sorted(sfull) == [0, 1] and sfull[0].tolist() == [1.5] * 3 and sfull[1].tolist() == [5.5] * 3
    assert sorted(full) == list(range(N_SCANS))
    for i in range(N_SCANS):
        assert np.array_equal(full[i], _render(i).numpy())
