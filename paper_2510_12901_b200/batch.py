"""Data-parallel batches of independent sensor frames.

The forward path has no exchange step inside a scan or frame, so multi-GPU work is a
round-robin shard of independent frames per rank (one process per GPU, scene replicated)
with no collective on the data path.  Collectives (torch.distributed: NCCL on GPUs, gloo
in the CPU tests) are used only to reduce timers / counters and, optionally, to gather
outputs to rank 0.
"""
from __future__ import annotations


def shard_indices(n_total: int, world: int, rank: int) -> list[int]:
    """Frames of rank `rank`: i with i mod world == rank (round robin)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world / rank")
    return list(range(rank, n_total, world))


def reduce_max(value: float, device="cpu") -> float:
    """Max over ranks (device time of the slowest rank); identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(values: dict, device="cpu") -> dict:
    """Sum of integer counters over ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return dict(values)
    keys = sorted(values)
    t = torch.tensor([int(values[k]) for k in keys], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return {k: int(v) for k, v in zip(keys, t.tolist())}


def gather_frames(local: dict, n_total: int, device="cpu", owner=None, like=None):
    """Gather {frame index: tensor} from every rank onto rank 0 (fixed-size all_gather of
    a stacked buffer; frames of one batch have equal shapes).  owner(i) = the rank holding
    frame i (default: round robin, i mod world); like = a tensor of the frame shape / dtype
    (needed when a rank holds no frame).  Returns the full {index: tensor} dict on rank 0,
    None elsewhere."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return dict(local)
    world, rank = dist.get_world_size(), dist.get_rank()
    own = owner if owner is not None else (lambda i: i % world)
    frames_of = [[i for i in range(n_total) if own(i) == r] for r in range(world)]
    per = max(1, max(len(f) for f in frames_of))
    sample = like if like is not None else next(iter(local.values()))
    buf = torch.zeros((per,) + tuple(sample.shape), dtype=sample.dtype, device=device)
    for k, i in enumerate(frames_of[rank]):
        buf[k] = local[i].to(device)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    if rank != 0:
        return None
    full = {}
    for r in range(world):
        for k, i in enumerate(frames_of[r]):
            full[i] = out[r][k]
    return full
