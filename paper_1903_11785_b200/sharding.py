"""Frame sharding across GPUs.

Frames are independent (pipeline.py:115-220 keeps no cross-frame state), so
N processes (one per GPU, torchrun) split a sequence by frame index with no
collective on the data path. The helpers here are the whole multi-GPU layer:
frame assignment, the max-over-ranks timer reduction the benchmark uses,
and the optional gather of finished per-frame results to rank 0 (for the
bundle writer; outside the timed hot path).
"""

from __future__ import annotations

import os


def world():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def frames_for_rank(rank: int, world_size: int, n_frames: int) -> list:
    """Round-robin: frame f -> rank f mod N (balanced to within one frame)."""
    if not (0 <= rank < world_size):
        raise ValueError(f"rank {rank} outside world of {world_size}")
    return list(range(rank, n_frames, world_size))


def reduce_max(value: float, group=None) -> float:
    """Max over ranks (device timers: the slowest rank defines the job time)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def reduce_sum(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def gather_to_rank0(items: dict, group=None):
    """Gather {frame_id: payload} dicts (e.g. mesh arrays + visibility bits)
    from every rank to rank 0; returns the merged dict on rank 0, None
    elsewhere. Host objects, so it works over gloo and nccl alike."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return dict(items)
    out = [None] * dist.get_world_size(group) if dist.get_rank(group) == 0 else None
    dist.gather_object(items, out, dst=0, group=group)
    if out is None:
        return None
    merged = {}
    for part in out:
        merged.update(part)
    return dict(sorted(merged.items()))
