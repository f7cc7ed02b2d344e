"""Multi-GPU partitioning of the hot path: one process per GPU, independent
units, no collective on the data path.

A unit is a (batch, kv-head) pair carrying all G query heads of its group, so dK/dV
accumulation over the group stays on one GPU (mirrors the group loop, engine.cpp:330-331).
Units are split into contiguous, balanced ranges (the masks of the BASELINE configs are
(b,h)-broadcast, so every unit carries the same work)."""
from __future__ import annotations


def shard_units(num_units: int, rank: int, world: int) -> range:
    """Contiguous balanced range of units owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(num_units, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def unit_heads(batch: int, kv_heads: int, group: int, units: range):
    """Expand (b, kv-head) units into (b, q-head) pairs."""
    out = []
    for u in units:
        b, kh = divmod(u, kv_heads)
        if b >= batch:
            raise ValueError("unit out of range")
        out.extend((b, kh * group + g) for g in range(group))
    return out


def max_over_ranks(value: float, group=None) -> float:
    """Job time = the slowest rank (device-timed values, never wall clock)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
