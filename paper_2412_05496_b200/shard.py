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


def rect_split(batch: int, kv_heads: int, world: int):
    """Split a job's (batch, kv-head) unit grid into `world` equal rectangles: kv heads are split
    first (a rank keeps every batch element, so its inputs stay (B', H', L, D) tensors and the
    ALiBi slopes of its heads are a contiguous slice), then batches. Returns (wb, wh)."""
    from math import gcd
    wh = gcd(world, kv_heads)
    wb = world // wh
    if batch % wb != 0:
        raise ValueError(f"cannot split {batch}x{kv_heads} (batch x kv-head) units into {world} rectangles")
    return wb, wh


def rect_shard(batch: int, kv_heads: int, world: int, rank: int):
    """(b0, b1, kh0, kh1) of `rank`'s rectangle of (batch, kv-head) units."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    wb, wh = rect_split(batch, kv_heads, world)
    rb, rh = divmod(rank, wh)
    nb, nh = batch // wb, kv_heads // wh
    return rb * nb, (rb + 1) * nb, rh * nh, (rh + 1) * nh


def slice_job(q, k, v, do, group: int, shard):
    """This rank's contiguous inputs: q/dO heads [kh0*G, kh1*G), k/v heads [kh0, kh1), batches
    [b0, b1) (a kv batch of 1 is shared by every query batch element)."""
    b0, b1, kh0, kh1 = shard
    kb = slice(None) if k.shape[0] == 1 else slice(b0, b1)
    qs = q[b0:b1, kh0 * group:kh1 * group].contiguous()
    dos = do[b0:b1, kh0 * group:kh1 * group].contiguous() if do is not None else None
    return qs, k[kb, kh0:kh1].contiguous(), v[kb, kh0:kh1].contiguous(), dos


def shard_score(score, group: int, shard):
    """The score_mod of a shard: ALiBi slopes are indexed by q head, so a rank keeps its slice."""
    from dataclasses import replace
    if score.slopes is None:
        return score
    _, _, kh0, kh1 = shard
    return replace(score, slopes=list(score.slopes)[kh0 * group:kh1 * group])
