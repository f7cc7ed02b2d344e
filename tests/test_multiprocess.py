"""CPU, world_size 2 over gloo: the N>1 host path. Each rank computes its shard of a small
attention problem with the oracle (the GPU kernel is not needed to test the partitioning),
shards are disjoint and cover the job, the gathered result equals the single-process result
bit for bit, and the job time is the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import torch
    import torch.distributed as dist

    import pyoracle as O
    from paper_2412_05496_b200.shard import max_over_ranks, shard_units, unit_heads

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, Hq, Hkv, L, D = 2, 4, 2, 48, 8
    G = Hq // Hkv
    q = O.random_f32(1, (B, Hq, L, D))
    k = O.random_f32(2, (B, Hkv, L, D))
    v = O.random_f32(3, (B, Hkv, L, D))
    m = O.causal()
    bm = O.create_block_mask(m, 1, 1, L, L, 16, 16)
    units = shard_units(B * Hkv, rank, world)
    pairs = unit_heads(B, Hkv, G, units)
    local = np.zeros((B, Hq, L, D), np.float32)
    for b, kh in sorted({(b, h // G) for b, h in pairs}):
        o, _ = O.forward(q[b:b + 1, kh * G:(kh + 1) * G], k[b:b + 1, kh:kh + 1], v[b:b + 1, kh:kh + 1],
                         m, O.Score(), bm, gqa=G)
        local[b, kh * G:(kh + 1) * G] = o[0]
    t = torch.from_numpy(local)
    dist.all_reduce(t)  # shards are disjoint: the sum assembles the job's output
    slowest = max_over_ranks(0.5 + rank)
    if rank == 0:
        full, _ = O.forward(q, k, v, m, O.Score(), bm, gqa=G)
        out_q.put((np.array_equal(t.numpy(), full), slowest, [list(shard_units(B * Hkv, r, world)) for r in range(world)]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    equal, slowest, shards = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert equal
    assert slowest == 1.5
    assert shards == [[0, 1], [2, 3]]


def test_shard_units_balanced():
    from paper_2412_05496_b200.shard import shard_units
    for n in (1, 4, 16, 64, 2048, 7):
        for w in (1, 2, 4, 8):
            rs = [shard_units(n, r, w) for r in range(w)]
            assert sum(len(r) for r in rs) == n
            assert [x for r in rs for x in r] == list(range(n))
            assert max(len(r) for r in rs) - min(len(r) for r in rs) <= 1
