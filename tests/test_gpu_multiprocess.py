"""GPU, world_size 2: one job partitioned into (batch, kv-head) rectangles (shard.rect_shard), each
rank running fa.forward / fa.backward on its shard with no collective on the data path; the
shards are gathered over gloo and must equal the single-process run bit for bit (forward
outputs, lse, and gradients in the deterministic backward mode). Both ranks share cuda:0 (the
test box has one GPU); the partitioning logic is the one bench.py --strong uses on N GPUs."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _job(fa, dev, name):
    import numpy as np
    if name == "c2":
        B, Hq, Hkv, L, D = 2, 4, 4, 2048, 128
        mask, score = fa.sliding_window(300), fa.alibi(fa.alibi_slopes(Hq))
    else:
        B, Hq, Hkv, L, D = 2, 8, 2, 1536, 128
        mask, score = fa.causal(), fa.soft_cap(50.0)
    _ = np
    q, do = (fa.random_tensor(s, (B, Hq, L, D), device=dev) for s in (1, 4))
    k, v = (fa.random_tensor(s, (B, Hkv, L, D), device=dev) for s in (2, 3))
    return (B, Hq, Hkv, L, D), mask, score, (q, k, v, do)


def _run(fa, geo, mask, score, tensors, dev):
    B, Hq, Hkv, L, D = geo
    q, k, v, do = tensors
    cfg = fa.AttentionConfig(gqa_group=q.shape[1] // k.shape[1])
    bm = fa.create_block_mask(mask, 1, 1, L, L, device=dev)
    res = fa.forward(q, k, v, score, bm, cfg)
    g = fa.backward(q, k, v, res, do, score, bm, cfg=cfg, deterministic=True)
    return [t.cpu() for t in (res.out, res.lse, g.dq, g.dk, g.dv)]


def _worker(rank, world, port, name, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2412_05496_b200 as fa
    from paper_2412_05496_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    geo, mask, score, full = _job(fa, dev, name)
    B, Hq, Hkv, L, D = geo
    G = Hq // Hkv
    sh = shard.rect_shard(B, Hkv, world, rank)
    part = shard.slice_job(*full, G, sh)
    mine = _run(fa, (sh[1] - sh[0], (sh[3] - sh[2]) * G, sh[3] - sh[2], L, D), mask,
                shard.shard_score(score, G, sh), part, dev)
    gathered = [None] * world
    dist.all_gather_object(gathered, (sh, mine))  # off the data path: result check only
    if rank == 0:
        ref = _run(fa, geo, mask, score, full, dev)
        ok = True
        for (b0, b1, kh0, kh1), outs in gathered:
            qh, kh = slice(kh0 * G, kh1 * G), slice(kh0, kh1)
            for got, want, hs in zip(outs, ref, (qh, qh, qh, kh, kh)):
                ok = ok and torch.equal(got, want[b0:b1, hs])
        out_q.put((ok, [g[0] for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2", "gqa"])
def test_two_rank_gpu_shards_bitwise(name, dev):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, shards = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert ok, shards
    assert all(p.exitcode == 0 for p in procs)
