"""GPU: the forward, backward and decode calls are stream-ordered with no host synchronisation
on the default path, so a whole training / serving step can be captured in a CUDA graph and
replayed (the B200 replacement of a tracing compiler): replays equal eager execution bit for bit
(the fused backward's dQ adds are order-dependent, so the graph replays the deterministic mode
and compares dK/dV of the default mode)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_fwd_bwd_step_in_a_cuda_graph(fa, dev):
    B, H, L, D = 1, 4, 1024, 128
    q = fa.random_tensor(1, (B, H, L, D), device=dev)
    k = fa.random_tensor(2, (B, H, L, D), device=dev)
    v = fa.random_tensor(3, (B, H, L, D), device=dev)
    do = fa.random_tensor(4, (B, H, L, D), device=dev)
    score = fa.alibi(fa.alibi_slopes(H))
    bm = fa.create_block_mask(fa.sliding_window(300), 1, 1, L, L, device=dev)
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm up on the capturing stream (per-stream scratch words)
        for _ in range(2):
            res = fa.forward(q, k, v, score, bm)
            g = fa.backward(q, k, v, res, do, score, bm, deterministic=True)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        res_g = fa.forward(q, k, v, score, bm)
        g_g = fa.backward(q, k, v, res_g, do, score, bm, deterministic=True)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    res_e = fa.forward(q, k, v, score, bm)
    g_e = fa.backward(q, k, v, res_e, do, score, bm, deterministic=True)
    torch.cuda.synchronize()
    assert torch.equal(res_g.out, res_e.out) and torch.equal(res_g.lse, res_e.lse)
    for a, b in ((g_g.dq, g_e.dq), (g_g.dk, g_e.dk), (g_g.dv, g_e.dv)):
        assert torch.equal(a, b)


def test_decode_step_in_a_cuda_graph(fa, dev):
    B, Hq, Hkv, L, D, ps = 4, 8, 2, 700, 128, 128
    cache = fa.PagedKVCache(B, B * 6 + B, ps, Hkv, D, device=dev)
    kl = fa.random_tensor(11, (B, Hkv, L, D), device=dev)
    for b in range(B):
        cache.assign(b, kl[b:b + 1], kl[b:b + 1])
    q = fa.random_tensor(12, (B, Hq, 2, D), device=dev)
    off = L - 2
    pt = cache.page_table()
    pbm = fa.convert_block_mask(fa.create_block_mask(fa.offset_mask(fa.causal(), off), 1, 1, 2, L, device=dev), pt)
    cfg = fa.AttentionConfig(gqa_group=Hq // Hkv)

    def step():
        return fa.decode(q, cache.k_phys(), cache.v_phys(), off, fa.causal(), fa.noop_score(), pbm, cfg=cfg,
                         page_table=pt)
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        out_g = step()
    graph.replay()
    torch.cuda.synchronize()
    out_e = step()
    torch.cuda.synchronize()
    assert torch.equal(out_g.out, out_e.out) and torch.equal(out_g.lse, out_e.lse)


def test_serving_step_append_convert_decode_in_a_cuda_graph(fa, dev):
    """A whole serving step — the device page pool's batched append of one token per sequence,
    the asynchronous convert_block_mask and the paged GQA decode — holds no host round trip, so
    it captures into a CUDA graph; the replayed step equals the same step run eagerly."""
    B, Hq, Hkv, L0, D, ps = 4, 8, 2, 383, 128, 128
    cache = fa.PagedKVCache(B, B * 4, ps, Hkv, D, device=dev)
    kl = fa.random_tensor(21, (B, Hkv, L0 + 1, D), device=dev)
    vl = fa.random_tensor(22, (B, Hkv, L0 + 1, D), device=dev)
    cache.assign_batch(list(range(B)), [L0] * B, torch.cat([kl[b:b + 1, :, :L0] for b in range(B)], 2),
                       torch.cat([vl[b:b + 1, :, :L0] for b in range(B)], 2))
    ids = torch.arange(B, dtype=torch.int32, device=dev)
    ones = torch.ones(B, dtype=torch.int32, device=dev)
    kn = torch.cat([kl[b:b + 1, :, L0:] for b in range(B)], 2)
    vn = torch.cat([vl[b:b + 1, :, L0:] for b in range(B)], 2)
    q = fa.random_tensor(23, (B, Hq, 1, D), device=dev)
    cfg = fa.AttentionConfig(gqa_group=Hq // Hkv)
    lbm = fa.create_block_mask(fa.offset_mask(fa.causal(), L0), 1, 1, 1, L0 + 1, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    pbm = fa.convert_block_mask(lbm, cache.page_table())  # allocation of the converted mask
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm the capturing stream's scratch words (no pool mutation)
        fa.convert_block_mask(lbm, cache.page_table(), out=pbm, status=status)
        fa.decode(q, cache.k_phys(), cache.v_phys(), L0 - 1, fa.causal(), fa.noop_score(),
                  fa.convert_block_mask(fa.create_block_mask(fa.offset_mask(fa.causal(), L0 - 1), 1, 1, 1, L0,
                                                             device=dev), cache.page_table()),
                  cfg=cfg, page_table=cache.page_table())
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        cache.append_batch(ids, ones, kn, vn, sync=False)
        pt = cache.page_table(max_seq_len=L0 + 1)
        fa.convert_block_mask(lbm, pt, out=pbm, status=status)
        res_g = fa.decode(q, cache.k_phys(), cache.v_phys(), L0, fa.causal(), fa.noop_score(), pbm, cfg=cfg,
                          page_table=pt)
    graph.replay()
    torch.cuda.synchronize()
    assert cache.status() == B and int(status.item()) == 0
    assert [cache.seq_len(b) for b in range(B)] == [L0 + 1] * B
    pt = cache.page_table()
    res_e = fa.decode(q, cache.k_phys(), cache.v_phys(), L0, fa.causal(), fa.noop_score(),
                      fa.convert_block_mask(lbm, pt), cfg=cfg, page_table=pt)
    unpaged = fa.decode(q, kl, vl, L0, fa.causal(), fa.noop_score(), lbm, cfg=cfg)
    torch.cuda.synchronize()
    assert torch.equal(res_g.out, res_e.out) and torch.equal(res_g.lse, res_e.lse)
    assert torch.equal(res_g.out, unpaged.out)
