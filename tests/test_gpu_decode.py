"""Paged split-KV decode on the GPU: vs the oracle (decode = forward rows with the offset shift,
engine.cpp:403-427), paged == unpaged bit for bit (acceptance.cpp:312-345 contract), and the
page-converted BlockMask bit-exact vs convert_block_mask (paged_kv.cpp:154-228)."""
import dataclasses

import numpy as np
import pytest
import torch

from helpers import lse_err, mask_pair, score_pair

pytestmark = pytest.mark.gpu


def make_cache(fa, dev, B, H, L, D, ps=128, seed=0xFA6E5):
    cache = fa.PagedKVCache(B, B * (-(-L // ps)) + B, ps, H, D, device=dev)
    cache.shuffle_free_pages(seed)
    kl = fa.random_tensor(31, (B, H, L, D), device=dev)
    vl = fa.random_tensor(32, (B, H, L, D), device=dev)
    for b in range(B):
        cache.assign(b, kl[b:b + 1], vl[b:b + 1])
    return cache, kl, vl


@pytest.mark.parametrize("sname", ["noop", "alibi"])
@pytest.mark.parametrize("splits", [0, 1, 3])
def test_paged_decode_vs_oracle_and_unpaged(fa, O, dev, sname, splits):
    B, H, L, D, n_new = 3, 4, 1000, 128, 1
    off = L - n_new
    cache, kl, vl = make_cache(fa, dev, B, H, L, D)
    q = fa.random_tensor(33, (B, H, n_new, D), device=dev)
    fs, os_ = score_pair(sname, H)
    lbm = fa.create_block_mask(fa.offset_mask(fa.causal(), off), 1, 1, n_new, L, device=dev)
    pt = cache.page_table()
    pbm = fa.convert_block_mask(lbm, pt)
    paged = fa.decode(q, cache.k_phys(), cache.v_phys(), off, fa.causal(), fs, pbm, page_table=pt,
                      num_splits=splits)
    unpaged = fa.decode(q, kl, vl, off, fa.causal(), fs, lbm, num_splits=splits)
    torch.cuda.synchronize()
    assert torch.equal(paged.out, unpaged.out) and torch.equal(paged.lse, unpaged.lse)
    om = O.causal(off)
    os_.q_offset = off
    o_ref, l_ref = O.forward(q.float().cpu().numpy(), kl.float().cpu().numpy(), vl.float().cpu().numpy(),
                             om, os_, O.create_block_mask(om, 1, 1, n_new, L))
    assert np.abs(paged.out.float().cpu().numpy() - o_ref).max() <= 2e-2
    assert lse_err(paged.lse.cpu().numpy(), l_ref) <= 2e-2


def test_chunked_decode_rows_match_forward(fa, dev):
    # test_engine.cpp:443-491: decode of rows [off, off+n) equals those rows of the full forward
    B, H, L, D, n = 1, 2, 640, 128, 4
    q = fa.random_tensor(41, (B, H, L, D), device=dev)
    k = fa.random_tensor(42, (B, H, L, D), device=dev)
    v = fa.random_tensor(43, (B, H, L, D), device=dev)
    full = fa.forward(q, k, v, fa.noop_score(), fa.create_block_mask(fa.causal(), 1, 1, L, L, device=dev))
    off = 300
    bm = fa.create_block_mask(fa.offset_mask(fa.causal(), off), 1, 1, n, L, device=dev)
    step = fa.decode(q[:, :, off:off + n].contiguous(), k, v, off, fa.causal(), fa.noop_score(), bm)
    torch.cuda.synchronize()
    assert (step.out.float() - full.out[:, :, off:off + n].float()).abs().max().item() <= 2e-2
    assert (step.lse - full.lse[:, :, off:off + n]).abs().max().item() <= 2e-2


def test_convert_block_mask_exact(fa, O, dev):
    B, L, ps = 4, 1000, 128
    cache = fa.PagedKVCache(B, B * 8 + B, ps, 1, 64, device=dev)
    cache.shuffle_free_pages(0x1234)
    t = torch.zeros((1, 1, L, 64), dtype=torch.bfloat16, device=dev)
    for b in range(B):
        cache.assign(b, t, t)
    pt = cache.page_table()
    lbm = fa.create_block_mask(fa.causal(), 1, 1, L, L, device=dev)
    pbm = fa.convert_block_mask(lbm, pt)
    obm = O.create_block_mask(O.causal(), 1, 1, L, L)
    want = O.convert_block_mask(obm, np.array(pt.table, np.int32).reshape(B, -1), pt.num_physical_pages)
    assert np.array_equal(pbm.kv_indices.cpu().numpy(), want.partial_idx)
    assert np.array_equal(pbm.full_kv_indices.cpu().numpy(), want.full_idx)
    assert np.array_equal(pbm.kv_num_blocks.cpu().numpy(), want.partial_num)
    if O.ref_available():
        tbl, p2l, own = O.ref_paged_layout(B, B * 8 + B, ps, 0x1234, L)
        assert np.array_equal(tbl.reshape(-1), np.array(pt.table, np.int32))   # same LIFO + shuffle
        assert np.array_equal(p2l, np.array(pt.phys_to_logical, np.int32))
        rpn, rpi, rfn, rfi = O.ref_convert_block_mask(O.causal(), 1, 1, L, L, ps, tbl, B * 8 + B)
        assert np.array_equal(pbm.kv_indices.cpu().numpy(), rpi)
        assert np.array_equal(pbm.full_kv_indices.cpu().numpy(), rfi)


def test_unmapped_block_raises(fa, dev):
    cache = fa.PagedKVCache(2, 4, 128, 1, 64, device=dev)
    t = torch.zeros((1, 1, 128, 64), dtype=torch.bfloat16, device=dev)
    cache.assign(0, t, t)  # batch 1 left unmapped
    lbm = fa.create_block_mask(fa.causal(), 1, 1, 128, 128, device=dev)
    with pytest.raises(fa.UnmappedBlock):
        fa.convert_block_mask(lbm, cache.page_table())


def test_offset_out_of_range(fa, dev):
    q = fa.random_tensor(1, (1, 1, 1, 128), device=dev)
    k = fa.random_tensor(2, (1, 1, 256, 128), device=dev)
    bm = fa.create_block_mask(fa.offset_mask(fa.causal(), 255), 1, 1, 1, 256, device=dev)
    with pytest.raises(fa.OffsetOutOfRange):
        fa.decode(q, k, k, 256, fa.causal(), fa.noop_score(), bm)


@pytest.mark.parametrize("Hq,Hkv,n_new,L,sname,mname", [(8, 2, 1, 1000, "noop", "causal"),
                                                        (8, 2, 3, 1000, "alibi", "causal"),
                                                        (4, 4, 5, 777, "noop", "causal"),
                                                        (16, 1, 8, 640, "softcap", "causal"),
                                                        (8, 2, 70, 900, "noop", "causal"),
                                                        (8, 2, 4, 1000, "alibi", "sliding:300"),
                                                        (4, 1, 6, 850, "stacked", "sliding:130")])
def test_packed_rows_decode_vs_oracle_and_unpaged(fa, O, dev, Hq, Hkv, n_new, L, sname, mname):
    """GQA groups and multi-token steps (several rows per kv head) take the tensor-core decode,
    which packs the G heads x n_new rows into one 128-row tile so every page streams once per
    (batch element, kv head): vs the oracle (decode = forward rows with the offset shift,
    engine.cpp:403-427), and paged == unpaged bit for bit (acceptance.cpp:312-345)."""
    B, D = 3, 128
    off = L - n_new
    G = Hq // Hkv
    cache, kl, vl = make_cache(fa, dev, B, Hkv, L, D)
    q = fa.random_tensor(34, (B, Hq, n_new, D), device=dev)
    fs, os_ = score_pair(sname, Hq)
    cfg = fa.AttentionConfig(gqa_group=G)
    fm, om = mask_pair(mname, L)
    lbm = fa.create_block_mask(fa.offset_mask(fm, off), 1, 1, n_new, L, device=dev)
    pt = cache.page_table()
    pbm = fa.convert_block_mask(lbm, pt)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        paged = fa.decode(q, cache.k_phys(), cache.v_phys(), off, fm, fs, pbm, cfg=cfg, page_table=pt)
        torch.cuda.synchronize()
    assert any("decode_tc_kernel" in e.name for e in prof.events()), "the tensor-core decode did not run"
    unpaged = fa.decode(q, kl, vl, off, fm, fs, lbm, cfg=cfg)
    torch.cuda.synchronize()
    assert torch.equal(paged.out, unpaged.out) and torch.equal(paged.lse, unpaged.lse)
    om = dataclasses.replace(om, q_offset=off)
    os_.q_offset = off
    o_ref, l_ref = O.forward(q.float().cpu().numpy(), kl.float().cpu().numpy(), vl.float().cpu().numpy(),
                             om, os_, O.create_block_mask(om, 1, 1, n_new, L), gqa=G)
    assert np.abs(paged.out.float().cpu().numpy() - o_ref).max() <= 2e-2
    assert lse_err(paged.lse.cpu().numpy(), l_ref) <= 2e-2
