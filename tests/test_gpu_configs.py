"""Parity at the BASELINE.json geometries that the per-variant grids do not reach.

* C3 backward: one head of and_mask(document_mask(8 docs), causal), S=16384, D=128 bf16.
* C4 backward: one GQA group (4 q heads on 1 kv head) of causal + soft_cap(50), S=8192.
* C5 paged decode at full size: B64 H32 KV_LEN 32768, page 128; the page-converted BlockMask
  (64,1,1,16448) bit-exact vs convert_block_mask, paged output == unpaged output bit for bit
  (acceptance.cpp:312-345), 8 (b, h) rows within 2e-2 of the oracle.

The checker is the reference itself (oracle/_ref, backward<float> of engine.cpp:174-401 run
with all host threads) where it was built, else the C restatement (oracle/flex_oracle.c).
Gate: O/lse max-abs <= 2e-2; gradients max-abs / max(1, max|ref|) <= 2e-2.
"""
import os

import numpy as np
import pytest
import torch

from helpers import c3_doc_ids, lse_err, rel_err

pytestmark = pytest.mark.gpu

SEED = 0x5EED0001
TOL = 2e-2


def _bwd_check(fa, O, dev, fm, om, fs, os_, B, Hq, Hkv, L, D, seed):
    q = fa.random_tensor(seed + 1, (B, Hq, L, D), device=dev)
    k = fa.random_tensor(seed + 2, (B, Hkv, L, D), device=dev)
    v = fa.random_tensor(seed + 3, (B, Hkv, L, D), device=dev)
    do = fa.random_tensor(seed + 4, (B, Hq, L, D), device=dev)
    cfg = fa.AttentionConfig(gqa_group=Hq // Hkv)
    bm = fa.create_block_mask(fm, 1, 1, L, L, device=dev)
    fwd = fa.forward(q, k, v, fs, bm, cfg)
    g = fa.backward(q, k, v, fwd, do, fs, bm, cfg=cfg)
    torch.cuda.synchronize()
    qf, kf, vf, dof = (x.float().cpu().numpy() for x in (q, k, v, do))
    got = [t.float().cpu().numpy() for t in (fwd.out, g.dq, g.dk, g.dv)]
    if O.ref_available():
        os.environ["BLOCKATTN_WORKERS"] = str(os.cpu_count() or 1)
        o_r, l_r, dq_r, dk_r, dv_r = O.ref_backward(qf, kf, vf, dof, om, os_, gqa=Hq // Hkv)
    else:
        obm = O.create_block_mask(om, 1, 1, L, L)
        o_r, l_r = O.forward(qf, kf, vf, om, os_, obm, gqa=Hq // Hkv)
        dq_r, dk_r, dv_r = O.backward(qf, kf, vf, got[0], fwd.lse.cpu().numpy(), dof, om, os_, obm,
                                      gqa=Hq // Hkv)
    e_o = float(np.abs(got[0] - o_r).max())
    e_l = lse_err(fwd.lse.cpu().numpy(), l_r)
    errs = [rel_err(a, b) for a, b in zip(got[1:], (dq_r, dk_r, dv_r))]
    return e_o, e_l, errs


def test_c3_backward_one_head(fa, O, dev):
    ids = c3_doc_ids()
    fm = fa.and_mask(fa.document_mask(ids), fa.causal())
    om = O.Mask(terms=O.MASK_DOCUMENT | O.MASK_CAUSAL, doc_ids=ids)
    e_o, e_l, errs = _bwd_check(fa, O, dev, fm, om, fa.noop_score(), O.Score(), 1, 1, 1, 16384, 128,
                                SEED)
    assert e_o <= TOL and e_l <= TOL, (e_o, e_l)
    assert max(errs) <= TOL, errs


def test_c4_backward_one_gqa_group(fa, O, dev):
    fm, om = fa.causal(), O.Mask(terms=O.MASK_CAUSAL)
    fs, os_ = fa.soft_cap(50.0), O.Score(terms=O.SCORE_SOFTCAP, cap=50.0)
    e_o, e_l, errs = _bwd_check(fa, O, dev, fm, om, fs, os_, 1, 4, 1, 8192, 128, SEED + 7)
    assert e_o <= TOL and e_l <= TOL, (e_o, e_l)
    assert max(errs) <= TOL, errs


def test_c5_paged_decode_full(fa, O, dev):
    B, H, L, D, ps = 64, 32, 32768, 128, 128
    pages = B * (L // ps) + B  # 16448 (bench.cpp:553-555)
    off = L - 1
    cache = fa.PagedKVCache(B, pages, ps, H, D, device=dev)
    cache.shuffle_free_pages(SEED ^ 0xFA6E5)
    kl = fa.random_tensor(SEED + 2, (B, H, L, D), device=dev)  # logical K/V, 17.2 GB each
    vl = fa.random_tensor(SEED + 3, (B, H, L, D), device=dev)
    for b in range(B):  # assign b = 0..63 in order, 256 pages each (bench.cpp:553-560)
        cache.assign(b, kl[b:b + 1], vl[b:b + 1])
    q = fa.random_tensor(SEED + 1, (B, H, 1, D), device=dev)
    lbm = fa.create_block_mask(fa.offset_mask(fa.causal(), off), 1, 1, 1, L, device=dev)
    pt = cache.page_table()
    pbm = fa.convert_block_mask(lbm, pt)
    assert (pbm.b_dims, pbm.h_dims, pbm.rows, pbm.cols) == (64, 1, 1, 16448)
    # converted BlockMask bit-exact vs convert_block_mask (paged_kv.cpp:154-228)
    om = O.causal(off)
    obm = O.create_block_mask(om, 1, 1, 1, L)
    table = np.asarray(pt.table, np.int32).reshape(B, -1)
    want = O.convert_block_mask(obm, table, pages)
    for got, w in ((pbm.kv_num_blocks, want.partial_num), (pbm.kv_indices, want.partial_idx),
                   (pbm.full_kv_num_blocks, want.full_num), (pbm.full_kv_indices, want.full_idx)):
        assert np.array_equal(got.cpu().numpy().astype(np.int64), np.asarray(w, np.int64).reshape(-1))
    if O.ref_available():
        rpn, rpi, rfn, rfi = O.ref_convert_block_mask(om, 1, 1, 1, L, ps, table, pages)
        assert np.array_equal(pbm.kv_indices.cpu().numpy(), rpi.reshape(-1))
        assert np.array_equal(pbm.kv_num_blocks.cpu().numpy(), rpn.reshape(-1))
    # paged == unpaged, bit for bit
    paged = fa.decode(q, cache.k_phys(), cache.v_phys(), off, fa.causal(), fa.noop_score(), pbm,
                      page_table=pt)
    unpaged = fa.decode(q, kl, vl, off, fa.causal(), fa.noop_score(), lbm)
    torch.cuda.synchronize()
    assert torch.equal(paged.out, unpaged.out) and torch.equal(paged.lse, unpaged.lse)
    # 8 (b, h) rows vs the oracle forward rows (decode == forward rows, engine.cpp:403-427)
    for b, h in ((0, 0), (7, 31), (13, 5), (21, 17), (34, 8), (45, 29), (58, 2), (63, 16)):
        o_r, l_r = O.forward(q[b:b + 1, h:h + 1].float().cpu().numpy(),
                             kl[b:b + 1, h:h + 1].float().cpu().numpy(),
                             vl[b:b + 1, h:h + 1].float().cpu().numpy(), om, O.Score(), obm)
        e_o = float(np.abs(paged.out[b:b + 1, h:h + 1].float().cpu().numpy() - o_r).max())
        e_l = lse_err(paged.lse[b:b + 1, h:h + 1].cpu().numpy(), l_r)
        assert e_o <= TOL and e_l <= TOL, (b, h, e_o, e_l)
