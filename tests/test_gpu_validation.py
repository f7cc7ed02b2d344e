"""GPU: the reference's data-dependent checks and counters through the Python API (ABI v3).

* OpCounters (engine.hpp:21-32): the reference's counter tests — block sparsity in the counters
  (test_engine.cpp:306-326), the full-block fast path is exactly accounted for
  (test_engine.cpp:273-304, acceptance.cpp:280-309), checked against the reference's own
  counters where oracle/_ref is built.
* NonFiniteInput for q/k/v (validate.hpp:36-38) and d_out (engine.cpp:196).
* UnmappedPhysicalIndex for a paged decode that visits another batch element's page
  (paged_kv.cpp:259-272).
* Deterministic backward: bitwise run-to-run reproducibility (test_engine.cpp:242-271,
  README.md:104-106).
"""
import dataclasses

import pytest
import torch

from helpers import mask_pair, rel_err, score_pair

pytestmark = pytest.mark.gpu


def test_counters_block_sparsity(fa, dev):
    # test_engine.cpp:306-326 (fp32 path and bf16 tensor-core path count identically)
    L, D = 512, 64
    for dt in (torch.float32, torch.bfloat16):
        q, k, v = (fa.random_tensor(701 + i, (1, 1, L, D), dtype=dt, device=dev) for i in range(3))
        c_ops, d_ops = fa.OpCounters(), fa.OpCounters()
        fa.forward(q, k, v, fa.noop_score(), fa.create_block_mask(fa.causal(), 1, 1, L, L, device=dev),
                   counters=c_ops)
        fa.forward(q, k, v, fa.noop_score(), fa.create_block_mask(fa.noop_mask(), 1, 1, L, L, device=dev),
                   counters=d_ops)
        assert c_ops.mask_evals == 4 * 128 * 128
        assert d_ops.mask_evals == 0
        assert c_ops.score_evals == L * (L + 1) // 2
        assert d_ops.score_evals == L * L
        assert 0.40 < c_ops.madds / d_ops.madds <= 0.60


def test_counters_full_block_fast_path(fa, dev):
    # test_engine.cpp:273-304: demoting full blocks adds exactly full_blocks * bs^2 * B * H mask
    # evaluations and nothing else; promoting empty blocks adds empties * bs^2 * B * H
    B, H, L, D, bs = 1, 2, 256, 8, 64
    q, k, v = (fa.random_tensor(601 + i, (B, H, L, D), dtype=torch.float32, device=dev) for i in range(3))
    cfg = fa.AttentionConfig(block_size_q=bs, block_size_kv=bs)
    bm = fa.create_block_mask(fa.causal(), 1, 1, L, L, bs, bs, device=dev)
    fast, slow, padded = fa.OpCounters(), fa.OpCounters(), fa.OpCounters()
    a = fa.forward(q, k, v, fa.noop_score(), bm, cfg, counters=fast)
    b = fa.forward(q, k, v, fa.noop_score(), fa.demote_full_to_partial(bm), cfg, counters=slow)
    c = fa.forward(q, k, v, fa.noop_score(), fa.promote_empty_to_partial(bm), cfg, counters=padded)
    torch.cuda.synchronize()
    rep = fa.sparsity(bm)
    assert torch.equal(a.out, b.out) and torch.equal(a.out, c.out)
    assert fast.madds == slow.madds == padded.madds
    assert fast.score_evals == slow.score_evals
    assert slow.mask_evals - fast.mask_evals == rep.full_blocks * bs * bs * B * H
    assert padded.mask_evals - fast.mask_evals == rep.empty_blocks * bs * bs * B * H


@pytest.mark.parametrize("mname,sname", [("causal", "noop"), ("sliding:100", "alibi"), ("doc", "softcap:20"),
                                         ("hash:909:128", "noop")])
def test_counters_match_reference(fa, O, dev, mname, sname):
    # mask_evals / score_evals exactly the reference's, forward and backward
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    B, H, L, D, bs = 1, 2, 300, 16, 64
    fm, om = mask_pair(mname, L)
    fs, os_ = score_pair(sname, H)
    q, k, v, do = (fa.random_tensor(900 + i, (B, H, L, D), dtype=torch.float32, device=dev) for i in range(4))
    cfg = fa.AttentionConfig(block_size_q=bs, block_size_kv=bs)
    bm = fa.create_block_mask(fm, 1, 1, L, L, bs, bs, device=dev)
    cf, cb = fa.OpCounters(), fa.OpCounters()
    res = fa.forward(q, k, v, fs, bm, cfg, counters=cf)
    fa.backward(q, k, v, res, do, fs, bm, cfg=cfg, counters=cb)
    want_f, want_b = O.ref_counters(q.cpu().numpy(), k.cpu().numpy(), v.cpu().numpy(), do.cpu().numpy(),
                                    om, os_, bs=bs)
    assert (cf.mask_evals, cf.score_evals) == (want_f[1], want_f[2])
    assert (cb.mask_evals, cb.score_evals) == (want_b[1], want_b[2])
    # madds: the reference adds D per accumulator rescale on top of ours (forward only)
    assert cf.madds <= want_f[0] and (want_f[0] - cf.madds) % D == 0
    assert cb.madds == want_b[0]


def test_nonfinite_inputs(fa, dev):
    q, k, v, do = (fa.random_tensor(50 + i, (1, 2, 256, 128), device=dev) for i in range(4))
    bm = fa.create_block_mask(fa.causal(), 1, 1, 256, 256, device=dev)
    res = fa.forward(q, k, v, fa.noop_score(), bm, validate=True)  # finite: no error
    fa.backward(q, k, v, res, do, fa.noop_score(), bm, validate=True)
    for name, t in (("q", q), ("k", k), ("v", v)):
        bad = t.clone()
        bad.view(-1)[12345] = float("nan") if name != "v" else float("inf")
        args = {"q": q, "k": k, "v": v}
        args[name] = bad
        with pytest.raises(fa.NonFiniteInput, match=name):
            fa.forward(args["q"], args["k"], args["v"], fa.noop_score(), bm, validate=True)
        with pytest.raises(fa.NonFiniteInput, match=name):
            fa.check_finite(("q", args["q"]), ("k", args["k"]), ("v", args["v"]))
    bad_do = do.clone()
    bad_do.view(-1)[-1] = float("-inf")
    with pytest.raises(fa.NonFiniteInput, match="d_out"):
        fa.backward(q, k, v, res, bad_do, fa.noop_score(), bm, validate=True)
    # fp32 path (CUDA-core backward): d_out scanned before the passes
    qf = q.float()
    bmf = fa.create_block_mask(fa.causal(), 1, 1, 256, 256, 64, 64, device=dev)
    cfg = fa.AttentionConfig(block_size_q=64, block_size_kv=64)
    rf = fa.forward(qf, qf, qf, fa.noop_score(), bmf, cfg)
    with pytest.raises(fa.NonFiniteInput, match="d_out"):
        fa.backward(qf, qf, qf, rf, bad_do.float(), fa.noop_score(), bmf, cfg=cfg, validate=True)


def test_unmapped_physical_index(fa, dev):
    B, H, L, D, ps = 2, 2, 512, 128, 128
    cache = fa.PagedKVCache(B, B * (L // ps) + B, ps, H, D, device=dev)
    cache.shuffle_free_pages(0x77)
    kl, vl = fa.random_tensor(1, (B, H, L, D), device=dev), fa.random_tensor(2, (B, H, L, D), device=dev)
    for b in range(B):
        cache.assign(b, kl[b:b + 1], vl[b:b + 1])
    q = fa.random_tensor(3, (B, H, 1, D), device=dev)
    lbm = fa.create_block_mask(fa.offset_mask(fa.causal(), L - 1), 1, 1, 1, L, device=dev)
    pt = cache.page_table()
    pbm = fa.convert_block_mask(lbm, pt)
    fa.decode(q, cache.k_phys(), cache.v_phys(), L - 1, fa.causal(), fa.noop_score(), pbm, page_table=pt,
              validate=True)  # every page is the row's own
    cols = pbm.cols
    idx = pbm.kv_indices.clone()
    idx[cols:2 * cols] = pbm.kv_indices[0:cols]  # batch 1 reads batch 0's pages
    bad = dataclasses.replace(pbm, kv_indices=idx)
    with pytest.raises(fa.UnmappedPhysicalIndex):
        fa.decode(q, cache.k_phys(), cache.v_phys(), L - 1, fa.causal(), fa.noop_score(), bad,
                  page_table=pt, validate=True)


@pytest.mark.parametrize("shape", [
    dict(B=1, Hq=4, Hkv=4, L=4096, mname="causal", sname="noop"),
    dict(B=2, Hq=4, Hkv=1, L=2048, mname="sliding:700", sname="alibi", Bkv=1),
    dict(B=1, Hq=2, Hkv=2, L=1000, mname="doc", sname="softcap:20", D=64),
])
def test_deterministic_backward_bitwise(fa, O, dev, shape):
    # test_engine.cpp:242-271: results independent of scheduling, bit for bit
    B, Hq, Hkv, L = shape["B"], shape["Hq"], shape["Hkv"], shape["L"]
    D, Bkv = shape.get("D", 128), shape.get("Bkv", B)
    fm, om = mask_pair(shape["mname"], L)
    fs, os_ = score_pair(shape["sname"], Hq)
    q, do = (fa.random_tensor(70 + i, (B, Hq, L, D), device=dev) for i in (0, 3))
    k, v = (fa.random_tensor(70 + i, (Bkv, Hkv, L, D), device=dev) for i in (1, 2))
    cfg = fa.AttentionConfig(gqa_group=Hq // Hkv)
    bm = fa.create_block_mask(fm, 1, 1, L, L, device=dev)
    res = fa.forward(q, k, v, fs, bm, cfg)
    runs = [fa.backward(q, k, v, res, do, fs, bm, cfg=cfg, deterministic=True) for _ in range(4)]
    torch.cuda.synchronize()
    for g in runs[1:]:
        assert torch.equal(g.dq, runs[0].dq) and torch.equal(g.dk, runs[0].dk) and torch.equal(g.dv, runs[0].dv)
    # and the deterministic gradients are the same gradients (vs the default mode and the oracle)
    g0 = fa.backward(q, k, v, res, do, fs, bm, cfg=cfg)
    assert (g0.dq.float() - runs[0].dq.float()).abs().max().item() <= 1e-2
    assert torch.equal(g0.dk, runs[0].dk) and torch.equal(g0.dv, runs[0].dv)
    qf, kf, vf, dof = (x.float().cpu().numpy() for x in (q, k, v, do))
    dq_r, _, _ = O.backward(qf, kf, vf, res.out.float().cpu().numpy(), res.lse.cpu().numpy(), dof, om, os_,
                            O.create_block_mask(om, 1, 1, L, L), gqa=Hq // Hkv)
    assert rel_err(runs[0].dq.float().cpu().numpy(), dq_r) <= 2e-2
