"""Backward parity on the GPU vs the oracle's backward (engine.cpp:174-401) on identical inputs.

Gate: max-abs(got - ref) / max(1, max|ref|) <= 2e-2 per gradient for bf16
(the reference's rel_grad_err form, bench.cpp:398-403); 1e-4 for the fp32 path.
"""
import numpy as np
import pytest
import torch

from helpers import mask_pair, rel_err, score_pair

pytestmark = pytest.mark.gpu


def run_bwd(fa, O, dev, mname, sname, B=1, Hq=2, Hkv=2, Lq=384, Lkv=384, D=128, bs=128,
            dtype=torch.bfloat16, Bkv=None, seed=300, mask_dims=(1, 1), deterministic=False):
    Bkv = B if Bkv is None else Bkv
    fm, om = mask_pair(mname, max(Lq, Lkv))
    fs, os_ = score_pair(sname, Hq)
    q = fa.random_tensor(seed + 1, (B, Hq, Lq, D), dtype=dtype, device=dev)
    k = fa.random_tensor(seed + 2, (Bkv, Hkv, Lkv, D), dtype=dtype, device=dev)
    v = fa.random_tensor(seed + 3, (Bkv, Hkv, Lkv, D), dtype=dtype, device=dev)
    do = fa.random_tensor(seed + 4, (B, Hq, Lq, D), dtype=dtype, device=dev)
    bm = fa.create_block_mask(fm, mask_dims[0], mask_dims[1], Lq, Lkv, bs, bs, device=dev)
    cfg = fa.AttentionConfig(gqa_group=Hq // Hkv, block_size_q=bs, block_size_kv=bs)
    fwd = fa.forward(q, k, v, fs, bm, cfg)
    g = fa.backward(q, k, v, fwd, do, fs, bm, cfg=cfg, deterministic=deterministic)
    torch.cuda.synchronize()
    qf, kf, vf, dof = (x.float().cpu().numpy() for x in (q, k, v, do))
    obm = O.create_block_mask(om, mask_dims[0], mask_dims[1], Lq, Lkv, bs, bs)
    o_ref, l_ref = O.forward(qf, kf, vf, om, os_, obm, gqa=Hq // Hkv)
    # the GPU backward consumes the GPU forward's O/lse; feed the oracle the same statistics
    o_gpu = fwd.out.float().cpu().numpy()
    l_gpu = fwd.lse.cpu().numpy()
    dq, dk, dv = O.backward(qf, kf, vf, o_gpu, l_gpu, dof, om, os_, obm, gqa=Hq // Hkv)
    return [rel_err(a.float().cpu().numpy(), b) for a, b in ((g.dq, dq), (g.dk, dk), (g.dv, dv))]


@pytest.mark.parametrize("mname", ["noop", "causal", "sliding:200", "doc_causal", "hash:909:200"])
@pytest.mark.parametrize("sname", ["noop", "alibi", "softcap:20", "stacked:5"])
def test_bwd_masks_scores(fa, O, dev, mname, sname):
    errs = run_bwd(fa, O, dev, mname, sname)
    assert max(errs) <= 2e-2, errs


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("shape", [(384, 384), (300, 500), (500, 260)])
def test_bwd_shapes(fa, O, dev, D, shape):
    errs = run_bwd(fa, O, dev, "causal" if shape[0] == shape[1] else "noop", "noop", Lq=shape[0],
                   Lkv=shape[1], D=D)
    assert max(errs) <= 2e-2, errs


def test_bwd_gqa_broadcast(fa, O, dev):
    # shared kv batch + GQA group loop (engine.cpp:326-331)
    errs = run_bwd(fa, O, dev, "causal", "alibi", B=2, Hq=4, Hkv=1, Bkv=1, Lq=256, Lkv=256)
    assert max(errs) <= 2e-2, errs


@pytest.mark.parametrize("mname", ["noop", "causal", "sliding:200", "doc_causal", "hash:909:200"])
@pytest.mark.parametrize("sname", ["noop", "alibi", "softcap:20"])
def test_bwd_deterministic_masks_scores(fa, O, dev, mname, sname):
    # the split backward (dK/dV-only kernel + the TMEM-accumulating dQ pass, bwd_dq.cuh)
    errs = run_bwd(fa, O, dev, mname, sname, deterministic=True)
    assert max(errs) <= 2e-2, errs


@pytest.mark.parametrize("D", [64, 128])
def test_bwd_deterministic_shapes_gqa(fa, O, dev, D):
    errs = run_bwd(fa, O, dev, "causal", "alibi", B=2, Hq=4, Hkv=2, Bkv=1, Lq=500, Lkv=500, D=D, deterministic=True)
    assert max(errs) <= 2e-2, errs
    errs = run_bwd(fa, O, dev, "noop", "noop", Lq=300, Lkv=700, D=D, deterministic=True)
    assert max(errs) <= 2e-2, errs


def test_bwd_fp32(fa, O, dev):
    errs = run_bwd(fa, O, dev, "causal", "softcap:20", B=2, Hq=4, Hkv=2, Lq=60, Lkv=60, D=16, bs=16,
                   dtype=torch.float32)
    assert max(errs) <= 1e-4, errs


def test_zero_dout_gives_zero_grads(fa, dev):
    # test_engine.cpp:388-402
    q = fa.random_tensor(1, (1, 2, 256, 128), device=dev)
    k = fa.random_tensor(2, (1, 2, 256, 128), device=dev)
    bm = fa.create_block_mask(fa.causal(), 1, 1, 256, 256, device=dev)
    fwd = fa.forward(q, k, k, fa.noop_score(), bm)
    g = fa.backward(q, k, k, fwd, torch.zeros_like(q), fa.noop_score(), bm)
    for t in (g.dq, g.dk, g.dv):
        assert torch.count_nonzero(t).item() == 0


def test_bwd_c2_slice(fa, O, dev):
    # BASELINE C2 geometry (sliding 1024 + ALiBi, S 8192, D 128) on one (b, h) slice
    B, H, L, D = 1, 1, 8192, 128
    fm, om = mask_pair("sliding:1024", L)
    sl = fa.alibi_slopes(16)[5]
    fs, os_ = fa.alibi([sl]), O.Score(terms=O.SCORE_ALIBI, slopes=np.array([sl]))
    q, k, v, do = (fa.random_tensor(0x5EED0001 + i, (B, H, L, D), device=dev) for i in range(1, 5))
    bm = fa.create_block_mask(fm, 1, 1, L, L, device=dev)
    fwd = fa.forward(q, k, v, fs, bm)
    g = fa.backward(q, k, v, fwd, do, fs, bm)
    torch.cuda.synchronize()
    qf, kf, vf, dof = (x.float().cpu().numpy() for x in (q, k, v, do))
    obm = O.create_block_mask(om, 1, 1, L, L)
    dq, dk, dv = O.backward(qf, kf, vf, fwd.out.float().cpu().numpy(), fwd.lse.cpu().numpy(), dof,
                            om, os_, obm)
    errs = [rel_err(a.float().cpu().numpy(), b) for a, b in ((g.dq, dq), (g.dk, dk), (g.dv, dv))]
    assert max(errs) <= 2e-2, errs
