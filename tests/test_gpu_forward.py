"""Forward parity on the GPU vs the oracle's forward<float> on identical (bf16-rounded) inputs.

Tolerances: bf16 tcgen05 path O max-abs <= 2e-2 and lse <= 2e-2 abs
(natural log, -inf in the same rows); fp32 CUDA-core path (config C1) <= 1e-4.
"""
import numpy as np
import pytest
import torch

from helpers import lse_err, mask_pair, score_pair

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
F32_TOL = 1e-4


def run_case(fa, O, dev, mname, sname, B=2, Hq=4, Hkv=4, Lq=512, Lkv=512, D=128, bs=128,
             dtype=torch.bfloat16, Bkv=None, mask_dims=(1, 1), seed=100, scale=None):
    Bkv = B if Bkv is None else Bkv
    fm, om = mask_pair(mname, max(Lq, Lkv))
    fs, os_ = score_pair(sname, Hq)
    q = fa.random_tensor(seed + 1, (B, Hq, Lq, D), dtype=dtype, device=dev)
    k = fa.random_tensor(seed + 2, (Bkv, Hkv, Lkv, D), dtype=dtype, device=dev)
    v = fa.random_tensor(seed + 3, (Bkv, Hkv, Lkv, D), dtype=dtype, device=dev)
    bm = fa.create_block_mask(fm, mask_dims[0], mask_dims[1], Lq, Lkv, bs, bs, device=dev)
    cfg = fa.AttentionConfig(scale=scale, gqa_group=Hq // Hkv, block_size_q=bs, block_size_kv=bs)
    res = fa.forward(q, k, v, fs, bm, cfg)
    torch.cuda.synchronize()
    qf, kf, vf = (x.float().cpu().numpy() for x in (q, k, v))
    obm = O.create_block_mask(om, mask_dims[0], mask_dims[1], Lq, Lkv, bs, bs)
    o_ref, l_ref = O.forward(qf, kf, vf, om, os_, obm, scale=scale, gqa=Hq // Hkv)
    got_o = res.out.float().cpu().numpy()
    return float(np.abs(got_o - o_ref).max()), lse_err(res.lse.cpu().numpy(), l_ref), res


MASKS = ["noop", "causal", "sliding:200", "doc_causal", "prefix:100", "hash:909:200"]
SCORES = ["noop", "alibi", "softcap:20", "stacked:5"]


@pytest.mark.parametrize("mname", MASKS)
@pytest.mark.parametrize("sname", SCORES)
def test_tcgen05_masks_scores(fa, O, dev, mname, sname):
    e_o, e_l, _ = run_case(fa, O, dev, mname, sname)
    assert e_o <= BF16_TOL and e_l <= BF16_TOL, (e_o, e_l)


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("shape", [(512, 512), (500, 700), (700, 300), (128, 1), (1, 128), (3000, 3000)])
def test_tcgen05_shapes(fa, O, dev, D, shape):
    Lq, Lkv = shape
    e_o, e_l, _ = run_case(fa, O, dev, "causal" if Lq == Lkv else "noop", "noop", B=1, Hq=2, Hkv=2,
                           Lq=Lq, Lkv=Lkv, D=D)
    assert e_o <= BF16_TOL and e_l <= BF16_TOL, (e_o, e_l)


def test_tcgen05_gqa_and_broadcast(fa, O, dev):
    # GQA 4:1 (engine.cpp:81) + kv batch broadcast (engine.cpp:80) + per-head hashed mask
    e_o, e_l, _ = run_case(fa, O, dev, "hash:77:150", "alibi", B=2, Hq=8, Hkv=2, Bkv=1, Lq=384,
                           Lkv=640, mask_dims=(2, 8))
    assert e_o <= BF16_TOL and e_l <= BF16_TOL, (e_o, e_l)


def test_tcgen05_explicit_scale(fa, O, dev):
    e_o, e_l, _ = run_case(fa, O, dev, "causal", "noop", scale=0.125)
    assert e_o <= BF16_TOL and e_l <= BF16_TOL


def test_gqa_equals_per_head(fa, dev):
    # test_engine.cpp:181-210 — each q head alone against its kv head gives the same bits
    B, Hq, Hkv, L, D = 1, 4, 2, 384, 128
    q = fa.random_tensor(201, (B, Hq, L, D), device=dev)
    k = fa.random_tensor(202, (B, Hkv, L, D), device=dev)
    v = fa.random_tensor(203, (B, Hkv, L, D), device=dev)
    bm = fa.create_block_mask(fa.causal(), 1, 1, L, L, device=dev)
    got = fa.forward(q, k, v, fa.noop_score(), bm, fa.AttentionConfig(gqa_group=2))
    for h in range(Hq):
        alone = fa.forward(q[:, h:h + 1].contiguous(), k[:, h // 2:h // 2 + 1].contiguous(),
                           v[:, h // 2:h // 2 + 1].contiguous(), fa.noop_score(), bm)
        assert torch.equal(got.out[:, h], alone.out[:, 0])
        assert torch.equal(got.lse[:, h], alone.lse[:, 0])


def test_fully_masked_rows(fa, dev):
    # test_engine.cpp:103-122 — never_mask: O = 0, lse = -inf; bf16 and fp32 paths
    for dtype, bs in ((torch.bfloat16, 128), (torch.float32, 4)):
        q = fa.random_tensor(1, (1, 1, 256, 128), dtype=dtype, device=dev)
        k = fa.random_tensor(2, (1, 1, 256, 128), dtype=dtype, device=dev)
        bm = fa.create_block_mask(fa.never_mask(), 1, 1, 256, 256, bs, bs, device=dev)
        res = fa.forward(q, k, k, fa.noop_score(), bm, fa.AttentionConfig(block_size_q=bs, block_size_kv=bs))
        assert torch.all(res.out == 0) and torch.all(torch.isneginf(res.lse))


def test_single_position_kat(fa, dev):
    # test_engine.cpp:85-101 / test_oracle.cpp:13-23: O = [5, -1.5], lse = 6 with scale 1
    q = torch.tensor([3.0, 0.0], device=dev).view(1, 1, 1, 2)
    k = torch.tensor([2.0, 5.0], device=dev).view(1, 1, 1, 2)
    v = torch.tensor([5.0, -1.5], device=dev).view(1, 1, 1, 2)
    bm = fa.create_block_mask(fa.noop_mask(), 1, 1, 1, 1, 16, 16, device=dev)
    res = fa.forward(q, k, v, fa.noop_score(), bm, fa.AttentionConfig(scale=1.0, block_size_q=16, block_size_kv=16))
    assert res.out.cpu().tolist() == [[[[5.0, -1.5]]]]
    assert abs(res.lse.item() - 6.0) < 1e-6


def test_zero_query_is_mean_of_v(fa, dev):
    # test_oracle.cpp:25-40: q = 0 -> uniform weights, O = mean(V), lse = ln L
    L, D = 256, 128
    q = torch.zeros((1, 1, L, D), dtype=torch.bfloat16, device=dev)
    k = fa.random_tensor(5, (1, 1, L, D), device=dev)
    v = fa.random_tensor(6, (1, 1, L, D), device=dev)
    bm = fa.create_block_mask(fa.noop_mask(), 1, 1, L, L, device=dev)
    res = fa.forward(q, k, v, fa.noop_score(), bm)
    mean = v.float().mean(dim=2, keepdim=True).expand(1, 1, L, D)
    assert (res.out.float() - mean).abs().max().item() <= 1e-2
    assert (res.lse - np.log(L)).abs().max().item() <= 1e-4


@pytest.mark.parametrize("bs", [16, 64])
@pytest.mark.parametrize("mname,sname", [("causal", "noop"), ("sliding:5", "alibi"),
                                         ("doc", "softcap:10"), ("prefix:7", "stacked:5"),
                                         ("hash:909:128", "noop")])
def test_fp32_simt_reference_shapes(fa, O, dev, bs, mname, sname):
    # the reference's oracle-equivalence grid (test_engine.cpp:124-179), fp32 at 1e-4
    for Lq, Lkv in ((64, 64), (60, 60), (32, 60), (60, 32)):
        md = (2, 4) if mname.startswith("hash") else (1, 1)
        e_o, e_l, _ = run_case(fa, O, dev, mname, sname, B=2, Hq=4, Hkv=4, Lq=Lq, Lkv=Lkv, D=8,
                               bs=bs, dtype=torch.float32, mask_dims=md)
        assert e_o <= F32_TOL and e_l <= F32_TOL, (Lq, Lkv, e_o, e_l)


def test_c1_fp32_full(fa, O, dev):
    # BASELINE config C1: causal B1 H4 S1024 D64 fp32, vs the reference forward<float>
    e_o, e_l, _ = run_case(fa, O, dev, "causal", "noop", B=1, Hq=4, Hkv=4, Lq=1024, Lkv=1024, D=64,
                           dtype=torch.float32, seed=0x5EED0001)
    assert e_o <= F32_TOL and e_l <= F32_TOL, (e_o, e_l)
    if O.ref_available():
        q = fa.random_tensor(0x5EED0002, (1, 4, 1024, 64), dtype=torch.float32, device=dev)
        bm = fa.create_block_mask(fa.causal(), 1, 1, 1024, 1024, device=dev)
        res = fa.forward(q, q, q, fa.noop_score(), bm)
        qn = q.cpu().numpy()
        ro, rl = O.ref_forward(qn, qn, qn, O.causal(), O.Score())
        assert np.abs(res.out.cpu().numpy() - ro).max() <= F32_TOL


def _slice_check(fa, O, dev, mname, sname, B, Hq, Hkv, L, D, b, h, seed):
    fm, om = mask_pair(mname, L)
    fs, _ = score_pair(sname, Hq)
    q = fa.random_tensor(seed + 1, (B, Hq, L, D), device=dev)
    k = fa.random_tensor(seed + 2, (B, Hkv, L, D), device=dev)
    v = fa.random_tensor(seed + 3, (B, Hkv, L, D), device=dev)
    bm = fa.create_block_mask(fm, 1, 1, L, L, device=dev)
    res = fa.forward(q, k, v, fs, bm, fa.AttentionConfig(gqa_group=Hq // Hkv))
    torch.cuda.synchronize()
    kh = h // (Hq // Hkv)
    qs, ks, vs = (x[b:b + 1, hh:hh + 1].float().cpu().numpy() for x, hh in ((q, h), (k, kh), (v, kh)))
    if sname == "alibi":
        os_ = O.Score(terms=O.SCORE_ALIBI, slopes=np.array([fa.alibi_slopes(Hq)[h]]))
    else:
        os_ = score_pair(sname, Hq)[1]
    o_ref, l_ref = O.forward(qs, ks, vs, om, os_, O.create_block_mask(om, 1, 1, L, L))
    e_o = float(np.abs(res.out[b:b + 1, h:h + 1].float().cpu().numpy() - o_ref).max())
    e_l = lse_err(res.lse[b:b + 1, h:h + 1].cpu().numpy(), l_ref)
    return e_o, e_l


@pytest.mark.parametrize("cfg", [
    ("sliding:1024", "alibi", 4, 16, 16, 8192, 128, 3, 15),   # C2 slice (b=3, h=15)
    ("doc_causal", "noop", 1, 32, 32, 16384, 128, 0, 7),      # C3 slice
    ("causal", "softcap:50", 2, 32, 8, 8192, 128, 1, 13),     # C4 slice (GQA group 3)
])
def test_config_slices(fa, O, dev, cfg):
    e_o, e_l = _slice_check(fa, O, dev, *cfg, seed=0x5EED0001)
    assert e_o <= BF16_TOL and e_l <= BF16_TOL, (e_o, e_l)


def test_long_rows_take_the_one_tile_kernel(fa, O, dev):
    """KV_LEN > 131072 (more than 1024 kv blocks per row) runs on the tensor cores through the
    one-tile kernel, which streams the visit lists from global memory (no CUDA-core fallback)."""
    B, H, L, D, w = 1, 1, 131072 + 3 * 128 + 77, 64, 200
    q = fa.random_tensor(91, (B, H, L, D), device=dev)
    k = fa.random_tensor(92, (B, H, L, D), device=dev)
    v = fa.random_tensor(93, (B, H, L, D), device=dev)
    bm = fa.create_block_mask(fa.sliding_window(w), 1, 1, L, L, device=dev)
    assert bm.cols > 1024
    res = fa.forward(q, k, v, fa.noop_score(), bm)
    torch.cuda.synchronize()
    # check the last 512 rows (the far end of the long rows) against the oracle
    lo = L - 512
    om = O.Mask(terms=O.MASK_SLIDING, window=w, q_offset=lo)
    qf = q[:, :, lo:].float().cpu().numpy()
    kf, vf = k.float().cpu().numpy(), v.float().cpu().numpy()
    o_ref, l_ref = O.forward(qf, kf, vf, om, O.Score(), O.create_block_mask(om, 1, 1, 512, L))
    assert np.abs(res.out[:, :, lo:].float().cpu().numpy() - o_ref).max() <= 2e-2
    assert np.abs(res.lse[:, :, lo:].cpu().numpy() - l_ref).max() <= 2e-2
    # the launch is the tensor-core one-tile kernel, not a CUDA-core fallback
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fa.forward(q, k, v, fa.noop_score(), bm)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    assert any("flex_fwd1t_kernel" in n for n in names), names
    assert not any("simt" in n for n in names), names


@pytest.mark.parametrize("mname", ["noop", "hash:313:60"])
def test_two_tile_kernel_at_the_widest_rows(fa, O, dev, mname):
    """1024 kv blocks per row (KV_LEN 131072), the widest the two-tile kernel takes: every lane
    of the list builder's column bitmap is populated and the union lists hold 1024 entries."""
    Lq, Lkv = 256, 131072
    e_o, e_l, _ = run_case(fa, O, dev, mname, "noop", B=1, Hq=1, Hkv=1, Lq=Lq, Lkv=Lkv, D=64)
    assert e_o <= BF16_TOL and e_l <= BF16_TOL, (e_o, e_l)
    from torch.profiler import ProfilerActivity, profile
    fm, _ = mask_pair(mname, Lkv)
    q = fa.random_tensor(1, (1, 1, Lq, 64), device=dev)
    kv = fa.random_tensor(2, (1, 1, Lkv, 64), device=dev)
    bm = fa.create_block_mask(fm, 1, 1, Lq, Lkv, device=dev)
    assert bm.cols == 1024
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fa.forward(q, kv, kv, fa.noop_score(), bm)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    assert any("flex_fwd_sm100_kernel" in n for n in names), names
