"""Mask library beyond the BASELINE configs: or_mask, neighbourhood
attention (na_naive) and the remap_mask pixel orders (tile_permutation, morton_permutation).
CPU: the oracle restatement against the reference compiled from its sources and against the
reference's own block-count KATs (test_block_mask.cpp:267-309); the product-side permutation
tables against the reference's. GPU: builder bit-exact and forward/backward parity."""
import numpy as np
import pytest

import paper_2412_05496_b200 as fa
import pyoracle as O
from helpers import bm_arrays, mask_pair, rel_err

KEYS = ("partial_num", "partial_idx", "full_num", "full_idx")


def computed_blocks(bm):
    return int(bm.partial_num.sum() + bm.full_num.sum())


def na_mask(h, w, k, order=None, tile=None):
    m = O.na_naive(h, w, k)
    if order == "tile":
        m.remap = O.tile_permutation_np(h, w, tile)
    elif order == "morton":
        m.remap = O.morton_permutation_np(h)
    return m


# ---------------- reference KATs on the oracle (test_block_mask.cpp:267-309) ----------------
@pytest.mark.parametrize("order,tile,bs,want", [
    (None, None, 32, 154), ("tile", 2, 32, 184), ("tile", 4, 32, 220), ("tile", 8, 32, 220),
    ("tile", 16, 32, 184), ("morton", None, 32, 220),
    (None, None, 16, 616), ("tile", 2, 16, 460), ("morton", None, 16, 484),
])
def test_na_block_counts_32x32(order, tile, bs, want):
    n = 32 * 32
    bm = O.create_block_mask(na_mask(32, 32, 5, order, tile), 1, 1, n, n, bs, bs)
    assert computed_blocks(bm) == want


@pytest.mark.parametrize("order,tile,want", [(None, None, 10), ("tile", 4, 10), ("morton", None, 16)])
def test_na_block_counts_16x16(order, tile, want):
    bm = O.create_block_mask(na_mask(16, 16, 5, order, tile), 1, 1, 256, 256, 64, 64)
    assert computed_blocks(bm) == want


# ---------------- oracle restatement vs the reference itself ----------------
@pytest.mark.parametrize("name,bs", [
    ("na:24:20:3", 16), ("na:16:16:5:tile:4", 32), ("na:16:16:7:morton", 16),
    ("or_sliding_prefix:20:37", 16), ("or_causal_hash:77:40", 16),
])
def test_oracle_matches_reference_block_mask(ref_lib, name, bs):
    _, om = mask_pair(name)
    L = om.na_height * om.na_width if om.terms & O.MASK_NATTEN else 200
    got = O.create_block_mask(om, 1, 1, L, L, bs, bs)
    want, want_t = O.ref_create_block_mask(om, 1, 1, L, L, bs, bs)
    got_t = O.transpose(got)
    for k in KEYS:
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
        assert np.array_equal(getattr(got_t, k), getattr(want_t, k)), "t_" + k


def test_oracle_forward_matches_reference(ref_lib):
    _, om = mask_pair("na:12:12:5:tile:4")
    L, D = 144, 32
    q, k, v = (O.random_f32(s, (1, 2, L, D)) for s in (1, 2, 3))
    bm = O.create_block_mask(om, 1, 1, L, L, 16, 16)
    o, lse = O.forward(q, k, v, om, O.Score(), bm)
    o_r, lse_r = O.ref_forward(q, k, v, om, O.Score(), bs=16)
    assert np.array_equal(o, o_r) and np.array_equal(lse, lse_r)


# ---------------- product-side permutations and errors (host code, no GPU) ----------------
@pytest.mark.parametrize("h,w,k,tile", [(32, 32, 5, 2), (32, 32, 5, 8), (12, 18, 3, 6)])
def test_tile_permutation_matches_reference(ref_lib, h, w, k, tile):
    got = fa.tile_permutation(fa.NAGeometry(h, w, k), tile)
    assert np.array_equal(np.asarray(got), O.ref_tile_permutation(h, w, k, tile))
    assert np.array_equal(np.asarray(got), O.tile_permutation_np(h, w, tile))


@pytest.mark.parametrize("n", [4, 16, 32])
def test_morton_permutation_matches_reference(ref_lib, n):
    got = fa.morton_permutation(fa.NAGeometry(n, n, 3))
    assert np.array_equal(np.asarray(got), O.ref_morton_permutation(n, n, 3))
    assert np.array_equal(np.asarray(got), O.morton_permutation_np(n))


def test_geometry_and_permutation_errors():
    with pytest.raises(fa.GeometryMismatch):
        fa.NAGeometry(8, 8, 4)          # even kernel
    with pytest.raises(fa.GeometryMismatch):
        fa.NAGeometry(4, 8, 5)          # kernel exceeds canvas
    with pytest.raises(fa.GeometryMismatch):
        fa.tile_permutation(fa.NAGeometry(12, 12, 3), 5)
    with pytest.raises(fa.GeometryMismatch):
        fa.morton_permutation(fa.NAGeometry(12, 12, 3))
    with pytest.raises(fa.GeometryMismatch):
        fa.remap_mask(fa.causal(), [0, 0, 1])
    assert fa.or_mask(fa.noop_mask(), fa.causal()) == fa.noop_mask()


# ---------------- GPU: builder bit-exact, forward / backward parity ----------------
@pytest.mark.gpu
@pytest.mark.parametrize("name,bs", [
    ("na:32:32:5", 128), ("na:32:32:5:tile:4", 128), ("na:32:32:5:morton", 128),
    ("na:24:20:3", 16), ("na:16:16:7:morton", 64),
    ("or_sliding_prefix:100:300", 128), ("or_causal_hash:77:40", 64),
])
def test_gpu_block_mask(fa, O, dev, name, bs):
    fm, om = mask_pair(name)
    L = om.na_height * om.na_width if om.terms & O.MASK_NATTEN else 1000
    bm = fa.create_block_mask(fm, 1, 1, L, L, bs, bs, device=dev)
    got = bm_arrays(bm)
    want = O.create_block_mask(om, 1, 1, L, L, bs, bs)
    want_t = O.transpose(want)
    for k in KEYS:
        assert np.array_equal(got[k], getattr(want, k)), k
        assert np.array_equal(got["t_" + k], getattr(want_t, k)), "t_" + k


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["na:32:32:5:tile:4", "na:32:32:5:morton", "or_sliding_prefix:100:300"])
def test_gpu_forward_backward(fa, O, dev, name):
    import torch
    fm, om = mask_pair(name)
    L = om.na_height * om.na_width if om.terms & O.MASK_NATTEN else 1024
    B, H, D = 1, 2, 128
    q, k, v, do = (fa.random_tensor(s, (B, H, L, D), device=dev) for s in (31, 32, 33, 34))
    bm = fa.create_block_mask(fm, 1, 1, L, L, device=dev)
    res = fa.forward(q, k, v, fa.noop_score(), bm)
    g = fa.backward(q, k, v, res, do, fa.noop_score(), bm)
    torch.cuda.synchronize()
    qf, kf, vf, dof = (x.float().cpu().numpy() for x in (q, k, v, do))
    obm = O.create_block_mask(om, 1, 1, L, L)
    o_ref, lse_ref = O.forward(qf, kf, vf, om, O.Score(), obm)
    assert float(np.abs(res.out.float().cpu().numpy() - o_ref).max()) <= 2e-2
    dq, dk, dv = O.backward(qf, kf, vf, o_ref, lse_ref, dof, om, O.Score(), obm)
    for got, want in ((g.dq, dq), (g.dk, dk), (g.dv, dv)):
        assert rel_err(got.float().cpu().numpy(), want) <= 2e-2
