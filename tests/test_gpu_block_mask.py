"""BlockMask builder on the GPU vs the oracle: all arrays bit-exact (int32 widened to i64,
zero tails included). Cases: the five BASELINE configs, the reference's own
structural KATs (test_block_mask.cpp) and brute-force soundness shapes (acceptance.cpp:168-243)."""
import numpy as np
import pytest

from helpers import bm_arrays, mask_pair

pytestmark = pytest.mark.gpu

KEYS = ("partial_num", "partial_idx", "full_num", "full_idx")


def check_exact(fa, O, dev, name, bd, hd, ql, kl, bsq, bskv, offset=0):
    fm, om = mask_pair(name, max(ql, kl))
    if offset:
        fm, om = fa.offset_mask(fm, offset), O.Mask(**{**om.__dict__, "q_offset": offset})
    bm = fa.create_block_mask(fm, bd, hd, ql, kl, bsq, bskv, device=dev)
    got = bm_arrays(bm)
    want = O.create_block_mask(om, bd, hd, ql, kl, bsq, bskv)
    want_t = O.transpose(want)
    for k in KEYS:
        assert np.array_equal(got[k], getattr(want, k)), (name, k)
        assert np.array_equal(got["t_" + k], getattr(want_t, k)), (name, "t_" + k)
    return got


@pytest.mark.parametrize("name,ql,kl", [
    ("causal", 1024, 1024),          # C1
    ("sliding:1024", 8192, 8192),    # C2
    ("doc_causal", 16384, 16384),    # C3
    ("causal", 8192, 8192),          # C4
])
def test_config_masks(fa, O, dev, name, ql, kl):
    check_exact(fa, O, dev, name, 1, 1, ql, kl, 128, 128)


def test_c5_decode_mask(fa, O, dev):
    # offset_mask(causal(), 32767) at Q_LEN=1: every tile ragged -> all 256 PARTIAL
    got = check_exact(fa, O, dev, "causal", 1, 1, 1, 32768, 128, 128, offset=32767)
    assert got["partial_num"].tolist() == [256] and got["full_num"].tolist() == [0]


def test_causal_counts(fa, dev):
    # test_block_mask.cpp:82-92 — causal 1024/128: 28 full + 8 partial of 64
    bm = fa.create_block_mask(fa.causal(), 1, 1, 1024, 1024, 128, 128, device=dev)
    rep = fa.sparsity(bm)
    assert (rep.total_blocks, rep.full_blocks, rep.partial_blocks) == (64, 28, 8)
    assert rep.density == pytest.approx(36 / 64)
    bm = fa.create_block_mask(fa.causal(), 1, 1, 4096, 4096, 64, 64, device=dev)
    assert fa.sparsity(bm).density == pytest.approx(2080 / 4096)


def test_causal_structure_256(fa, dev):
    # test_block_mask.cpp:40-60
    a = bm_arrays(fa.create_block_mask(fa.causal(), 1, 1, 256, 256, 64, 64, device=dev))
    for r in range(4):
        assert a["full_num"][r] == r and a["partial_num"][r] == 1
        assert a["partial_idx"][r * 4] == r
        assert list(a["full_idx"][r * 4:r * 4 + r]) == list(range(r))


def test_ragged_never_full(fa, dev):
    # test_block_mask.cpp:62-80 — kv = 200 overhangs the last of 4 blocks
    a = bm_arrays(fa.create_block_mask(fa.noop_mask(), 1, 1, 256, 200, 64, 64, device=dev))
    for r in range(4):
        assert a["full_num"][r] == 3 and a["partial_num"][r] == 1 and a["partial_idx"][r * 4] == 3


@pytest.mark.parametrize("case", [
    ("hash:1234:96", 2, 2, 100, 75, 16, 16),   # test_block_mask.cpp:156-170
    ("hash:77:128", 2, 3, 100, 75, 16, 16),    # transpose involution case :112
    ("hash:5:128", 2, 2, 90, 130, 32, 32),     # dense grid round trip :120
    ("causal", 1, 1, 200, 200, 64, 64),        # acceptance.cpp:207-211 ragged 200
    ("sliding:5", 1, 1, 60, 60, 16, 16),
    ("prefix:7", 1, 1, 60, 32, 16, 16),
    ("doc", 1, 1, 64, 64, 16, 16),
    ("never", 1, 1, 8, 8, 4, 4),
    ("noop", 1, 1, 1, 1, 16, 16),
    ("hash:909:128", 2, 4, 60, 60, 64, 64),
    ("causal", 1, 1, 1000, 777, 128, 128),
])
def test_exhaustive_small(fa, O, dev, case):
    check_exact(fa, O, dev, *case)


def test_matches_reference_library(fa, O, dev):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    fm, om = mask_pair("hash:4242:64")
    bm = bm_arrays(fa.create_block_mask(fm, 2, 2, 300, 250, 32, 32, device=dev))
    rbm, rbt = O.ref_create_block_mask(om, 2, 2, 300, 250, 32, 32)
    for k in KEYS:
        assert np.array_equal(bm[k], getattr(rbm, k))
        assert np.array_equal(bm["t_" + k], getattr(rbt, k))


def test_transpose_from_kv_side(fa, O, dev):
    fm, om = mask_pair("hash:31:100")
    bm = fa.create_block_mask(fm, 2, 3, 100, 75, 16, 16, device=dev, q_side=False)
    t = fa.transpose(bm)
    want = O.transpose(O.create_block_mask(om, 2, 3, 100, 75, 16, 16))
    assert np.array_equal(t.kv_indices.cpu().numpy(), want.partial_idx)
    assert np.array_equal(t.full_kv_indices.cpu().numpy(), want.full_idx)
    assert np.array_equal(t.kv_num_blocks.cpu().numpy(), want.partial_num)
