"""Fixture I/O and block-grid test aids against the reference built from
its sources: BlockMask and Tensor4 files byte-identical in both directions, PPM rendering,
corrupted-file negative controls (test_bench.cpp:248-271), and on the GPU the metamorphic
checks the reference runs with demote_full_to_partial / promote_empty_to_partial
(acceptance.cpp:280-309, test_engine.cpp:103-122)."""

import numpy as np
import pytest

import paper_2412_05496_b200 as fa
import pyoracle as O
from helpers import bm_arrays, mask_pair


def oracle_grid(om, ql, kl, bs):
    bm = O.create_block_mask(om, 1, 1, ql, kl, bs, bs)
    g = np.zeros((1, 1, bm.rows, bm.cols), np.int8)
    pi, fi = bm.partial_idx.reshape(bm.rows, bm.cols), bm.full_idx.reshape(bm.rows, bm.cols)
    for r in range(bm.rows):
        g[0, 0, r, pi[r, :bm.partial_num.reshape(-1)[r]]] = fa.KIND_PARTIAL
        g[0, 0, r, fi[r, :bm.full_num.reshape(-1)[r]]] = fa.KIND_FULL
    return g


def test_tensor_files_match_reference(ref_lib, tmp_path):
    import torch
    x = O.random_f32(5, (2, 3, 7, 16))
    ours, theirs = str(tmp_path / "ours.bin"), str(tmp_path / "ref.bin")
    fa.save_tensor(ours, torch.from_numpy(x))
    O.ref_save_tensor_f32(x, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(O.ref_load_tensor_f32(ours, x.shape), x)
    assert np.array_equal(fa.load_tensor(theirs).numpy(), x)
    with pytest.raises(fa.Error):
        fa.load_tensor(theirs, dtype=torch.float64)  # precision tag mismatch
    open(str(tmp_path / "trunc.bin"), "wb").write(open(theirs, "rb").read()[:-4])
    with pytest.raises(fa.Error):
        fa.load_tensor(str(tmp_path / "trunc.bin"))


@pytest.mark.parametrize("name,ql,kl,bs", [("causal", 1024, 1024, 128), ("hash:77:90", 200, 130, 16),
                                            ("na:16:16:5:morton", 256, 256, 32)])
def test_block_mask_files_match_reference(ref_lib, tmp_path, name, ql, kl, bs):
    _, om = mask_pair(name)
    theirs, ours = str(tmp_path / "ref.bm"), str(tmp_path / "ours.bm")
    O.ref_save_block_mask(om, 1, 1, ql, kl, bs, bs, theirs)
    bm = fa.load_block_mask(theirs, device="cpu")
    want = O.create_block_mask(om, 1, 1, ql, kl, bs, bs)
    for k in ("partial_num", "partial_idx", "full_num", "full_idx"):
        assert np.array_equal(getattr(bm, k).numpy().astype(np.int64), getattr(want, k)), k
    fa.save_block_mask(ours, bm)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    # grid round trip on the host
    g = oracle_grid(om, ql, kl, bs)
    assert np.array_equal(fa.to_dense(bm), g)
    bm2 = fa.block_mask_from_grid(g, bs, bs, ql, kl, device="cpu")
    fa.save_block_mask(ours, bm2)
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_corrupted_block_mask_files(ref_lib, tmp_path):
    _, om = mask_pair("causal")
    path = str(tmp_path / "c.bm")
    O.ref_save_block_mask(om, 1, 1, 256, 256, 64, 64, path)
    data = bytearray(open(path, "rb").read())
    bad = bytearray(data)
    bad[16:24] = (5).to_bytes(8, "little")  # rows no longer match q_len / bs_q
    open(str(tmp_path / "bad.bm"), "wb").write(bytes(bad))
    with pytest.raises(fa.Error):
        fa.load_block_mask(str(tmp_path / "bad.bm"), device="cpu")
    with pytest.raises(O.OracleError):
        O.ref_load_block_mask(str(tmp_path / "bad.bm"))
    open(str(tmp_path / "short.bm"), "wb").write(bytes(data[:100]))
    with pytest.raises(fa.Error):
        fa.load_block_mask(str(tmp_path / "short.bm"), device="cpu")


def test_render_matches_reference(ref_lib, tmp_path):
    _, om = mask_pair("causal")
    theirs = str(tmp_path / "ref.ppm")
    O.ref_write_ppm(om, 256, 256, 64, theirs)
    bm = fa.block_mask_from_grid(oracle_grid(om, 256, 256, 64), 64, 64, 256, 256, device="cpu")
    assert fa.render_ppm(bm) == open(theirs, "rb").read()
    txt = fa.render_ascii(bm)
    assert txt.count("\n") == 4 and txt.splitlines()[0] == "▒□□□" and txt.splitlines()[3] == "███▒"
    with pytest.raises(fa.IndexOutOfRange):
        fa.render_ascii(bm, 1, 0)


@pytest.mark.gpu
def test_gpu_block_mask_file_and_transpose(fa, O, dev, tmp_path):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    fm, om = mask_pair("sliding:300")
    bm = fa.create_block_mask(fm, 1, 1, 2000, 2000, 64, 64, device=dev)
    ours, theirs = str(tmp_path / "g.bm"), str(tmp_path / "r.bm")
    fa.save_block_mask(ours, bm)
    O.ref_save_block_mask(om, 1, 1, 2000, 2000, 64, 64, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    back = fa.load_block_mask(theirs, device=dev, mask=fm)
    a, b = bm_arrays(back), bm_arrays(bm)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["causal", "sliding:300", "doc_causal"])
def test_gpu_demote_and_promote_are_exact(fa, O, dev, name):
    import torch
    fm, _ = mask_pair(name, 1024)
    B, H, L, D = 1, 2, 1024, 128
    q, k, v, do = (fa.random_tensor(s, (B, H, L, D), device=dev) for s in (41, 42, 43, 44))
    bm = fa.create_block_mask(fm, 1, 1, L, L, device=dev)
    base = fa.forward(q, k, v, fa.noop_score(), bm)
    g0 = fa.backward(q, k, v, base, do, fa.noop_score(), bm)
    for aid in (fa.demote_full_to_partial, fa.promote_empty_to_partial):
        bm2 = aid(bm)
        assert fa.sparsity(bm2).total_blocks == fa.sparsity(bm).total_blocks
        res = fa.forward(q, k, v, fa.noop_score(), bm2)
        torch.cuda.synchronize()
        assert torch.equal(res.out, base.out) and torch.equal(res.lse, base.lse), aid.__name__
        g = fa.backward(q, k, v, res, do, fa.noop_score(), bm2)
        for x, y in ((g.dq, g0.dq), (g.dk, g0.dk), (g.dv, g0.dv)):
            assert float((x.float() - y.float()).abs().max()) <= 1e-2, aid.__name__
