"""Generate tests/golden/*.npz from the UNMODIFIED reference library (oracle/_ref, built from
/root/reference sources by `make -C oracle ref`). Run here (the reference is not on the GPU
box); the fixtures are committed so the oracle stays pinned where the reference is absent.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as O  # noqa: E402


def masks():
    sl = O.alibi_slopes(4)
    return {
        "causal": (O.causal(), O.Score()),
        "sliding5_alibi": (O.sliding_window(5), O.Score(terms=O.SCORE_ALIBI, slopes=sl)),
        "prefix7_softcap10": (O.Mask(terms=O.MASK_PREFIX, prefix=7), O.Score(terms=O.SCORE_SOFTCAP, cap=10.0)),
        "doc_stacked": (O.Mask(terms=O.MASK_DOCUMENT, doc_ids=O.make_doc_ids(64, 4, 0x5EED ^ 0xD0C5)),
                        O.Score(terms=3, cap=5.0, slopes=sl)),
        "hash909": (O.Mask(terms=O.MASK_HASH, hash_seed=909, hash_density=128), O.Score()),
    }


def main():
    out = {}
    # BlockMask fixtures (reference create_block_mask + transpose, all arrays incl. visit lists)
    bm_cases = {
        "bm_causal_1024_128": (O.causal(), 1, 1, 1024, 1024, 128, 128),
        "bm_sliding1024_8192": (O.sliding_window(1024), 1, 1, 8192, 8192, 128, 128),
        "bm_hash1234_2x2_100x75": (O.Mask(terms=O.MASK_HASH, hash_seed=1234, hash_density=96), 2, 2, 100, 75, 16, 16),
        "bm_causal_ragged200": (O.causal(), 1, 1, 200, 200, 64, 64),
        "bm_decode_c5": (O.causal(32767), 1, 1, 1, 32768, 128, 128),
    }
    for name, (m, bd, hd, ql, kl, bq, bk) in bm_cases.items():
        bm, bt = O.ref_create_block_mask(m, bd, hd, ql, kl, bq, bk)
        for k in ("partial_num", "partial_idx", "full_num", "full_idx"):
            out[f"{name}/{k}"] = getattr(bm, k)
            out[f"{name}/t_{k}"] = getattr(bt, k)
        for k, v in bm.extra.items():
            out[f"{name}/{k}"] = v
        out[f"{name}/geom"] = np.array([bd, hd, ql, kl, bq, bk], np.int64)
    # forward/backward fixtures (reference forward<float>/backward<float>) on small shapes
    B, H, L, D = 2, 4, 60, 8
    q = O.random_f32(101, (B, H, L, D))
    k = O.random_f32(102, (B, H, L, D))
    v = O.random_f32(103, (B, H, L, D))
    do = O.random_f32(104, (B, H, L, D))
    for name, (m, s) in masks().items():
        md = (B, H) if name.startswith("hash") else (1, 1)
        o, lse, dq, dk, dv = O.ref_backward(q, k, v, do, m, s, mask_dims=md, bs=16)
        out[f"attn_{name}/out"], out[f"attn_{name}/lse"] = o, lse
        out[f"attn_{name}/dq"], out[f"attn_{name}/dk"], out[f"attn_{name}/dv"] = dq, dk, dv
    out["attn_inputs/q"], out["attn_inputs/k"], out["attn_inputs/v"], out["attn_inputs/do"] = q, k, v, do
    # decode fixture: one step at offset 59 over the same k/v (engine.cpp:403-427)
    o_d, l_d = O.ref_decode(q[:, :, 59:60], k, v, 59, O.causal(), O.Score(), bs=16)
    out["decode/out"], out["decode/lse"] = o_d, l_d
    # paged layout fixture (PagedKVCache LIFO + deterministic_shuffle + assign)
    t, p2l, own = O.ref_paged_layout(4, 4 * 8 + 4, 128, 0x1234, 1000)
    out["paged/table"], out["paged/p2l"], out["paged/owner"] = t, p2l, own
    np.savez_compressed(os.path.join(HERE, "reference_fixtures.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
