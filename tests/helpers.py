"""Shared test helpers: matched (GPU API, oracle) modifier pairs and comparisons."""
from __future__ import annotations

import numpy as np

import paper_2412_05496_b200 as fa
import pyoracle as O

# BASELINE.json configs C1-C5: doc lengths of C3 pinned literally
C3_DOC_LENGTHS = [1004, 350, 639, 2533, 190, 1601, 7058, 3009]


def c3_doc_ids():
    ids = np.concatenate([np.full(n, i, dtype=np.int64) for i, n in enumerate(C3_DOC_LENGTHS)])
    assert len(ids) == 16384
    return ids


def mask_pair(name: str, L: int = 0, offset: int = 0):
    """(fa.MaskMod, O.Mask) for a named variant."""
    if name == "noop":
        return fa.noop_mask(), O.Mask()
    if name == "causal":
        return fa.causal(), O.Mask(terms=O.MASK_CAUSAL)
    if name.startswith("sliding"):
        w = int(name.split(":")[1]) if ":" in name else 1024
        return fa.sliding_window(w), O.Mask(terms=O.MASK_SLIDING, window=w)
    if name.startswith("doc"):
        ids = c3_doc_ids() if L == 16384 else O.make_doc_ids(L, 4, 0x5EED ^ 0xD0C5)
        causal = name.endswith("causal")
        m = fa.document_mask(ids)
        if causal:
            m = fa.and_mask(m, fa.causal())
        return m, O.Mask(terms=O.MASK_DOCUMENT | (O.MASK_CAUSAL if causal else 0), doc_ids=ids)
    if name.startswith("prefix"):
        p = int(name.split(":")[1]) if ":" in name else max(1, L // 4)
        return fa.prefix_lm(p), O.Mask(terms=O.MASK_PREFIX, prefix=p)
    if name.startswith("hash"):
        seed = int(name.split(":")[1]) if ":" in name else 909
        dens = int(name.split(":")[2]) if name.count(":") > 1 else 128
        return fa.hash_mask(seed, dens), O.Mask(terms=O.MASK_HASH, hash_seed=seed, hash_density=dens)
    if name == "never":
        return fa.never_mask(), O.Mask(terms=O.MASK_NEVER)
    if name.startswith("na"):
        # na:H:W:K[:tile:T | :morton] — neighbourhood attention on an H x W canvas (L = H*W)
        parts = name.split(":")
        h, w, k = int(parts[1]), int(parts[2]), int(parts[3])
        g = fa.NAGeometry(h, w, k)
        fm, om = fa.na_naive(g), O.na_naive(h, w, k)
        if len(parts) > 4:
            perm = fa.tile_permutation(g, int(parts[5])) if parts[4] == "tile" else fa.morton_permutation(g)
            fm = fa.remap_mask(fm, perm)
            om = O.Mask(**{**om.__dict__, "remap": np.asarray(perm, dtype=np.int64)})
        return fm, om
    if name.startswith("or_"):
        # or_sliding_prefix:W:P  /  or_causal_hash:S:D
        parts = name.split(":")
        if parts[0] == "or_sliding_prefix":
            w, p = int(parts[1]), int(parts[2])
            return (fa.or_mask(fa.sliding_window(w), fa.prefix_lm(p)),
                    O.Mask(terms=O.MASK_SLIDING, or_terms=O.MASK_PREFIX, window=w, prefix=p))
        if parts[0] == "or_causal_hash":
            seed, dens = int(parts[1]), int(parts[2])
            return (fa.or_mask(fa.causal(), fa.hash_mask(seed, dens)),
                    O.Mask(terms=O.MASK_CAUSAL, or_terms=O.MASK_HASH, hash_seed=seed, hash_density=dens))
    raise KeyError(name)


def score_pair(name: str, H: int = 1):
    if name == "noop":
        return fa.noop_score(), O.Score()
    if name == "alibi":
        sl = fa.alibi_slopes(H)
        return fa.alibi(sl), O.Score(terms=O.SCORE_ALIBI, slopes=np.array(sl))
    if name.startswith("softcap"):
        cap = float(name.split(":")[1]) if ":" in name else 20.0
        return fa.soft_cap(cap), O.Score(terms=O.SCORE_SOFTCAP, cap=cap)
    if name.startswith("stacked"):
        cap = float(name.split(":")[1]) if ":" in name else 5.0
        sl = fa.alibi_slopes(H)
        return (fa.compose(fa.soft_cap(cap), fa.alibi(sl)),
                O.Score(terms=O.SCORE_ALIBI | O.SCORE_SOFTCAP, cap=cap, slopes=np.array(sl)))
    raise KeyError(name)


def bm_arrays(bm):
    """kv-side and q-side arrays of a device BlockMask, widened to int64 numpy."""
    g = lambda t: t.cpu().numpy().astype(np.int64)  # noqa: E731
    out = dict(partial_num=g(bm.kv_num_blocks), partial_idx=g(bm.kv_indices),
               full_num=g(bm.full_kv_num_blocks), full_idx=g(bm.full_kv_indices))
    if bm.q_num_blocks is not None:
        out.update(t_partial_num=g(bm.q_num_blocks), t_partial_idx=g(bm.q_indices),
                   t_full_num=g(bm.full_q_num_blocks), t_full_idx=g(bm.full_q_indices))
    return out


def rel_err(got, want):
    """The reference's rel_grad_err form (bench.cpp:398-403)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.abs(got - want).max()) / max(1.0, float(np.abs(want).max()))


def lse_err(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    ninf_g, ninf_w = np.isneginf(got), np.isneginf(want)
    assert np.array_equal(ninf_g, ninf_w), "-inf rows differ"
    fin = ~ninf_w
    return float(np.abs(got[fin] - want[fin]).max()) if fin.any() else 0.0
