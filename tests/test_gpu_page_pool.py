"""GPU: the device page pool (fa_page_pool_*) against the reference PagedKVCache
(paged_kv.cpp:13-152) on random call scripts — one call at a time and as batched updates that
stop at the first failing request — bit for bit in the page table, phys->logical map, owners,
sequence lengths, free page count and the physical K/V written by the fused token scatter;
then a decode serving loop (append one token per sequence on the device, convert, decode)
against the unpaged decode."""
import numpy as np
import pytest
import torch

from page_scripts import APPEND, ASSIGN, ERASE, SHUFFLE, make_script, run_host

pytestmark = pytest.mark.gpu

_CODES = None


def _code(fa, e):
    global _CODES
    if _CODES is None:
        _CODES = {fa.OutOfPages: 9, fa.IndexOutOfRange: 3, fa.ShapeMismatch: 1}
    return _CODES.get(type(e), 99)


def _want(O, B, P, ps, H, D, ops, tok):
    if O.ref_available():
        return O.ref_paged_script(B, P, ps, H, D, ops, tok)
    return run_host(B, P, ps, H, D, ops, tok)


def _state(cache):
    pt = cache.page_table()
    B, P = cache.batches, cache.num_pages
    return (np.array(pt.table, np.int32).reshape(B, P), np.array(pt.phys_to_logical, np.int32),
            np.array(pt.owner, np.int32), np.array(pt.seq_len, np.int64), cache.free_pages(),
            cache.k.float().cpu().numpy(), cache.v.float().cpu().numpy())


def _tokens(tok, base, n, H, D, dev):
    t = torch.from_numpy(tok[base:base + n * H * D].reshape(1, H, n, D)).to(dev, torch.bfloat16)
    return t, -t


@pytest.mark.parametrize("seed", range(4))
def test_single_calls_vs_reference(fa, O, dev, seed):
    B, P, ps, H, D = 5, 23, 4, 2, 8
    ops, tok = make_script(seed, B, P, ps, 120, H, D)
    want = _want(O, B, P, ps, H, D, ops, tok)
    cache = fa.PagedKVCache(B, P, ps, H, D, device=dev)
    status, base = [], 0
    for kind, b, n, sd in ops:
        st = 0
        try:
            if kind == SHUFFLE:
                cache.shuffle_free_pages(sd)
            elif kind == ERASE:
                cache.erase(b)
            else:
                kt, vt = _tokens(tok, base, n, H, D, dev)
                base += n * H * D
                (cache.assign if kind == ASSIGN else cache.append_tokens)(b, kt, vt)
        except fa.Error as e:
            st = _code(fa, e)
        status.append(st)
    assert np.array_equal(np.array(status, np.int32), want[0])
    for name, w, g in zip(("table", "p2l", "owner", "seq", "free", "k", "v"), want[1:], _state(cache)):
        assert np.array_equal(np.asarray(w), np.asarray(g)), name


@pytest.mark.parametrize("seed", range(4))
def test_batched_updates_vs_reference(fa, O, dev, seed):
    """Runs of same-kind calls on distinct sequences go in one launch; a failure at request f
    leaves requests < f applied, and the script resumes at f + 1 (the reference's caught
    exception)."""
    B, P, ps, H, D = 7, 40, 4, 2, 8
    ops, tok = make_script(100 + seed, B, P, ps, 160, H, D)
    want = _want(O, B, P, ps, H, D, ops, tok)
    offs, base = [], 0
    for kind, b, n, _ in ops:
        offs.append(base)
        if kind in (ASSIGN, APPEND):
            base += n * H * D
    cache = fa.PagedKVCache(B, P, ps, H, D, device=dev)
    status = [0] * len(ops)
    i = 0
    while i < len(ops):
        kind = ops[i][0]
        if kind == SHUFFLE:
            cache.shuffle_free_pages(ops[i][3])
            i += 1
            continue
        j, seen = i, set()
        while j < len(ops) and ops[j][0] == kind and ops[j][1] not in seen and j - i < B:
            seen.add(ops[j][1])
            j += 1
        run = ops[i:j]
        ids = [o[1] for o in run]
        try:
            if kind == ERASE:
                cache.erase_batch(ids)
            else:
                ns = [o[2] for o in run]
                kt = torch.cat([_tokens(tok, offs[i + r], run[r][2], H, D, dev)[0] for r in range(len(run))], 2)
                fn = cache.assign_batch if kind == ASSIGN else cache.append_batch
                fn(ids, ns, kt, -kt)
            i = j
        except fa.Error as e:
            # the pool reports how many requests were applied before the failure
            applied = _applied(cache)
            status[i + applied] = _code(fa, e)
            i += applied + 1
    assert np.array_equal(np.array(status, np.int32), want[0])
    for name, w, g in zip(("table", "p2l", "owner", "seq", "free", "k", "v"), want[1:], _state(cache)):
        assert np.array_equal(np.asarray(w), np.asarray(g)), name


def _applied(cache):
    import ctypes as C
    from paper_2412_05496_b200 import _lib
    a = C.c_int32(0)
    _lib.load().fa_page_pool_status(C.byref(cache._pool), C.byref(a), None)
    return a.value


def test_duplicate_batch_in_one_update(fa, dev):
    cache = fa.PagedKVCache(4, 8, 16, 1, 8, device=dev)
    with pytest.raises(fa.ShapeMismatch, match="twice"):
        cache.append_batch([0, 1, 0], [3, 3, 3])
    assert [cache.seq_len(b) for b in range(4)] == [3, 3, 0, 0]  # requests before the repeat applied
    with pytest.raises(fa.ShapeMismatch, match="tokens"):
        cache.append_batch([2], [5], torch.zeros(1, 1, 4, 8, device=dev), torch.zeros(1, 1, 4, 8, device=dev))
    assert cache.seq_len(2) == 0


def test_serving_loop_append_convert_decode(fa, dev):
    """Each step appends one token per sequence with one device-side batched update (no host
    sync), converts the logical BlockMask through the live page table and decodes; the paged
    result equals the unpaged decode over the logical cache bit for bit."""
    B, H, D, ps, L0, steps = 6, 4, 128, 128, 250, 12
    P = B * 4
    cache = fa.PagedKVCache(B, P, ps, H, D, device=dev)
    cache.shuffle_free_pages(0xFA6E5)
    kl = fa.random_tensor(51, (B, H, L0 + steps, D), device=dev)
    vl = fa.random_tensor(52, (B, H, L0 + steps, D), device=dev)
    cache.assign_batch(list(range(B)), [L0] * B, torch.cat([kl[b:b + 1, :, :L0] for b in range(B)], 2),
                       torch.cat([vl[b:b + 1, :, :L0] for b in range(B)], 2))
    ids = torch.arange(B, dtype=torch.int32, device=dev)
    ones = torch.ones(B, dtype=torch.int32, device=dev)
    for s in range(steps):
        L = L0 + s + 1
        kn = torch.cat([kl[b:b + 1, :, L - 1:L] for b in range(B)], 2)
        vn = torch.cat([vl[b:b + 1, :, L - 1:L] for b in range(B)], 2)
        cache.append_batch(ids, ones, kn, vn, sync=False)
        q = fa.random_tensor(60 + s, (B, H, 1, D), device=dev)
        off = L - 1
        lbm = fa.create_block_mask(fa.offset_mask(fa.causal(), off), 1, 1, 1, L, device=dev)
        pbm = fa.convert_block_mask(lbm, cache.page_table())
        paged = fa.decode(q, cache.k_phys(), cache.v_phys(), off, fa.causal(), fa.noop_score(), pbm,
                          page_table=cache.page_table())
        ubm = fa.create_block_mask(fa.offset_mask(fa.causal(), off), 1, 1, 1, L, device=dev)
        unpaged = fa.decode(q, kl[:, :, :L].contiguous(), vl[:, :, :L].contiguous(), off, fa.causal(),
                            fa.noop_score(), ubm)
        torch.cuda.synchronize()
        assert torch.equal(paged.out, unpaged.out) and torch.equal(paged.lse, unpaged.lse), s
    assert cache.status() == B
    assert [cache.seq_len(b) for b in range(B)] == [L0 + steps] * B
