"""CPU: the page allocator restatement (paging.PageAllocator + write_tokens) pinned to the
reference PagedKVCache (paged_kv.cpp:13-152, compiled in oracle/_ref) on random call scripts
with out-of-pages and out-of-range failures, and the host-side argument checks of the device
page pool (fa_page_pool_*) that run before any device work."""
import ctypes as C

import numpy as np
import pytest

from page_scripts import make_script, run_host


@pytest.mark.parametrize("seed", range(6))
def test_allocator_restatement_vs_reference(O, ref_lib, seed):
    B, P, ps, H, D = 5, 23, 4, 2, 8
    ops, tok = make_script(seed, B, P, ps, 120, H, D)
    want = O.ref_paged_script(B, P, ps, H, D, ops, tok)
    got = run_host(B, P, ps, H, D, ops, tok)
    names = ("status", "table", "p2l", "owner", "seq", "free", "k", "v")
    assert (want[0] == 9).any() and (want[0] == 3).any()  # the scripts do exercise the failures
    for n, w, g in zip(names, want, got):
        assert np.array_equal(np.asarray(w), np.asarray(g)), n


def test_page_pool_host_checks():
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    assert lib.fa_page_pool_bytes(0, 4) == 0
    assert lib.fa_page_pool_bytes(2, 4) > 0
    pool = _lib.PagePoolC()
    assert lib.fa_page_pool_init(C.byref(pool), C.c_void_p(0x1000), 1 << 20, 0, 4, 16, None) == 1
    assert b"must be >= 1" in lib.fa_last_error()
    assert lib.fa_page_pool_init(C.byref(pool), C.c_void_p(0x1000), 16, 2, 4, 16, None) == 1
    assert b"smaller than" in lib.fa_last_error()
    # update argument checks (no launch happens on failure)
    pool.batches, pool.num_pages, pool.page_size, pool.table = 2, 4, 16, 0x1000
    assert lib.fa_page_pool_update(C.byref(pool), 7, None, None, 0, None, None, None, None, 0, None) == 1
    assert lib.fa_page_pool_update(C.byref(pool), 1, None, None, 3, None, None, None, None, 0, None) == 1
    assert b"one request per sequence" in lib.fa_last_error()
    assert lib.fa_page_pool_update(C.byref(pool), 1, None, None, 1, None, None, None, None, 0, None) == 1
    assert b"batch_ids" in lib.fa_last_error()
    t = pool_table = lib.fa_page_pool_table(C.byref(pool))
    assert (t.batches, t.max_logical_pages, t.num_physical_pages, t.page_size) == (2, 4, 4, 16)
    assert pool_table.max_seq_len == 0
