"""Random PagedKVCache call scripts (assign / append_tokens / erase / shuffle_free_pages) and a
host restatement of their effect (paging.PageAllocator + numpy K/V, write_tokens
paged_kv.cpp:54-70), shared by the CPU pin against the reference (tests/test_page_pool.py) and
the GPU device-pool parity test (tests/test_gpu_page_pool.py)."""
from __future__ import annotations

import numpy as np

from paper_2412_05496_b200.paging import OutOfPagesError, PageAllocator

ASSIGN, APPEND, ERASE, SHUFFLE = 0, 1, 2, 3


def make_script(seed, B, num_pages, page_size, n_ops, heads, dim, bad_batch=True):
    """ops = [(kind, b, n, seed)] and the packed token values (small integers, exact in bf16)."""
    rng = np.random.default_rng(seed)
    ops, ntok = [], 0
    for _ in range(n_ops):
        r = rng.random()
        if r < 0.05:
            ops.append((SHUFFLE, 0, 0, int(rng.integers(1, 2**63))))
            continue
        b = int(rng.integers(0, B))
        if bad_batch and rng.random() < 0.03:
            b = B + int(rng.integers(0, 3))  # IndexOutOfRange
        if r < 0.35:
            n = int(rng.integers(1, 3 * page_size * num_pages // B + 2))
            ops.append((ASSIGN, b, n, 0))
        elif r < 0.85:
            n = int(rng.integers(1, 2 * page_size + 2))
            ops.append((APPEND, b, n, 0))
        else:
            ops.append((ERASE, b, 0, 0))
            continue
        if 0 <= b < B:
            ntok += n * heads * dim
        else:
            ntok += n * heads * dim  # the reference builds the tensors before check_batch
    tok = rng.integers(-100, 101, size=ntok).astype(np.float32)
    return ops, tok


def run_host(B, num_pages, page_size, heads, dim, ops, tok):
    """Sequential restatement: per-op status, final page table state and physical K/V."""
    pa = PageAllocator(B, num_pages, page_size)
    kp = np.zeros((1, heads, num_pages * page_size, dim), np.float32)
    vp = np.zeros_like(kp)
    status, base = [], 0
    for kind, b, n, sd in ops:
        st = 0
        if kind == SHUFFLE:
            pa.shuffle_free_pages(sd)
        elif kind == ERASE:
            if 0 <= b < B:
                pa.erase(b)
            else:
                st = 3
        else:
            t = tok[base:base + n * heads * dim].reshape(heads, n, dim)
            base += n * heads * dim
            if not 0 <= b < B:
                st = 3
            else:
                start = 0 if kind == ASSIGN else pa.seq[b]
                try:
                    (pa.assign if kind == ASSIGN else pa.append)(b, n)
                except OutOfPagesError:
                    st = 9
                if st == 0:
                    for i in range(n):
                        pos = start + i
                        phys = pa.lookup(b, pos // page_size) * page_size + pos % page_size
                        kp[0, :, phys] = t[:, i]
                        vp[0, :, phys] = -t[:, i]
        status.append(st)
    table = np.array(pa.table, np.int32).reshape(B, num_pages)
    return (np.array(status, np.int32), table, np.array(pa.phys_to_logical, np.int32),
            np.array(pa.owner, np.int32), np.array(pa.seq, np.int64), len(pa.free), kp, vp)
