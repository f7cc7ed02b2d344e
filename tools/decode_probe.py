"""Paged decode throughput beyond the C5 geometry: GQA (q heads sharing a kv head) and
multi-row steps (n_new > 1), reported as UNIQUE K/V bytes read per second (what the HBM must
deliver at least once per step)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2412_05496_b200 as fa  # noqa: E402
from perf_probe import timeit  # noqa: E402


def run(B, Hq, Hkv, L, n_new, D=128, ps=128):
    dev = torch.device("cuda:0")
    pages = B * (L // ps) + B
    cache = fa.PagedKVCache(B, pages, ps, Hkv, D, device=dev)
    cache.shuffle_free_pages(0x5EED0001 ^ 0xFA6E5)
    for b in range(B):
        kb = fa.random_tensor(100 + b, (1, Hkv, L, D), device=dev)
        cache.assign(b, kb, kb)
    q = fa.random_tensor(7, (B, Hq, n_new, D), device=dev)
    off = L - n_new
    lbm = fa.create_block_mask(fa.offset_mask(fa.causal(), off), 1, 1, n_new, L, device=dev)
    pt = cache.page_table()
    pbm = fa.convert_block_mask(lbm, pt)
    cfg = fa.AttentionConfig(gqa_group=Hq // Hkv)
    t = timeit(lambda: fa.decode(q, cache.k_phys(), cache.v_phys(), off, fa.causal(), fa.noop_score(), pbm,
                                 cfg=cfg, page_table=pt))
    gb = 2 * B * Hkv * L * D * 2 / 1e9
    print(f"decode B{B} Hq{Hq} Hkv{Hkv} L{L} n_new{n_new}: {t:.3f} ms  {gb / t:.3f} TB/s unique K/V "
          f"({gb / t / 6.5418 * 100:.1f}% of 6541.8 GB/s)", flush=True)
    del cache


if __name__ == "__main__":
    for (B, Hq, Hkv, L, n) in [(64, 32, 32, 32768, 1), (64, 32, 8, 32768, 1), (64, 32, 8, 32768, 4),
                               (64, 32, 32, 32768, 4), (64, 64, 8, 16384, 1), (16, 32, 8, 32768, 16)]:
        run(B, Hq, Hkv, L, n)
