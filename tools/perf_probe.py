"""Quick device-timed probe of every hot-path kernel at the BASELINE configs (not the bench
contract; bench.py is). Usage: python tools/perf_probe.py [fwd|bwd|decode|mask ...]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2412_05496_b200 as fa  # noqa: E402

DOCS = [1004, 350, 639, 2533, 190, 1601, 7058, 3009]
PEAK = 1649.8


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def configs(dev):
    ids = torch.tensor(np.concatenate([np.full(n, i) for i, n in enumerate(DOCS)]), dtype=torch.int32)
    return {
        "C2": dict(B=4, Hq=16, Hkv=16, L=8192, mask=fa.sliding_window(1024), score=fa.alibi(fa.alibi_slopes(16)),
                   gf=257.95),
        "C3": dict(B=1, Hq=32, Hkv=32, L=16384, mask=fa.and_mask(fa.document_mask(ids), fa.causal()),
                   score=fa.noop_score(), gf=568.85),
        "C4": dict(B=2, Hq=32, Hkv=8, L=8192, mask=fa.causal(), score=fa.soft_cap(50.0), gf=1099.65),
    }


def main(which):
    dev = torch.device("cuda:0")
    only = [w.split("_only_")[1] for w in which if "_only_" in w]
    if only:
        which = which + ["fwd"]
    for name, c in configs(dev).items():
        if only and name not in only:
            continue
        D = 128
        q = fa.random_tensor(1, (c["B"], c["Hq"], c["L"], D), device=dev)
        k = fa.random_tensor(2, (c["B"], c["Hkv"], c["L"], D), device=dev)
        v = fa.random_tensor(3, (c["B"], c["Hkv"], c["L"], D), device=dev)
        t_mask = timeit(lambda: fa.create_block_mask(c["mask"], 1, 1, c["L"], c["L"], device=dev))
        bm = fa.create_block_mask(c["mask"], 1, 1, c["L"], c["L"], device=dev)
        cfg = fa.AttentionConfig(gqa_group=c["Hq"] // c["Hkv"])
        if "fwd" in which:
            t = timeit(lambda: fa.forward(q, k, v, c["score"], bm, cfg))
            print(f"{name} fwd {t:.3f} ms  {c['gf'] / t:.1f} TFLOPS  ({c['gf'] / t / PEAK * 100:.1f}% of {PEAK})"
                  f"  mask build {t_mask * 1000:.1f} us", flush=True)
        if "bwd" in which:
            do = fa.random_tensor(4, q.shape, device=dev)
            res = fa.forward(q, k, v, c["score"], bm, cfg)
            t = timeit(lambda: fa.backward(q, k, v, res, do, c["score"], bm, cfg=cfg), iters=3, warm=1)
            print(f"{name} bwd {t:.3f} ms  {2.5 * c['gf'] / t:.1f} TFLOPS", flush=True)
        del q, k, v
    if "decode" in which:
        B, H, L, D, ps = 64, 32, 32768, 128, 128
        pages = B * (L // ps) + B
        cache = fa.PagedKVCache(B, pages, ps, H, D, device=dev)
        cache.shuffle_free_pages(0x5EED0001 ^ 0xFA6E5)
        for b in range(B):
            kb = fa.random_tensor(100 + b, (1, H, L, D), device=dev)
            cache.assign(b, kb, kb)
            del kb
        q = fa.random_tensor(7, (B, H, 1, D), device=dev)
        lbm = fa.create_block_mask(fa.offset_mask(fa.causal(), L - 1), 1, 1, 1, L, device=dev)
        pt = cache.page_table()
        pbm = fa.convert_block_mask(lbm, pt)
        for splits in (1, 2, 0):
            t = timeit(lambda: fa.decode(q, cache.k_phys(), cache.v_phys(), L - 1, fa.causal(), fa.noop_score(),
                                         pbm, page_table=pt, num_splits=splits))
            gb = 2 * B * H * L * D * 2 / 1e9
            print(f"C5 decode splits={splits} {t:.3f} ms  {gb / t:.3f} TB/s ({gb / t / 6.5418 * 100:.1f}% of 6541.8 GB/s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["fwd", "decode"])
