"""Time create_block_mask (+ transpose) for the BASELINE masks and the mask library on the GPU."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2412_05496_b200 as fa  # noqa: E402

DOC = [1004, 350, 639, 2533, 190, 1601, 7058, 3009]
dev = torch.device("cuda:0")
ids = np.concatenate([np.full(n, i) for i, n in enumerate(DOC)])
g = fa.NAGeometry(128, 128, 15)
cases = [("C2 sliding(1024)", fa.sliding_window(1024), 8192),
         ("C3 doc&causal", fa.and_mask(fa.document_mask(ids), fa.causal()), 16384),
         ("C4 causal", fa.causal(), 8192),
         ("C5 offset causal q=1", fa.offset_mask(fa.causal(), 32767), (1, 32768)),
         ("prefix_lm(2048)", fa.prefix_lm(2048), 8192),
         ("na_naive 128x128 k15", fa.na_naive(g), 16384),
         ("na_tiled 128x128 k15 t8", fa.remap_mask(fa.na_naive(g), fa.tile_permutation(g, 8)), 16384),
         ("hash(909)", fa.hash_mask(909, 128), 4096)]
for name, m, L in cases:
    ql, kl = (L, L) if isinstance(L, int) else L
    for _ in range(3):
        fa.create_block_mask(m, 1, 1, ql, kl, device=dev)
    torch.cuda.synchronize()
    n = 20
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            keep = [fa.create_block_mask(m, 1, 1, ql, kl, device=dev) for _ in range(n)]
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1000
    print(f"{name:28s} {us:9.2f} us  {ql * kl / us / 1e6:8.3f} T evals/s")
