"""Same-box context bar: torch.nn.attention.flex_attention compiled with the
Triton backend — the paper's own system — on the BASELINE configs C2-C4, fwd and fwd+bwd,
counted with the same live FLOPs as bench.py. Context only, not the reference arm.
Usage: python tools/torch_flex_bar.py [C2 C3 C4]"""
import json
import os
import sys

import numpy as np
import torch
from torch.nn.attention.flex_attention import create_block_mask, flex_attention

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DOCS = [1004, 350, 639, 2533, 190, 1601, 7058, 3009]
GF = {"C2": 257.95, "C3": 568.85, "C4": 1099.65}


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def main(names):
    dev = "cuda"
    out = {}
    fa = torch.compile(flex_attention, dynamic=False)
    for name in names:
        D = 128
        if name == "C2":
            B, Hq, Hkv, L = 4, 16, 16, 8192
            slopes = torch.tensor([-(2 ** (-8.0 * (h + 1) / Hq)) for h in range(Hq)], device=dev)

            def mask_mod(b, h, q, kv):
                return (q >= kv) & (q - kv <= 1024)

            def score_mod(s, b, h, q, kv):
                return s + slopes[h] * (q - kv)
        elif name == "C3":
            B, Hq, Hkv, L = 1, 32, 32, 16384
            ids = torch.tensor(np.concatenate([np.full(n, i) for i, n in enumerate(DOCS)]), device=dev)

            def mask_mod(b, h, q, kv):
                return (q >= kv) & (ids[q] == ids[kv])

            score_mod = None
        else:
            B, Hq, Hkv, L = 2, 32, 8, 8192

            def mask_mod(b, h, q, kv):
                return q >= kv

            def score_mod(s, b, h, q, kv):
                return 50.0 * torch.tanh(s / 50.0)
        bm = create_block_mask(mask_mod, None, None, L, L, device=dev, BLOCK_SIZE=128)
        q = torch.randn(B, Hq, L, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
        k = torch.randn(B, Hkv, L, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
        v = torch.randn(B, Hkv, L, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
        do = torch.randn(B, Hq, L, D, device=dev, dtype=torch.bfloat16)
        kw = dict(score_mod=score_mod, block_mask=bm, enable_gqa=Hq != Hkv)
        try:
            t_f = timeit(lambda: fa(q, k, v, **kw))

            def fb():
                o = fa(q, k, v, **kw)
                o.backward(do)
            t_fb = timeit(fb)
            out[name] = {"fwd_ms": round(t_f, 4), "fwd_tflops": round(GF[name] / t_f, 1),
                         "fwd_bwd_ms": round(t_fb, 4), "fwd_bwd_tflops": round(3.5 * GF[name] / t_fb, 1)}
        except Exception as e:  # reported, not fatal
            out[name] = {"error": str(e)[:300]}
        print(name, out[name], flush=True)
        del q, k, v, do, bm
        torch.cuda.empty_cache()
    print(json.dumps({"context": "torch.nn.attention.flex_attention (torch %s, Triton backend, torch.compile)"
                      % torch.__version__, "configs": out}))


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3", "C4"])
