"""Backward timing, default vs deterministic dQ order, at the BASELINE configs C2-C4."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2412_05496_b200 as fa  # noqa: E402
from perf_probe import configs, timeit  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    for name, c in configs(dev).items():
        D = 128
        q = fa.random_tensor(1, (c["B"], c["Hq"], c["L"], D), device=dev)
        k = fa.random_tensor(2, (c["B"], c["Hkv"], c["L"], D), device=dev)
        v = fa.random_tensor(3, (c["B"], c["Hkv"], c["L"], D), device=dev)
        do = fa.random_tensor(4, q.shape, device=dev)
        bm = fa.create_block_mask(c["mask"], 1, 1, c["L"], c["L"], device=dev)
        cfg = fa.AttentionConfig(gqa_group=c["Hq"] // c["Hkv"])
        res = fa.forward(q, k, v, c["score"], bm, cfg)
        for det in (False, True):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            t = timeit(lambda: fa.backward(q, k, v, res, do, c["score"], bm, cfg=cfg, deterministic=det,
                                           phase_events=ev), iters=5, warm=2)
            ph = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
            print(f"{name} bwd det={int(det)} {t:.3f} ms {2.5 * c['gf'] / t:.1f} TFLOPS  phases(pre/main/conv) "
                  + " ".join(f"{x:.3f}" for x in ph), flush=True)
        del q, k, v, do


if __name__ == "__main__":
    main()
