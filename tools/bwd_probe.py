"""Backward diagnostics at a BASELINE config: device time and, with the instrumented build
(make trace + FA_LIB_PATH), the per-phase cycle trace of CTA 0 (FA_BWD_TRACE).
Usage: python tools/bwd_probe.py [C2|C3|C4 ...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2412_05496_b200 as fa  # noqa: E402
from perf_probe import configs, timeit  # noqa: E402


def main(names):
    dev = torch.device("cuda:0")
    cs = configs(dev)
    for name in names:
        c = cs[name]
        D = 128
        q = fa.random_tensor(1, (c["B"], c["Hq"], c["L"], D), device=dev)
        k = fa.random_tensor(2, (c["B"], c["Hkv"], c["L"], D), device=dev)
        v = fa.random_tensor(3, (c["B"], c["Hkv"], c["L"], D), device=dev)
        do = fa.random_tensor(4, q.shape, device=dev)
        bm = fa.create_block_mask(c["mask"], 1, 1, c["L"], c["L"], device=dev)
        cfg = fa.AttentionConfig(gqa_group=c["Hq"] // c["Hkv"])
        res = fa.forward(q, k, v, c["score"], bm, cfg)
        run = lambda: fa.backward(q, k, v, res, do, c["score"], bm, cfg=cfg)  # noqa: E731
        t = timeit(run, iters=5, warm=2)
        print(f"{name} bwd exp=0 {t:.3f} ms  {2.5 * c['gf'] / t:.1f} TFLOPS", flush=True)
        os.environ["FA_BWD_TRACE"] = os.environ.get("TRACE_LEVEL", "1")
        run()
        torch.cuda.synchronize()
        del os.environ["FA_BWD_TRACE"]
        del q, k, v, do, res


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2"])
