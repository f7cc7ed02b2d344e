"""Forward per-step cycle trace of CTA 0 with the instrumented build (make ftrace):
    FA_LIB_PATH=paper_2412_05496_b200/build/ftrace/libflexattn_b200.so python tools/fwd_trace.py [C2|C3|C4 ...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2412_05496_b200 as fa  # noqa: E402
from perf_probe import configs  # noqa: E402


def main(names):
    dev = torch.device("cuda:0")
    cs = configs(dev)
    for name in names:
        c = cs[name]
        q = fa.random_tensor(1, (c["B"], c["Hq"], c["L"], 128), device=dev)
        k = fa.random_tensor(2, (c["B"], c["Hkv"], c["L"], 128), device=dev)
        v = fa.random_tensor(3, (c["B"], c["Hkv"], c["L"], 128), device=dev)
        bm = fa.create_block_mask(c["mask"], 1, 1, c["L"], c["L"], device=dev)
        cfg = fa.AttentionConfig(gqa_group=c["Hq"] // c["Hkv"])
        for _ in range(3):
            fa.forward(q, k, v, c["score"], bm, cfg)
        torch.cuda.synchronize()
        print(f"== {name}", file=sys.stderr, flush=True)
        os.environ["FA_FWD_TRACE"] = "1"
        fa.forward(q, k, v, c["score"], bm, cfg)
        torch.cuda.synchronize()
        del os.environ["FA_FWD_TRACE"]


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2"])
