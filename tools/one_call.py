"""One forward or backward call at a BASELINE config (for ncu captures).
Usage: python tools/one_call.py fwd|bwd C2|C3|C4"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2412_05496_b200 as fa  # noqa: E402
from perf_probe import configs  # noqa: E402

which, name = sys.argv[1], sys.argv[2]
dev = torch.device("cuda:0")
c = configs(dev)[name]
D = 128
q = fa.random_tensor(1, (c["B"], c["Hq"], c["L"], D), device=dev)
k = fa.random_tensor(2, (c["B"], c["Hkv"], c["L"], D), device=dev)
v = fa.random_tensor(3, (c["B"], c["Hkv"], c["L"], D), device=dev)
bm = fa.create_block_mask(c["mask"], 1, 1, c["L"], c["L"], device=dev)
cfg = fa.AttentionConfig(gqa_group=c["Hq"] // c["Hkv"])
res = fa.forward(q, k, v, c["score"], bm, cfg)
if which == "bwd":
    do = fa.random_tensor(4, q.shape, device=dev)
    fa.backward(q, k, v, res, do, c["score"], bm, cfg=cfg)
torch.cuda.synchronize()
print("done")
