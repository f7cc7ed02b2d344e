"""Host enqueue cost vs device time of the C2 fwd+bwd step through the public API (is the step
GPU-bound?), for 20 and 100 back-to-back steps.  python tools/enqueue_probe.py"""
import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
import bench
import paper_2412_05496_b200 as fa
dev = torch.device("cuda:0")
c = bench.CONFIGS["C2"]
mask, score = bench.build_mods(fa, c, dev)
cfg = fa.AttentionConfig(gqa_group=c["Hq"] // c["Hkv"])
q, k, v, do = bench.inputs_for(fa, c, 1, dev)
bm = fa.create_block_mask(mask, 1, 1, c["L"], c["L"], device=dev)
def step():
    res = fa.forward(q, k, v, score, bm, cfg)
    return fa.backward(q, k, v, res, do, score, bm, cfg=cfg)
for _ in range(5): step()
torch.cuda.synchronize()
for n in (20, 100):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); s.record()
    for _ in range(n): step()
    t1 = time.perf_counter(); e.record(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"n={n}: gpu {s.elapsed_time(e)/n:.4f} ms/step, python enqueue {1e3*(t1-t0)/n:.4f} ms/step, wall {1e3*(t2-t0)/n:.4f}")
# CPU cost of one step with the GPU idle
torch.cuda.synchronize()
t0 = time.perf_counter(); step(); t1 = time.perf_counter()
print(f"single step enqueue {1e3*(t1-t0):.3f} ms")
