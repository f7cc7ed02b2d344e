#!/usr/bin/env python
"""Benchmark of the B200-native FlexAttention hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

Workload (BASELINE.json configs[1], "C2"): sliding_window(1024) mask_mod + ALiBi score_mod,
B=4 H=16 S=8192 D=128 bf16, forward + backward. One step = forward + backward over one batch
with the BlockMask prebuilt (as the reference harness builds it outside the timed region,
bench.cpp:412-426); the builder is timed separately and reported as `block_mask_us`.
Metric: effective TFLOPS on unmasked FLOPs (fwd = 4*D*N_live, fwd+bwd = 3.5x fwd), whole job.

Multi-GPU (torchrun, one process per GPU): every rank runs its own C2 batch (weak scaling;
the path shards by (batch x head) with no collective); time = max over ranks.
`--impl reference` times the reference CPU implementation (oracle/_ref built from
/root/reference sources; the C restatement when that is absent) on one (b, h) slice of the
same workload per step, with all host threads, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ---- workloads (exact unmasked FLOPs measured with the reference builder) ----
CONFIGS = {
    "C2": dict(desc="sliding_window(1024)+alibi(alibi_slopes(16)) B4 H16 S8192 D128 bf16 fwd+bwd",
               B=4, Hq=16, Hkv=16, L=8192, D=128, mask="sliding", score="alibi",
               fwd_gflop=257.95, live_per_bh=7872000),
    "C3": dict(desc="and_mask(document_mask(8 docs), causal) B1 H32 S16384 D128 bf16 fwd+bwd",
               B=1, Hq=32, Hkv=32, L=16384, D=128, mask="doc_causal", score="noop",
               fwd_gflop=568.85, live_per_bh=34720028),
    "C4": dict(desc="causal + soft_cap(50) GQA 32/8 B2 S8192 D128 bf16 fwd+bwd",
               B=2, Hq=32, Hkv=8, L=8192, D=128, mask="causal", score="softcap",
               fwd_gflop=1099.65, live_per_bh=33558528),
}
# C5 (decode, HBM-bound): Q_LEN 1, paged KV (page 128) via the converted BlockMask
C5 = dict(desc="paged decode Q_LEN=1 B64 H32 KV_LEN 32768 page 128 D128 bf16, offset_mask(causal, 32767)",
          B=64, H=32, L=32768, D=128, ps=128)
DOC_LENGTHS = [1004, 350, 639, 2533, 190, 1601, 7058, 3009]
SEED = 0x5EED0001  # per-config seed S_c (bench.cpp:414); Q/K/V/dO = S_c+1..+4


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), float(d["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 6650.0, "fallback (B200_PROFILING.md)"


def profile_traffic(key):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of one kernel from
    the committed ncu --set full summary of this build (profiles/ncu_summary.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d["kernels"][key]["dram_bytes"]
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and throttle reasons during the timed region (NVML, else nvidia-smi)."""

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.dev, self.period = device_index, period_s
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    _REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def _sample(self):
        if self._nvml is not None:
            p = self._nvml
            mhz = p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM)
            mask = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            self.samples.append(mhz)
            for bit, name in self._REASONS.items():
                if mask & bit:
                    self.reasons.add(name)
            return
        out = subprocess.run(["nvidia-smi", f"--id={self.dev}", "--query-gpu=clocks.sm,clocks.max.sm,"
                              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        f = [x.strip() for x in out.stdout.strip().split(",")]
        self.samples.append(float(f[0]))
        self.max_mhz = float(f[1])
        for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), f[2:]):
            if val.lower() == "active":
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---- our arm ------------------------------------------------------------------------------
def build_mods(fa, c, dev):
    import numpy as np
    import torch
    if c["mask"] == "sliding":
        mask = fa.sliding_window(1024)
    elif c["mask"] == "causal":
        mask = fa.causal()
    else:
        ids = np.concatenate([np.full(n, i) for i, n in enumerate(DOC_LENGTHS)])
        mask = fa.and_mask(fa.document_mask(torch.tensor(ids, dtype=torch.int32)), fa.causal())
    score = {"alibi": fa.alibi(fa.alibi_slopes(c["Hq"])), "softcap": fa.soft_cap(50.0),
             "noop": fa.noop_score()}[c["score"]]
    return mask, score


def cpu_reference_sample(c, kind_pref="reference"):
    """Time the reference CPU fwd+bwd on one (b, h) slice of the workload (bounded sample)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    L, D = c["L"], c["D"]
    q, k, v, do = (O.bf16_round(O.random_f32(SEED + i, (1, 1, L, D))) for i in range(1, 5))
    if c["mask"] == "sliding":
        om = O.sliding_window(1024)
    elif c["mask"] == "causal":
        om = O.causal()
    else:
        ids = np.concatenate([np.full(n, i) for i, n in enumerate(DOC_LENGTHS)])
        om = O.Mask(terms=O.MASK_DOCUMENT | O.MASK_CAUSAL, doc_ids=ids)
    if c["score"] == "alibi":
        os_ = O.Score(terms=O.SCORE_ALIBI, slopes=O.alibi_slopes(c["Hq"])[:1])
    elif c["score"] == "softcap":
        os_ = O.Score(terms=O.SCORE_SOFTCAP, cap=50.0)
    else:
        os_ = O.Score()
    cores = os.cpu_count() or 1
    slice_gflop = 3.5 * c["fwd_gflop"] / (c["B"] * c["Hq"])
    if O.ref_available() and kind_pref == "reference":
        fwd_s, bwd_s = O.ref_time_fwd_bwd(q, k, v, do, om, os_, workers=cores)
        return dict(seconds=fwd_s + bwd_s, fwd_s=fwd_s, bwd_s=bwd_s, cores=cores, kind="reference",
                    gflop=slice_gflop)
    # C restatement (single-threaded port) when the reference library is not built
    bm = O.create_block_mask(om, 1, 1, L, L)
    t0 = time.perf_counter()
    o, lse = O.forward(q, k, v, om, os_, bm)
    t1 = time.perf_counter()
    O.backward(q, k, v, o, lse, do, om, os_, bm)
    t2 = time.perf_counter()
    return dict(seconds=t2 - t0, fwd_s=t1 - t0, bwd_s=t2 - t1, cores=1, kind="port", gflop=slice_gflop)


def timed_events(n):
    import torch
    return [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]


def inputs_for(fa, c, seed, dev):
    B, Hq, Hkv, L, D = c["B"], c["Hq"], c["Hkv"], c["L"], c["D"]
    q = fa.random_tensor(seed + 1, (B, Hq, L, D), device=dev)
    k = fa.random_tensor(seed + 2, (B, Hkv, L, D), device=dev)
    v = fa.random_tensor(seed + 3, (B, Hkv, L, D), device=dev)
    do = fa.random_tensor(seed + 4, (B, Hq, L, D), device=dev)
    return q, k, v, do


def measure_builder(fa, mask, L, dev, reps=20):
    """create_block_mask (+ transpose) device time, mask evaluations/s and output GB/s."""
    import torch
    for _ in range(3):
        bm = fa.create_block_mask(mask, 1, 1, L, L, device=dev)
    torch.cuda.synchronize()
    # device time: `reps` builds captured in one CUDA graph (a Python-level loop of builds is
    # host-bound at ~45 us per call, far above the two kernels' device time)
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            keep = [fa.create_block_mask(mask, 1, 1, L, L, device=dev) for _ in range(reps)]
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1000.0
    del keep, g
    R = C_ = -(-L // 128)
    out_bytes = 2 * (2 * R * C_ + R + C_) * 4  # 8 int32 arrays (SURVEY §8d builder bytes)
    if mask.doc_ids is not None:
        out_bytes += mask.doc_ids.numel() * 4
    return bm, {"us": round(us, 2), "timing": "device, CUDA graph of 20 builds", "evals_per_s": float(f"{L * L / (us * 1e-6):.4g}"),
                "gb_per_s": round(out_bytes / (us * 1e-6) / 1e9, 3), "bytes": out_bytes}


def measure_attention(fa, name, c, dev, steps, warmup, seed, stream):
    """fwd + bwd of one config: step time, per-phase and per-kernel device times (CUDA events on
    the launching stream; the backward records events around its preprocess / main / convert)."""
    import torch
    q, k, v, do = inputs_for(fa, c, seed, dev)
    mask, score = build_mods(fa, c, dev)
    cfg = fa.AttentionConfig(gqa_group=c["Hq"] // c["Hkv"])
    bm, builder = measure_builder(fa, mask, c["L"], dev)
    fwd_ev, bwd_ev, ph = timed_events(steps), timed_events(steps), [timed_events(1)[0] + timed_events(1)[0]
                                                                    for _ in range(steps)]

    def step(i=None):
        if i is not None:
            fwd_ev[i][0].record(stream)
        res = fa.forward(q, k, v, score, bm, cfg)
        if i is not None:
            fwd_ev[i][1].record(stream)
            bwd_ev[i][0].record(stream)
        g = fa.backward(q, k, v, res, do, score, bm, cfg=cfg, phase_events=ph[i] if i is not None else None)
        if i is not None:
            bwd_ev[i][1].record(stream)
        return res, g

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(steps):
        step(i)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    fwd_ms = statistics.mean(a.elapsed_time(b) for a, b in fwd_ev)
    bwd_ms = statistics.mean(a.elapsed_time(b) for a, b in bwd_ev)
    pre_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ph)
    main_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ph)
    conv_ms = statistics.mean(e[2].elapsed_time(e[3]) for e in ph)
    # the deterministic (split) backward: dK/dV kernel + the TMEM-accumulating dQ pass
    res = fa.forward(q, k, v, score, bm, cfg)
    det_ev = timed_events(steps)
    for i in range(-1, steps):
        if i >= 0:
            det_ev[i][0].record(stream)
        fa.backward(q, k, v, res, do, score, bm, cfg=cfg, deterministic=True)
        if i >= 0:
            det_ev[i][1].record(stream)
    torch.cuda.synchronize()
    det_ms = statistics.mean(a.elapsed_time(b) for a, b in det_ev)
    del q, k, v, do, res
    fg = c["fwd_gflop"]
    return {"workload": f"{name}: {c['desc']}", "ms_per_step": round(ms, 4),
            "fwd_bwd_tflops": round(3.5 * fg / ms, 2), "fwd_ms": round(fwd_ms, 4),
            "fwd_tflops": round(fg / fwd_ms, 2), "bwd_ms": round(bwd_ms, 4),
            "bwd_tflops": round(2.5 * fg / bwd_ms, 2),
            "bwd_kernels_ms": {"preprocess": round(pre_ms, 4), "main": round(main_ms, 4),
                               "dq_convert": round(conv_ms, 4)},
            "bwd_main_tflops": round(2.5 * fg / main_ms, 2),
            "bwd_deterministic_ms": round(det_ms, 4), "bwd_deterministic_tflops": round(2.5 * fg / det_ms, 2),
            "fwd_gflop": fg, "block_mask": builder}


def measure_c1(fa, dev, steps, stream):
    """C1: causal B1 H4 S1024 D64 fp32 forward (the reference's CPU-runnable case) on the
    exact-arithmetic CUDA-core kernel (1e-4 gate); 0.537 GFLOP of live pairs."""
    import torch
    B, H, L, D = 1, 4, 1024, 64
    q, k, v = (fa.random_tensor(SEED + i, (B, H, L, D), dtype=torch.float32, device=dev) for i in (1, 2, 3))
    bm = fa.create_block_mask(fa.causal(), 1, 1, L, L, device=dev)
    for _ in range(3):
        fa.forward(q, k, v, fa.noop_score(), bm)
    torch.cuda.synchronize()
    ev = timed_events(steps)
    for i in range(steps):
        ev[i][0].record(stream)
        fa.forward(q, k, v, fa.noop_score(), bm)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    gflop = 4 * D * B * H * (L * (L + 1) // 2) / 1e9
    return {"workload": "C1: causal B1 H4 S1024 D64 fp32 forward (CUDA-core exact path)", "ms": round(ms, 4),
            "tflops": round(gflop / ms, 3), "gflop": round(gflop, 4)}


def measure_decode(fa, dev, steps, warmup, stream, hbm):
    """C5: paged split-KV decode, HBM-bound (bytes = K + V of every visited page)."""
    import torch
    c = C5
    B, H, L, D, ps = c["B"], c["H"], c["L"], c["D"], c["ps"]
    pages = B * (L // ps) + B
    cache = fa.PagedKVCache(B, pages, ps, H, D, device=dev)
    cache.shuffle_free_pages(SEED ^ 0xFA6E5)
    for b in range(B):  # logical K/V generated per batch element and scattered into pages
        kb = fa.random_tensor(SEED + 2, (1, H, L, D), device=dev, first=b * H * L * D)
        vb = fa.random_tensor(SEED + 3, (1, H, L, D), device=dev, first=b * H * L * D)
        cache.assign(b, kb, vb)
    del kb, vb
    q = fa.random_tensor(SEED + 1, (B, H, 1, D), device=dev)
    off = L - 1
    lbm = fa.create_block_mask(fa.offset_mask(fa.causal(), off), 1, 1, 1, L, device=dev)
    pt = cache.page_table()
    pbm = fa.convert_block_mask(lbm, pt)
    kp, vp = cache.k_phys(), cache.v_phys()

    def call():
        return fa.decode(q, kp, vp, off, fa.causal(), fa.noop_score(), pbm, page_table=pt)

    for _ in range(warmup):
        call()
    torch.cuda.synchronize()
    ev = timed_events(steps)
    for i in range(steps):
        ev[i][0].record(stream)
        call()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    kv_bytes = 2 * B * H * L * D * 2
    other = B * H * D * 2 * 2 + B * H * 4 + pbm.kv_indices.numel() * 4 * 2
    gbs = (kv_bytes + other) / (ms * 1e-3) / 1e9
    del cache, kp, vp
    return {"workload": f"C5: {c['desc']}", "ms_per_step": round(ms, 4), "gb_per_s": round(gbs, 1),
            "hbm_frac": round(gbs / hbm, 4), "bytes_per_step": kv_bytes + other,
            "gflop": round(4 * B * H * L * D / 1e9, 2),
            "l2": "34.4 GB of K/V per step >> 126 MB L2 (no flush needed)"}


def bind_to_gpu_numa(local):
    """Pin this process to the CPUs of the GPU's NUMA node (sysfs local_cpulist), so the pinned
    host buffers of the e2e leg live next to the GPU's PCIe root; returns the previous mask."""
    import torch
    prev = os.sched_getaffinity(0)
    try:
        pr = torch.cuda.get_device_properties(local)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        if cpus and cpus != prev:
            os.sched_setaffinity(0, cpus)
    except Exception:  # no sysfs entry / attribute: leave the mask as it is
        pass
    return prev


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cpu_mask = bind_to_gpu_numa(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_2412_05496_b200 as fa
    from paper_2412_05496_b200 import shard

    c = CONFIGS[args.config]
    B, Hq, Hkv, L, D = c["B"], c["Hq"], c["Hkv"], c["L"], c["D"]
    mask, score = build_mods(fa, c, dev)
    cfg = fa.AttentionConfig(gqa_group=Hq // Hkv)
    if args.strong and world > 1:
        # strong scaling: ONE job of the config; this rank owns a contiguous range of its
        # (batch, kv head) units with all G q heads of each (engine.cpp:311-331), no collective
        G = Hq // Hkv
        sh = shard.rect_shard(B, Hkv, world, rank)
        q, k, v, do = shard.slice_job(*inputs_for(fa, c, SEED, dev), G, sh)
        score = shard.shard_score(score, G, sh)
        my_frac = (sh[1] - sh[0]) * (sh[3] - sh[2]) / (B * Hkv)
        torch.cuda.empty_cache()
        job_gflop = 3.5 * c["fwd_gflop"]
        scaling = "strong"
        parallelism = (f"dp{world}: one {args.config} job split into {world} rectangles of its {B * Hkv} "
                       f"(batch, kv-head) units, no collective")
    else:
        seed = SEED + 1000003 * rank  # each rank: its own batch of the sharded job
        q, k, v, do = inputs_for(fa, c, seed, dev)
        job_gflop = 3.5 * c["fwd_gflop"] * world
        my_frac = 1.0
        scaling = "weak"
        parallelism = f"dp{world}: one (b,h)-shard per GPU, no collective"
    bm = fa.create_block_mask(mask, 1, 1, L, L, device=dev)

    stream = torch.cuda.current_stream()
    steps = args.steps
    fwd_ev, bwd_ev = timed_events(steps), timed_events(steps)
    ph = [timed_events(1)[0] + timed_events(1)[0] for _ in range(steps)]

    def step(i=None):
        if i is not None:
            fwd_ev[i][0].record(stream)
        res = fa.forward(q, k, v, score, bm, cfg)
        if i is not None:
            fwd_ev[i][1].record(stream)
            bwd_ev[i][0].record(stream)
        g = fa.backward(q, k, v, res, do, score, bm, cfg=cfg, phase_events=ph[i] if i is not None else None)
        if i is not None:
            bwd_ev[i][1].record(stream)
        return res, g

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    launches0 = fa.launch_count()
    sampler = ClockSampler(local)
    with sampler:
        barrier()
        torch.cuda.synchronize()
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(steps):
            step(i)
        t_end.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = fa.launch_count() - launches0
    ms = t_start.elapsed_time(t_end)
    fwd_ms = statistics.mean(a.elapsed_time(b) for a, b in fwd_ev)
    bwd_ms = statistics.mean(a.elapsed_time(b) for a, b in bwd_ev)
    main_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ph)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms, fwd_ms, bwd_ms, main_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, fwd_ms, bwd_ms, main_ms = t.tolist()

    # ---- e2e: same step through the public API with host buffers, H2D + D2H inside ----
    # Every step copies its four inputs host->device and its five results device->host (pinned
    # memory). Steps are software-pipelined over three streams (H2D of step i+1 and D2H of step
    # i-1 overlap step i's kernels; PCIe is full duplex), with double-buffered device inputs.
    host = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (q, k, v, do)]
    for h_, d_ in zip(host, (q, k, v, do)):
        h_.copy_(d_)
    outs = [[torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (q, q, k, v)] for _ in range(2)]
    lse_h = [torch.empty(q.shape[:3], dtype=torch.float32, pin_memory=True) for _ in range(2)]
    dbuf = [[torch.empty_like(x) for x in (q, k, v, do)] for _ in range(2)]
    e2e_steps = max(2, min(steps, 24))  # pipeline fill and drain amortised over the steps
    s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def e2e_run(nsteps):
        comp_done, d2h_done, keep = [], [], []
        for i in range(nsteps):
            ib = i % 2
            with torch.cuda.stream(s_h2d):
                if i >= 2:
                    s_h2d.wait_event(comp_done[i - 2])  # device inputs of step i-2 consumed
                for d_, h_ in zip(dbuf[ib], host):
                    d_.copy_(h_, non_blocking=True)
                h2d_ev = torch.cuda.Event()
                h2d_ev.record(s_h2d)
            stream.wait_event(h2d_ev)
            dq_, dk_, dv_, ddo = dbuf[ib]
            res = fa.forward(dq_, dk_, dv_, score, bm, cfg)
            g = fa.backward(dq_, dk_, dv_, res, ddo, score, bm, cfg=cfg)
            ev = torch.cuda.Event()
            ev.record(stream)
            comp_done.append(ev)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev)
                if i >= 2:
                    s_d2h.wait_event(d2h_done[i - 2])  # host output buffers of step i-2 written
                for o_h, o_d in zip(outs[ib], (res.out, g.dq, g.dk, g.dv)):
                    o_h.copy_(o_d, non_blocking=True)
                lse_h[ib].copy_(res.lse, non_blocking=True)
                dv_ev = torch.cuda.Event()
                dv_ev.record(s_d2h)
                d2h_done.append(dv_ev)
            keep.append((res, g))  # results stay alive until their D2H has run
        stream.wait_event(d2h_done[-1])
        return keep

    e2e_run(2)
    torch.cuda.synchronize()
    barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    s_h2d.wait_stream(stream)
    keep = e2e_run(e2e_steps)
    s1.record(stream)
    torch.cuda.synchronize()
    del keep
    e2e_ms = s0.elapsed_time(s1) / e2e_steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
        barrier()
    h2d = sum(x.numel() * x.element_size() for x in host)
    d2h = sum(x.numel() * x.element_size() for x in outs[0]) + lse_h[0].numel() * 4
    del host, outs, lse_h, dbuf, q, k, v, do
    torch.cuda.empty_cache()

    peak, hbm, peak_kind = peaks()
    # ---- every other BASELINE workload, one GPU (rank 0 of a single-process run) ----
    per_config = {}
    if world == 1 and not args.headline_only:
        for name in ("C2", "C3", "C4"):
            per_config[name] = measure_attention(fa, name, CONFIGS[name], dev, max(5, min(steps, 20)),
                                                 max(3, args.warmup), SEED, stream)
            per_config[name]["pct_of_peak_fwd_bwd"] = round(100 * per_config[name]["fwd_bwd_tflops"] / peak, 2)
            torch.cuda.empty_cache()
        per_config["C1"] = measure_c1(fa, dev, max(5, min(steps, 20)), stream)
        try:
            per_config["C5"] = measure_decode(fa, dev, max(5, min(steps, 20)), max(3, args.warmup), stream, hbm)
        except Exception as e:  # reported, not fatal
            per_config["C5"] = {"error": str(e)[:200]}
        torch.cuda.empty_cache()

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    ms_per_step = ms / steps
    tflops = job_gflop / ms_per_step
    bwd_gflop = 2.5 * c["fwd_gflop"]
    achieved = bwd_gflop * my_frac / main_ms  # the dominant kernel alone, this GPU
    line = {
        "metric": f"effective TFLOPS (unmasked FLOPs) fwd+bwd, {args.config} "
                  f"{'sliding_window(1024)+ALiBi' if args.config == 'C2' else c['desc']}",
        "value": round(tflops, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: SplitMix64 uniform[-1,1) (random.hpp) generated on device, bf16 RNE",
        "config": {"workload": f"{args.config}: {c['desc']}", "global_batch": B * (world if scaling == "weak" else 1),
                   "seq_len": L, "heads_q": Hq, "heads_kv": Hkv, "head_dim": D, "parallelism": parallelism,
                   "l2": "inputs 4 x 134 MB > 126 MB L2 (no flush needed)",
                   "block_mask": "built once outside the timed region (builder timed separately)"},
        "fwd_tflops": round(c["fwd_gflop"] * my_frac / fwd_ms, 2), "bwd_tflops": round(bwd_gflop * my_frac / bwd_ms, 2),
        "fwd_ms": round(fwd_ms, 4), "bwd_ms": round(bwd_ms, 4),
        "pct_of_peak": round(100.0 * tflops / world / peak, 2), "peak_tflops": peak, "peak_kind": peak_kind,
        "roofline": {"bound": "tensor", "kernel": "flex_bwd_sm100_kernel (backward main kernel alone)",
                     "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4), "traffic": profile_traffic(f"{args.config}_bwd_main"),
                     "kernel_ms": round(main_ms, 4),
                     "algorithmic_per_launch": f"{bwd_gflop * my_frac:.2f} GFLOP = 2.5 x 4*D*N_live"},
        "e2e": {"value": round(job_gflop / e2e_ms, 2), "unit": "TFLOP/s",
                "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                "ms_per_step": round(e2e_ms, 3),
                "note": f"{e2e_steps} steps pipelined over H2D / compute / D2H streams"},
        "gpu_launches": int(launches),
        "clocks": sampler.summary(),
    }
    if per_config:
        line["configs"] = per_config
    if world == 1 and not args.no_cpu_baseline:
        try:
            os.sched_setaffinity(0, cpu_mask)  # the CPU reference gets every host core again
            cb = cpu_reference_sample(c)
            line["cpu_baseline"] = {
                "value": round(cb["gflop"] / cb["seconds"] / 1000.0, 6), "unit": "TFLOP/s",
                "cores": cb["cores"], "kind": cb["kind"],
                "sample": f"one (b,h) slice of {args.config} (1/{B * Hq} of the batch) fwd+bwd, "
                          f"{cb['seconds']:.2f} s (fwd {cb['fwd_s']:.2f} s, bwd {cb['bwd_s']:.2f} s)"}
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "none",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---- reference arm ------------------------------------------------------------------------
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    c = CONFIGS[args.config]
    for _ in range(args.warmup):
        cpu_reference_sample(c)
    times, cb = [], None
    for _ in range(args.steps):
        cb = cpu_reference_sample(c)
        times.append(cb["seconds"])
    sec = statistics.median(times)
    value = cb["gflop"] / sec / 1000.0
    line = {
        "impl": "reference",
        "metric": "effective TFLOPS (unmasked FLOPs) fwd+bwd, C2 sliding_window(1024)+ALiBi",
        "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1000.0, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: SplitMix64 uniform[-1,1) (random.hpp), bf16-rounded, held as fp32",
        "config": {"workload": f"{args.config}: {c['desc']}", "sample": "one (b,h) slice per step",
                   "parallelism": f"BLOCKATTN_WORKERS={cb['cores']} host threads"},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": cb["cores"], "kind": cb["kind"],
                         "sample": f"one (b,h) slice of {args.config} (1/{c['B'] * c['Hq']}) fwd+bwd per step"},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--headline-only", action="store_true", help="skip the per-config C2-C5 measurements")
    ap.add_argument("--strong", action="store_true",
                    help="N>1: split ONE job's (batch, kv-head) units across the ranks (strong scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
