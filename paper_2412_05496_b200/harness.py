"""GPU port of the reference's run / verify harness (bench.cpp, bench_cli.cpp; SURVEY.md §8f
rank 4): the same variant names, config keys (key = value or JSON), grid order, seeds
(cfg.seed + 1000003 * point, Q/K/V = seed + 1..3) and CSV schema

    variant,B,Hq,Hkv,qlen,kvlen,D,bs,mode,median_ns,madds,density,maxabs_err,rmse

with every point computed by the sm_100a kernels and checked against a dense float64 PyTorch
restatement of the same math on the same (dtype-rounded) inputs. Thresholds: the reference's
for float32 (bench.cpp:30-37); for bf16 the tolerance the north star states (2e-2).

    python -m paper_2412_05496_b200.harness run --variant "causal, alibi" --qlen 1024 --mode forward
    python -m paper_2412_05496_b200.harness verify
Exit codes as bench_cli: 0 ok, 1 error (bad config / variant), 2 a correctness check failed.
"""
from __future__ import annotations

import argparse
import json
import math
import re
import sys
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import api as fa

CSV_HEADER = "variant,B,Hq,Hkv,qlen,kvlen,D,bs,mode,median_ns,madds,density,maxabs_err,rmse"
MODES = ("forward", "backward", "decode", "paged")
# bench.cpp:30-37 (float32 engine) and the bf16 tolerance of the north star
TOL = {torch.float32: dict(fwd=1e-4, rmse=1e-5, bwd=1e-4, bwd_rmse=1e-5, decode=1e-4),
       torch.bfloat16: dict(fwd=2e-2, rmse=5e-3, bwd=2e-2, bwd_rmse=5e-3, decode=2e-2)}


class ConfigParse(fa.Error):
    pass


class UnknownVariant(fa.Error):
    pass


@dataclass
class BenchConfig:
    """BenchConfig (bench.hpp:37-52)."""
    variants: List[str] = field(default_factory=list)
    batch: int = 1
    q_heads: int = 1
    kv_heads: int = 1
    dim: int = 16
    q_lens: List[int] = field(default_factory=list)
    kv_lens: List[int] = field(default_factory=list)
    block_sizes: List[int] = field(default_factory=lambda: [128])
    modes: List[str] = field(default_factory=lambda: ["forward"])
    repeats: int = 5
    seed: int = 0x5EED0001
    page_size: int = 0
    dtype: torch.dtype = torch.float32

    def validate(self):
        if not self.variants:
            raise ConfigParse("config: no variant")
        if not self.q_lens:
            raise ConfigParse("config: no q_len")
        if self.batch < 1 or self.q_heads < 1 or self.kv_heads < 1 or self.dim < 1:
            raise ConfigParse("config: batch, heads and dim must be >= 1")
        if self.q_heads % self.kv_heads:
            raise ConfigParse("config: q_heads must be a multiple of kv_heads")
        if self.repeats < 3:
            raise ConfigParse("config: repeats must be >= 3")
        for m in self.modes:
            if m not in MODES:
                raise ConfigParse(f"unknown mode '{m}'")


def _split_top(s: str) -> List[str]:
    out, cur, depth = [], "", 0
    for ch in s:
        depth += ch == "("
        depth -= ch == ")"
        if ch == "," and depth == 0:
            out.append(cur.strip())
            cur = ""
        else:
            cur += ch
    if cur.strip() or not out:
        out.append(cur.strip())
    return out


def parse_config_text(text: str, is_json: bool) -> BenchConfig:
    """load_config / parse_config_text (bench.cpp:212-353)."""
    cfg = BenchConfig()
    if is_json:
        items = json.loads(text).items()
    else:
        items = []
        for line in text.splitlines():
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ConfigParse(f"config: expected key = value, got '{line}'")
            k, v = line.split("=", 1)
            items.append((k.strip(), v.strip()))
    ints = lambda v: [int(x) for x in (v if isinstance(v, list) else _split_top(str(v)))]  # noqa: E731
    strs = lambda v: [str(x).strip() for x in (v if isinstance(v, list) else _split_top(str(v)))]  # noqa: E731
    for k, v in items:
        if k == "variant":
            cfg.variants = strs(v)
        elif k in ("batch", "q_heads", "kv_heads", "dim", "repeats", "page_size"):
            setattr(cfg, k, int(v))
        elif k == "seed":
            cfg.seed = int(str(v), 0)
        elif k == "q_len":
            cfg.q_lens = ints(v)
        elif k == "kv_len":
            cfg.kv_lens = ints(v)
        elif k == "block_size":
            cfg.block_sizes = ints(v)
        elif k == "mode":
            cfg.modes = strs(v)
        elif k == "dtype":
            cfg.dtype = {"float32": torch.float32, "bf16": torch.bfloat16}[str(v)]
        else:
            raise ConfigParse(f"config: unknown key '{k}'")
    cfg.validate()
    return cfg


def load_config(path: str) -> BenchConfig:
    try:
        text = open(path).read()
    except OSError:
        raise ConfigParse(f"config: cannot open {path}") from None
    return parse_config_text(text, path.endswith(".json"))


# ---- variants (bench.cpp:146-191) --------------------------------------------------------------
_GOLD, _M64 = 0x9E3779B97F4A7C15, (1 << 64) - 1


def _splitmix(state: int):
    state = (state + _GOLD) & _M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return state, z ^ (z >> 31)


def make_doc_ids(length: int, ndocs: int, seed: int) -> np.ndarray:
    """make_doc_ids (bench.cpp:115-129): ndocs - 1 distinct cut points from SplitMix64."""
    ndocs = max(1, min(ndocs, length))
    st, cuts = seed & _M64, set()
    while len(cuts) < ndocs - 1:
        st, z = _splitmix(st)
        cuts.add(1 + z % (length - 1))
    ids = np.zeros(length, np.int64)
    doc = 0
    for t in range(length):
        doc += t in cuts
        ids[t] = doc
    return ids


@dataclass
class Variant:
    canonical: str
    mask: fa.MaskMod
    score: fa.ScoreMod
    dense: object  # (q_idx, kv_idx) -> bool tensor, for the float64 check
    slopes: Optional[list] = None
    cap: float = 0.0
    doc_ids: Optional[np.ndarray] = None


def make_variant(text: str, q_heads: int, q_len: int, kv_len: int, seed: int) -> Variant:
    t = text.strip()
    m = re.fullmatch(r"\s*([a-z_]+)\s*(?:\((.*)\))?\s*", t)
    if not m:
        raise ConfigParse(f"variant '{t}': cannot parse")
    name = m.group(1)
    args = [] if m.group(2) is None else [float(a) for a in _split_top(m.group(2))]

    def need(lo, hi):
        if not lo <= len(args) <= hi:
            raise ConfigParse(f"variant '{name}': expected {lo}..{hi} argument(s), got {len(args)}")

    def ia(i):
        if abs(args[i] - round(args[i])) > 1e-9:
            raise ConfigParse(f"variant '{name}': argument {i + 1} must be an integer")
        return int(round(args[i]))

    def square():
        if q_len != kv_len:
            raise ConfigParse(f"variant '{name}': needs q_len == kv_len")
        side = int(round(math.sqrt(q_len)))
        if side * side != q_len:
            raise ConfigParse(f"variant '{name}': token count {q_len} is not a square canvas")
        return fa.NAGeometry(side, side, ia(0))

    ones = lambda q, k: torch.ones(len(q), len(k), dtype=torch.bool, device=q.device)  # noqa: E731
    mask, score, dense, slopes, cap, doc_ids = fa.noop_mask(), fa.noop_score(), ones, None, 0.0, None
    if name == "noop":
        need(0, 0)
    elif name == "causal":
        need(0, 0)
        mask, dense = fa.causal(), lambda q, k: q[:, None] >= k[None, :]
    elif name == "sliding_window":
        need(1, 1)
        w = ia(0)
        mask = fa.sliding_window(w)
        dense = lambda q, k: (q[:, None] >= k[None, :]) & (q[:, None] - k[None, :] <= w)  # noqa: E731
    elif name == "document":
        need(0, 1)
        ids = make_doc_ids(max(q_len, kv_len), ia(0) if args else 4, seed ^ 0xD0C5)
        mask, doc_ids = fa.document_mask(ids), ids
        tid = torch.as_tensor(ids)
        dense = lambda q, k: tid.to(q.device)[q][:, None] == tid.to(q.device)[k][None, :]  # noqa: E731
    elif name == "prefix_lm":
        need(0, 1)
        p = ia(0) if args else max(1, q_len // 4)
        mask = fa.prefix_lm(p)
        dense = lambda q, k: (k[None, :] < p) | (q[:, None] >= k[None, :])  # noqa: E731
    elif name == "alibi":
        need(0, 0)
        slopes = fa.alibi_slopes(q_heads)
        score = fa.alibi(slopes)
    elif name == "soft_cap":
        need(1, 1)
        cap = args[0]
        score = fa.soft_cap(cap)
    elif name in ("na_naive", "na_tiled", "na_morton"):
        need(*(2, 2) if name == "na_tiled" else (1, 1))
        g = square()
        mask = fa.na_naive(g)
        perm = None
        if name == "na_tiled":
            perm = fa.tile_permutation(g, ia(1))
        elif name == "na_morton":
            perm = fa.morton_permutation(g)
        if perm is not None:
            mask = fa.remap_mask(mask, perm)
        fwd = torch.as_tensor(perm if perm is not None else list(range(g.tokens())))
        w, rad = g.canvas_w, g.kernel // 2

        def dense(q, k, fwd=fwd, w=w, rad=rad):
            f = fwd.to(q.device)
            a, b = f[q], f[k]
            dr = (a // w)[:, None] - (b // w)[None, :]
            dc = (a % w)[:, None] - (b % w)[None, :]
            return torch.maximum(dr.abs(), dc.abs()) <= rad
    else:
        raise UnknownVariant(f"unknown variant '{name}'")
    return Variant(t, mask, score, dense, slopes, cap, doc_ids)


# ---- dense float64 restatement (same math as the reference's dense oracle) ----------------------
def _dense_forward(q, k, v, var: Variant, scale, G, q_pos=None):
    q64, k64, v64 = q.double(), k.double(), v.double()
    if G > 1:
        k64, v64 = k64.repeat_interleave(G, 1), v64.repeat_interleave(G, 1)
    Lq, Lk = q.shape[2], k.shape[2]
    qi = torch.arange(Lq, device=q.device) if q_pos is None else q_pos
    ki = torch.arange(Lk, device=q.device)
    s = torch.einsum("bhqd,bhkd->bhqk", q64, k64) * scale
    if var.slopes is not None:
        sl = torch.tensor(var.slopes, dtype=torch.float64, device=q.device)[None, :, None, None]
        s = s + sl * (qi[:, None] - ki[None, :]).double()
    if var.cap:
        s = var.cap * torch.tanh(s / var.cap)
    live = var.dense(qi, ki)
    s = s.masked_fill(~live, -math.inf)
    lse = torch.logsumexp(s, -1)
    p = torch.exp(s - lse[..., None]).nan_to_num(0.0)
    return p @ v64, lse


@dataclass
class BenchRow:
    variant: str
    batch: int
    q_heads: int
    kv_heads: int
    q_len: int
    kv_len: int
    dim: int
    block_size: int
    mode: str
    median_ns: int = 0
    madds: int = 0
    density: float = 0.0
    max_abs_err: float = 0.0
    rmse_err: float = 0.0
    ok: bool = True
    detail: str = ""


def _median_ns(repeats, fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(int(e0.elapsed_time(e1) * 1e6))
    return sorted(ts)[len(ts) // 2]


def _rmse(a, b):
    return float(torch.sqrt(torch.mean((a.double() - b.double()) ** 2)))


def run_point(cfg: BenchConfig, variant_text: str, mode: str, q_len: int, kv_len: int, bs: int,
              point_idx: int, with_timing: bool = True, device="cuda") -> BenchRow:
    """run_point (bench.cpp:428-592) on the GPU."""
    dev = torch.device(device)
    seed = cfg.seed + 1000003 * point_idx
    var = make_variant(variant_text, cfg.q_heads, q_len, kv_len, seed)
    G = cfg.q_heads // cfg.kv_heads
    acfg = fa.AttentionConfig(gqa_group=G, block_size_q=bs, block_size_kv=bs)
    scale = 1.0 / math.sqrt(cfg.dim)
    q = fa.random_tensor(seed + 1, (cfg.batch, cfg.q_heads, q_len, cfg.dim), dtype=cfg.dtype, device=dev)
    k = fa.random_tensor(seed + 2, (cfg.batch, cfg.kv_heads, kv_len, cfg.dim), dtype=cfg.dtype, device=dev)
    v = fa.random_tensor(seed + 3, (cfg.batch, cfg.kv_heads, kv_len, cfg.dim), dtype=cfg.dtype, device=dev)
    bm = fa.create_block_mask(var.mask, 1, 1, q_len, kv_len, bs, bs, device=dev)
    rep = fa.sparsity(bm)
    row = BenchRow(var.canonical, cfg.batch, cfg.q_heads, cfg.kv_heads, q_len, kv_len, cfg.dim, bs, mode,
                   density=rep.density)
    tol = TOL[cfg.dtype]
    qi, ki = torch.arange(q_len, device=dev), torch.arange(kv_len, device=dev)
    live = int(var.dense(qi, ki).sum()) * cfg.batch * cfg.q_heads

    def fail(why):
        row.ok = False
        row.detail = (row.detail + "; " if row.detail else "") + why

    if mode == "forward":
        got = fa.forward(q, k, v, var.score, bm, acfg)
        want, lse = _dense_forward(q, k, v, var, scale, G)
        row.madds = 2 * cfg.dim * live  # q.k and p.v per live pair
        row.max_abs_err = float((got.out.double() - want).abs().max())
        row.rmse_err = _rmse(got.out, want)
        if row.max_abs_err > tol["fwd"]:
            fail(f"max abs {row.max_abs_err:.3g} > {tol['fwd']:.3g} vs dense float64")
        if row.rmse_err > tol["rmse"]:
            fail(f"rmse {row.rmse_err:.3g} > {tol['rmse']:.3g} vs dense float64")
        if with_timing:
            row.median_ns = _median_ns(cfg.repeats, lambda: fa.forward(q, k, v, var.score, bm, acfg))
    elif mode == "backward":
        fwd = fa.forward(q, k, v, var.score, bm, acfg)
        grads = fa.backward(q, k, v, fwd, fwd.out, var.score, bm, cfg=acfg)
        q64, k64, v64 = (x.double().requires_grad_(True) for x in (q, k, v))
        o64, _ = _dense_forward(q64, k64, v64, var, scale, G)
        o64.backward(fwd.out.double())
        row.madds = 4 * cfg.dim * live  # q.k, dO.v, p.dO, ds.q, ds.k share two recomputes
        errs = [float((g.double() - w.grad).abs().max()) / max(1.0, float(w.grad.abs().max()))
                for g, w in ((grads.dq, q64), (grads.dk, k64), (grads.dv, v64))]
        row.max_abs_err = max(errs)
        # relative to the gradient's scale, like the max-abs check (ALiBi/long rows give |grad| >> 1)
        row.rmse_err = max(_rmse(g, w.grad) / max(1.0, float(w.grad.abs().max()))
                           for g, w in ((grads.dq, q64), (grads.dk, k64), (grads.dv, v64)))
        if row.max_abs_err > tol["bwd"]:
            fail(f"grad rel err {row.max_abs_err:.3g} > {tol['bwd']:.3g} vs dense float64")
        if row.rmse_err > tol["bwd_rmse"]:
            fail(f"grad rmse {row.rmse_err:.3g} > {tol['bwd_rmse']:.3g} vs dense float64")
        if with_timing:
            row.median_ns = _median_ns(cfg.repeats, lambda: fa.backward(q, k, v, fwd, fwd.out, var.score, bm,
                                                                        cfg=acfg))
    elif mode in ("decode", "paged"):
        if kv_len < q_len:
            raise ConfigParse("decode mode: kv_len must be >= q_len")
        off = q_len - 1
        q_step = q[:, :, off:q_len].contiguous()
        bm_step = fa.create_block_mask(fa.offset_mask(var.mask, off), 1, 1, 1, kv_len, bs, bs, device=dev)
        row.density = fa.sparsity(bm_step).density
        if mode == "decode":
            call = lambda: fa.decode(q_step, k, v, off, var.mask, var.score, bm_step, acfg)  # noqa: E731
        elif cfg.dtype != torch.bfloat16:
            raise ConfigParse("paged mode: the paged cache is bf16 (use dtype = bf16)")
        else:
            ps = cfg.page_size or bs
            pages = cfg.batch * (-(-kv_len // ps)) + cfg.batch
            cache = fa.PagedKVCache(cfg.batch, pages, ps, cfg.kv_heads, cfg.dim, dtype=cfg.dtype, device=dev)
            cache.shuffle_free_pages(seed ^ 0xFA6E5)
            for b in range(cfg.batch):
                cache.assign(b, k[b:b + 1], v[b:b + 1])
            pt = cache.page_table()
            pbm = fa.convert_block_mask(bm_step, pt)
            pmask = var.mask
            if var.doc_ids is not None:  # the id table must span the logical page range
                pmask = fa.document_mask(np.pad(var.doc_ids, (0, max(0, pages * ps - len(var.doc_ids))), "edge"))
            call = lambda: fa.decode(q_step, cache.k_phys(), cache.v_phys(), off, pmask, var.score,  # noqa: E731
                                     pbm, acfg, page_table=pt)
        got = call()
        want, _ = _dense_forward(q_step, k, v, var, scale, G, q_pos=torch.tensor([off], device=dev))
        row.madds = 2 * cfg.dim * int(var.dense(torch.tensor([off], device=dev), ki).sum()) * cfg.batch * cfg.q_heads
        row.max_abs_err = float((got.out.double() - want).abs().max())
        row.rmse_err = _rmse(got.out, want)
        if row.max_abs_err > tol["decode"]:
            fail(f"decode step differs from the dense row by {row.max_abs_err:.3g} > {tol['decode']:.3g}")
        if with_timing:
            row.median_ns = _median_ns(cfg.repeats, call)
    else:
        raise ConfigParse(f"unknown mode '{mode}'")
    return row


def run_bench(cfg: BenchConfig, with_timing: bool = True, device="cuda") -> List[BenchRow]:
    """run_bench (bench.cpp:596-612): variant, mode, q_len, kv_len, block size order."""
    rows, idx = [], 0
    for var in cfg.variants:
        for mode in cfg.modes:
            for ql in cfg.q_lens:
                for kl in (cfg.kv_lens or [ql]):
                    for bs in cfg.block_sizes:
                        rows.append(run_point(cfg, var, mode, ql, kl, bs, idx, with_timing, device))
                        idx += 1
    return rows


def _csv_escape(s: str) -> str:
    return s if ("," not in s and '"' not in s) else '"' + s.replace('"', '""') + '"'


def to_csv(rows: List[BenchRow], with_timing: bool = True) -> str:
    """to_csv (bench.cpp:615-653): %.9g floats, median_ns 0 without timing."""
    out = [CSV_HEADER]
    for r in rows:
        out.append(",".join([_csv_escape(r.variant), str(r.batch), str(r.q_heads), str(r.kv_heads), str(r.q_len),
                             str(r.kv_len), str(r.dim), str(r.block_size), r.mode,
                             str(r.median_ns if with_timing else 0), str(r.madds), f"{r.density:.9g}",
                             f"{r.max_abs_err:.9g}", f"{r.rmse_err:.9g}"]))
    return "\n".join(out) + "\n"


_VERIFY_VARIANTS = ["noop", "causal", "sliding_window(100)", "document(4)", "prefix_lm(64)", "alibi",
                    "soft_cap(20)", "na_naive(5)", "na_tiled(5,4)", "na_morton(5)"]
# float32 (CUDA-core paths, the reference's tolerances) and bf16 (tcgen05 paths, paged decode)
VERIFY_GRIDS = [
    BenchConfig(variants=_VERIFY_VARIANTS, batch=1, q_heads=4, kv_heads=2, dim=64, q_lens=[256],
                block_sizes=[64, 128], modes=["forward", "backward", "decode"], repeats=3, dtype=torch.float32),
    BenchConfig(variants=_VERIFY_VARIANTS, batch=2, q_heads=4, kv_heads=2, dim=128, q_lens=[256],
                block_sizes=[128], modes=["forward", "backward", "decode", "paged"], repeats=3,
                dtype=torch.bfloat16),
]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--config")
    r.add_argument("--variant", default="causal")
    r.add_argument("--qlen", type=int, nargs="+", default=[1024])
    r.add_argument("--kvlen", type=int, nargs="*", default=[])
    r.add_argument("--bs", type=int, nargs="+", default=[128])
    r.add_argument("--mode", nargs="+", default=["forward"])
    r.add_argument("--batch", type=int, default=1)
    r.add_argument("--heads", type=int, default=4)
    r.add_argument("--kv-heads", type=int, default=0)
    r.add_argument("--dim", type=int, default=64)
    r.add_argument("--dtype", default="float32", choices=["float32", "bf16"])
    r.add_argument("--no-timing", action="store_true")
    r.add_argument("--out")
    sub.add_parser("verify")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "verify":
            rows = [r for g in VERIFY_GRIDS for r in run_bench(g, with_timing=False)]
            bad = [x for x in rows if not x.ok]
            for x in rows:
                print(f"{'PASS' if x.ok else 'FAIL'} {x.variant} {x.mode} bs={x.block_size} "
                      f"err={x.max_abs_err:.3g} {x.detail}")
            return 2 if bad else 0
        if a.config:
            cfg = load_config(a.config)
        else:
            cfg = BenchConfig(variants=_split_top(a.variant), batch=a.batch, q_heads=a.heads,
                              kv_heads=a.kv_heads or a.heads, dim=a.dim, q_lens=a.qlen, kv_lens=a.kvlen,
                              block_sizes=a.bs, modes=a.mode,
                              dtype=torch.bfloat16 if a.dtype == "bf16" else torch.float32)
            cfg.validate()
        rows = run_bench(cfg, with_timing=not a.no_timing)
        text = to_csv(rows, with_timing=not a.no_timing)
        if a.out:
            open(a.out, "w").write(text)
        else:
            sys.stdout.write(text)
        return 2 if any(not x.ok for x in rows) else 0
    except fa.Error as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
