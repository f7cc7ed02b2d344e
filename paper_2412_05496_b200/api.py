"""Host-side mirror of the reference ``blockattn`` API over the sm_100a C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/blockattn/*.hpp so the parity tests read like the
reference's own tests. Device memory, streams and dtypes come from PyTorch
(plumbing only); every computation is one of this package's CUDA kernels,
reached through ``libflexattn_b200.so``. There is no CPU path.

    create_block_mask   block_mask.hpp:109-110   -> fa_create_block_mask
    transpose           block_mask.hpp:115       -> (q-side arrays, fa_transpose_block_mask)
    forward             engine.hpp:68-71         -> fa_flex_fwd
    backward            engine.hpp:78-82         -> fa_flex_bwd
    decode              engine.hpp:92-96         -> fa_flex_decode
    PagedKVCache        paged_kv.hpp:50-89       -> fa_page_pool_* (allocator + K/V on the device)
    convert_block_mask  paged_kv.hpp:101         -> fa_convert_block_mask
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import (FA_BF16, FA_F32, FA_FLAG_DETERMINISTIC, FA_FLAG_VALIDATE, BlockMaskC, BwdArgs,
                   DecodeArgs, FwdArgs, MaskDesc, OpCountersC, PagePoolC, PageTableC, ScoreDesc, TensorC,
                   FA_FLAG_NO_SYNC, PAGE_ASSIGN, PAGE_APPEND, PAGE_ERASE)

# ---------------------------------------------------------------- errors (errors.hpp:11-101)


class Error(RuntimeError):
    """blockattn::Error."""


class ShapeMismatch(Error): pass
class NonFiniteInput(Error): pass
class IndexOutOfRange(Error): pass
class NonPositiveCap(Error): pass
class GeometryMismatch(Error): pass
class BlockMaskMismatch(Error): pass
class StaleStatistics(Error): pass
class OffsetOutOfRange(Error): pass
class OutOfPages(Error): pass
class UnmappedBlock(Error): pass
class UnmappedPhysicalIndex(Error): pass
class CudaError(Error): pass
class Unsupported(Error): pass


_STATUS = {1: ShapeMismatch, 2: NonFiniteInput, 3: IndexOutOfRange, 4: NonPositiveCap,
           5: GeometryMismatch, 6: BlockMaskMismatch, 7: StaleStatistics, 8: OffsetOutOfRange,
           9: OutOfPages, 10: UnmappedBlock, 11: UnmappedPhysicalIndex, 100: CudaError,
           101: Unsupported}


def _check(status: int) -> None:
    if status != 0:
        lib = _lib.load()
        msg = lib.fa_last_error().decode(errors="replace")
        raise _STATUS.get(status, Error)(msg or lib.fa_status_name(status).decode())


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# ---------------------------------------------------------------- modifiers (mask_library.hpp)
MASK_CAUSAL, MASK_SLIDING, MASK_DOCUMENT, MASK_PREFIX, MASK_HASH, MASK_NEVER = 1, 2, 4, 8, 16, 32
MASK_NATTEN = 64
SCORE_ALIBI, SCORE_SOFT_CAP = 1, 2


@dataclass(frozen=True)
class MaskMod:
    """A mask_mod: AND of primitive terms (and_mask), optionally ORed with a second term group
    (or_mask) and evaluated on permuted positions (remap_mask), with an optional q offset."""
    terms: int = 0
    window: int = 0
    prefix: int = 0
    q_offset: int = 0
    hash_seed: int = 0
    hash_density: int = 128
    doc_ids: Optional[torch.Tensor] = field(default=None, compare=False)
    or_terms: int = 0
    na_height: int = 0
    na_width: int = 0
    na_kernel: int = 0
    remap: Optional[torch.Tensor] = field(default=None, compare=False)

    def desc(self, device) -> MaskDesc:
        d = MaskDesc()
        d.terms, d.window, d.prefix, d.q_offset = self.terms, self.window, self.prefix, self.q_offset
        d.hash_seed, d.hash_density = self.hash_seed, self.hash_density
        d.or_terms = self.or_terms
        d.na_height, d.na_width, d.na_kernel = self.na_height, self.na_width, self.na_kernel
        if self.doc_ids is not None:
            ids = _device_cache(self, "doc_ids", self.doc_ids, torch.int32, device)
            d.doc_ids = ids.data_ptr()
            d.doc_len = ids.numel()
        if self.remap is not None:
            rm = _device_cache(self, "remap", self.remap, torch.int32, device)
            d.remap = rm.data_ptr()
            d.remap_len = rm.numel()
            if self.terms == MASK_NATTEN and not self.or_terms and 0 < self.na_width < 65536 \
                    and self.na_height < 65536:
                # (row, col) of every slot's token: the kernels skip the per-position division
                t = torch.as_tensor(self.remap).to(torch.int64)
                rc = ((t // self.na_width) << 16) | (t % self.na_width)
                d.remap_rc = _device_cache(self, "remap_rc", rc, torch.int32, device).data_ptr()
        return d


@dataclass(frozen=True)
class ScoreMod:
    """A score_mod: soft_cap and/or alibi (composed as soft_cap(alibi(s)))."""
    terms: int = 0
    cap: float = 0.0
    slopes: Optional[Sequence[float]] = field(default=None, compare=False)
    q_offset: int = 0

    @property
    def identity(self) -> bool:
        return self.terms == 0

    def desc(self, device) -> ScoreDesc:
        d = ScoreDesc()
        d.terms, d.cap, d.q_offset = self.terms, float(self.cap), self.q_offset
        if self.slopes is not None:
            t = torch.as_tensor(list(self.slopes) if not torch.is_tensor(self.slopes) else self.slopes,
                                dtype=torch.float32)
            sl = _device_cache(self, "slopes", t, torch.float32, device)
            d.slopes = sl.data_ptr()
            d.num_slopes = sl.numel()
        return d


_CACHE: dict = {}


def _device_cache(owner, name, t, dtype, device):
    key = (id(owner), name, str(device))
    hit = _CACHE.get(key)
    if hit is not None and hit[0] is owner:
        return hit[1]
    dev = torch.as_tensor(t).to(device=device, dtype=dtype).contiguous()
    _CACHE[key] = (owner, dev)
    return dev


def noop_mask() -> MaskMod:
    return MaskMod()


def causal() -> MaskMod:
    """q >= kv (mask_library.cpp:13-15)."""
    return MaskMod(terms=MASK_CAUSAL)


def sliding_window(window: int) -> MaskMod:
    """q >= kv and q - kv <= window (mask_library.cpp:17-22)."""
    if window < 0:
        raise IndexOutOfRange(f"sliding_window: window must be >= 0, got {window}")
    return MaskMod(terms=MASK_SLIDING, window=int(window))


def document_mask(doc_ids) -> MaskMod:
    """ids[q] == ids[kv] (mask_library.cpp:24-34)."""
    return MaskMod(terms=MASK_DOCUMENT, doc_ids=torch.as_tensor(doc_ids).to(torch.int32))


def prefix_lm(prefix_len: int) -> MaskMod:
    """kv < prefix_len or q >= kv (mask_library.cpp:36-41)."""
    if prefix_len < 0:
        raise IndexOutOfRange(f"prefix_lm: prefix_len must be >= 0, got {prefix_len}")
    return MaskMod(terms=MASK_PREFIX, prefix=int(prefix_len))


def hash_mask(seed: int, density256: int = 128) -> MaskMod:
    """Test aid of the reference (tests/test_support.hpp:16-29)."""
    return MaskMod(terms=MASK_HASH, hash_seed=int(seed), hash_density=int(density256))


def never_mask() -> MaskMod:
    """Test aid of the reference (tests/test_support.hpp:31-35)."""
    return MaskMod(terms=MASK_NEVER)


def _merge_params(a: MaskMod, b: MaskMod, what: str) -> dict:
    if a.q_offset != b.q_offset:
        raise Unsupported(f"{what}: operands with different offsets")
    if a.remap is not None or b.remap is not None:
        raise Unsupported(f"{what}: remapped operands (apply remap_mask last)")
    for attr in ("window", "prefix", "hash_seed"):
        if getattr(a, attr) and getattr(b, attr) and getattr(a, attr) != getattr(b, attr):
            raise Unsupported(f"{what}: conflicting {attr}")
    if (a.terms | a.or_terms) & MASK_NATTEN and (b.terms | b.or_terms) & MASK_NATTEN and \
            (a.na_height, a.na_width, a.na_kernel) != (b.na_height, b.na_width, b.na_kernel):
        raise Unsupported(f"{what}: two different neighbourhood geometries")
    if a.doc_ids is not None and b.doc_ids is not None:
        raise Unsupported(f"{what}: two document masks")
    na = a if (a.terms | a.or_terms) & MASK_NATTEN else b
    hd = a.hash_density if (a.terms | a.or_terms) & MASK_HASH else b.hash_density
    return dict(window=a.window or b.window, prefix=a.prefix or b.prefix, q_offset=a.q_offset,
                hash_seed=a.hash_seed or b.hash_seed, hash_density=hd,
                doc_ids=a.doc_ids if a.doc_ids is not None else b.doc_ids,
                na_height=na.na_height, na_width=na.na_width, na_kernel=na.na_kernel)


def or_mask(a: MaskMod, b: MaskMod) -> MaskMod:
    """or_mask (mask_library.cpp:100-104) of two single-group masks: the device evaluates
    (AND of a's terms) OR (AND of b's terms) with shared parameters."""
    if a.or_terms or b.or_terms:
        raise Unsupported("or_mask: operands that are already OR-combinations")
    kw = _merge_params(a, b, "or_mask")
    if a.terms == 0 or b.terms == 0:  # or with noop_mask is noop_mask
        return MaskMod(**kw)
    return MaskMod(terms=a.terms, or_terms=b.terms, **kw)


@dataclass(frozen=True)
class NAGeometry:
    """Neighbourhood-attention canvas (mask_library.hpp NAGeometry, mask_library.cpp:121-135):
    tokens are the pixels of a height x width canvas in row-major order."""
    canvas_h: int
    canvas_w: int
    kernel: int

    def __post_init__(self):
        if self.canvas_h < 1 or self.canvas_w < 1:
            raise GeometryMismatch(f"NAGeometry: canvas dims must be >= 1, got {self.canvas_h}x{self.canvas_w}")
        if self.kernel < 1 or self.kernel % 2 == 0:
            raise GeometryMismatch(f"NAGeometry: kernel must be odd and >= 1, got {self.kernel}")
        if self.kernel > min(self.canvas_h, self.canvas_w):
            raise GeometryMismatch(f"NAGeometry: kernel {self.kernel} exceeds canvas "
                                   f"{self.canvas_h}x{self.canvas_w}")

    def tokens(self) -> int:
        return self.canvas_h * self.canvas_w


def na_naive(g: NAGeometry) -> MaskMod:
    """2-D neighbourhood attention: max(|dr|, |dc|) <= kernel // 2 (mask_library.cpp:137-149)."""
    return MaskMod(terms=MASK_NATTEN, na_height=g.canvas_h, na_width=g.canvas_w, na_kernel=g.kernel)


def tile_permutation(g: NAGeometry, tile: int) -> list:
    """Slot -> pixel table visiting tile x tile squares in row-major order, pixels row-major
    inside a tile (mask_library.cpp:164-181)."""
    if tile < 1 or g.canvas_h % tile or g.canvas_w % tile:
        raise GeometryMismatch(f"tile_permutation: tile {tile} must divide canvas {g.canvas_h}x{g.canvas_w}")
    return [r * g.canvas_w + c
            for tr in range(0, g.canvas_h, tile) for tc in range(0, g.canvas_w, tile)
            for r in range(tr, tr + tile) for c in range(tc, tc + tile)]


def morton_permutation(g: NAGeometry) -> list:
    """Slot -> pixel table in Z (Morton) order, column bits in the even positions
    (mask_library.cpp:183-201); square power-of-two canvases only."""
    n = g.canvas_h
    if g.canvas_h != g.canvas_w or n & (n - 1):
        raise GeometryMismatch(f"morton_permutation: canvas must be square with power-of-two side, "
                               f"got {g.canvas_h}x{g.canvas_w}")
    out = [0] * (n * n)
    for r in range(n):
        for c in range(n):
            slot, bit = 0, 0
            while (1 << bit) < n:
                slot |= ((c >> bit) & 1) << (2 * bit)
                slot |= ((r >> bit) & 1) << (2 * bit + 1)
                bit += 1
            out[slot] = r * n + c
    return out


def remap_mask(base: MaskMod, forward_table) -> MaskMod:
    """mask(q, kv) = base(fwd[q], fwd[kv]) (mask_library.cpp:203-215); the table must be a
    bijection on [0, len) (GeometryMismatch otherwise)."""
    fwd = [int(x) for x in forward_table]
    if sorted(fwd) != list(range(len(fwd))):
        raise GeometryMismatch(f"Permutation: forward is not a bijection on [0, {len(fwd)})")
    if base.remap is not None:
        raise Unsupported("remap_mask: base is already remapped")
    return replace(base, remap=torch.tensor(fwd, dtype=torch.int32))


def and_mask(a: MaskMod, b: MaskMod) -> MaskMod:
    """and_mask (mask_library.cpp:94-98) for masks expressible as one term set."""
    if a.or_terms or b.or_terms:
        raise Unsupported("and_mask: OR-combined operands")
    kw = _merge_params(a, b, "and_mask")
    return MaskMod(terms=a.terms | b.terms, **kw)


def offset_mask(m: MaskMod, offset: int) -> MaskMod:
    """q -> q + offset (mask_library.cpp:106-110)."""
    return replace(m, q_offset=m.q_offset + int(offset))


def noop_score() -> ScoreMod:
    return ScoreMod()


def alibi_slopes(heads: int) -> list:
    """-2^(-8(h+1)/H) (mask_library.cpp:71-81)."""
    if heads < 1:
        raise IndexOutOfRange(f"alibi_slopes: heads must be >= 1, got {heads}")
    return [-(2.0 ** (-8.0 * (h + 1) / heads)) for h in range(heads)]


def alibi(slopes) -> ScoreMod:
    """s + slopes[h] * (q - kv) (mask_library.cpp:53-69)."""
    return ScoreMod(terms=SCORE_ALIBI, slopes=list(map(float, slopes)))


def soft_cap(cap: float) -> ScoreMod:
    """cap * tanh(s / cap) (mask_library.cpp:83-92)."""
    if not (cap > 0.0) or not math.isfinite(cap):
        raise NonPositiveCap(f"soft_cap: cap must be finite and > 0, got {cap}")
    return ScoreMod(terms=SCORE_SOFT_CAP, cap=float(cap))


def compose(outer: ScoreMod, inner: ScoreMod) -> ScoreMod:
    """outer(inner(s)) (modifiers.hpp:57-66); supported: soft_cap(alibi(s)) and identities."""
    if outer.identity:
        return inner
    if inner.identity:
        return outer
    if outer.terms == SCORE_SOFT_CAP and inner.terms == SCORE_ALIBI and outer.q_offset == inner.q_offset:
        return ScoreMod(terms=SCORE_ALIBI | SCORE_SOFT_CAP, cap=outer.cap, slopes=inner.slopes,
                        q_offset=inner.q_offset)
    raise Unsupported("compose: only soft_cap(alibi(s)) is compiled")


def offset_score(s: ScoreMod, offset: int) -> ScoreMod:
    """q -> q + offset (mask_library.cpp:112-119)."""
    return replace(s, q_offset=s.q_offset + int(offset))


# ---------------------------------------------------------------- config (config.hpp:16-45)
@dataclass
class AttentionConfig:
    scale: Optional[float] = None
    gqa_group: int = 1
    block_size_q: int = 128
    block_size_kv: int = 128

    def effective_scale(self, head_dim: int) -> float:
        return self.scale if self.scale is not None else 1.0 / math.sqrt(head_dim)

    def validate(self):
        if self.scale is not None and not (math.isfinite(self.scale) and self.scale > 0):
            raise ShapeMismatch("AttentionConfig: scale must be finite and positive")
        if self.gqa_group < 1:
            raise ShapeMismatch(f"AttentionConfig: gqa_group must be >= 1, got {self.gqa_group}")
        if self.block_size_q < 1 or self.block_size_kv < 1:
            raise ShapeMismatch("AttentionConfig: block sizes must be >= 1")


# ---------------------------------------------------------------- BlockMask (block_mask.hpp:35-79)
@dataclass
class BlockMask:
    """Device BlockMask: FlexAttention names over the reference layout.

    kv_num_blocks == partial_num, kv_indices == partial_idx, full_kv_* == full_*;
    q_* arrays are the same fields of transpose(bm). int32 on the device.
    ``mask`` is the runtime mask (the reference's runtime_mask minus bounds,
    which the kernels apply from q_len/kv_len).
    """
    b_dims: int
    h_dims: int
    rows: int
    cols: int
    bs_q: int
    bs_kv: int
    q_len: int
    kv_len: int
    kv_num_blocks: torch.Tensor
    kv_indices: torch.Tensor
    full_kv_num_blocks: torch.Tensor
    full_kv_indices: torch.Tensor
    q_num_blocks: Optional[torch.Tensor] = None
    q_indices: Optional[torch.Tensor] = None
    full_q_num_blocks: Optional[torch.Tensor] = None
    full_q_indices: Optional[torch.Tensor] = None
    mask: Optional[MaskMod] = None

    # reference-style accessors
    @property
    def partial_num(self): return self.kv_num_blocks
    @property
    def partial_idx(self): return self.kv_indices
    @property
    def full_num(self): return self.full_kv_num_blocks
    @property
    def full_idx(self): return self.full_kv_indices

    def has_runtime_mask(self) -> bool:
        return self.mask is not None

    def c(self) -> BlockMaskC:
        s = BlockMaskC()
        s.b_dims, s.h_dims, s.rows, s.cols = self.b_dims, self.h_dims, self.rows, self.cols
        s.bs_q, s.bs_kv, s.q_len, s.kv_len = self.bs_q, self.bs_kv, self.q_len, self.kv_len
        for name in ("kv_num_blocks", "kv_indices", "full_kv_num_blocks", "full_kv_indices",
                     "q_num_blocks", "q_indices", "full_q_num_blocks", "full_q_indices"):
            t = getattr(self, name)
            setattr(s, name, t.data_ptr() if t is not None else None)
        return s

    def with_mask(self, user_mask: MaskMod) -> "BlockMask":
        return replace(self, mask=user_mask)

    @property
    def device(self):
        return self.kv_num_blocks.device


def _geometry(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv):
    lib = _lib.load()
    rows, cols, ws = C.c_int64(), C.c_int64(), C.c_size_t()
    _check(lib.fa_block_mask_geometry(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv,
                                      C.byref(rows), C.byref(cols), C.byref(ws)))
    return rows.value, cols.value, ws.value


def create_block_mask(mask: MaskMod, b_dims: int, h_dims: int, q_len: int, kv_len: int,
                      bs_q: int = 128, bs_kv: int = 128, device="cuda", q_side: bool = True) -> BlockMask:
    """create_block_mask (block_mask.cpp:79-115) + transpose, on the GPU."""
    if mask is None:
        raise ShapeMismatch("create_block_mask: mask has no callable")
    rows, cols, ws = _geometry(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv)
    dev = torch.device(device)
    i32 = dict(dtype=torch.int32, device=dev)
    n = b_dims * h_dims
    bm = BlockMask(b_dims, h_dims, rows, cols, bs_q, bs_kv, q_len, kv_len,
                   torch.empty(n * rows, **i32), torch.empty(n * rows * cols, **i32),
                   torch.empty(n * rows, **i32), torch.empty(n * rows * cols, **i32), mask=mask)
    if q_side:
        bm.q_num_blocks = torch.empty(n * cols, **i32)
        bm.q_indices = torch.empty(n * cols * rows, **i32)
        bm.full_q_num_blocks = torch.empty(n * cols, **i32)
        bm.full_q_indices = torch.empty(n * cols * rows, **i32)
    work = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev)
    cbm = bm.c()
    md = mask.desc(dev)
    with torch.cuda.device(dev):
        _check(_lib.load().fa_create_block_mask(C.byref(md), b_dims, h_dims, q_len, kv_len, bs_q, bs_kv,
                                                C.byref(cbm), C.c_void_p(work.data_ptr()), ws,
                                                C.c_void_p(_stream())))
    bm._work = work  # keep alive until the stream consumed it
    return bm


def transpose(bm: BlockMask) -> BlockMask:
    """transpose (block_mask.cpp:161-178): q/kv roles swapped, same device arrays reused."""
    if bm.q_num_blocks is None:
        dev = bm.device
        i32 = dict(dtype=torch.int32, device=dev)
        n = bm.b_dims * bm.h_dims
        bm.q_num_blocks = torch.empty(n * bm.cols, **i32)
        bm.q_indices = torch.empty(n * bm.cols * bm.rows, **i32)
        bm.full_q_num_blocks = torch.empty(n * bm.cols, **i32)
        bm.full_q_indices = torch.empty(n * bm.cols * bm.rows, **i32)
        ws = n * bm.rows * bm.cols
        work = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev)
        cbm = bm.c()
        _check(_lib.load().fa_transpose_block_mask(C.byref(cbm), C.c_void_p(work.data_ptr()), ws,
                                                   C.c_void_p(_stream())))
        bm._work_t = work
    t = BlockMask(bm.b_dims, bm.h_dims, bm.cols, bm.rows, bm.bs_kv, bm.bs_q, bm.kv_len, bm.q_len,
                  bm.q_num_blocks, bm.q_indices, bm.full_q_num_blocks, bm.full_q_indices,
                  bm.kv_num_blocks, bm.kv_indices, bm.full_kv_num_blocks, bm.full_kv_indices,
                  mask=None)
    return t


@dataclass
class SparsityReport:
    total_blocks: int
    full_blocks: int
    partial_blocks: int
    empty_blocks: int
    density: float


def sparsity(bm: BlockMask) -> SparsityReport:
    """sparsity (block_mask.cpp:180-191)."""
    total = bm.b_dims * bm.h_dims * bm.rows * bm.cols
    part = int(bm.kv_num_blocks.sum().item())
    full = int(bm.full_kv_num_blocks.sum().item())
    return SparsityReport(total, full, part, total - part - full,
                          0.0 if total == 0 else (part + full) / total)


# ---------------------------------------------------------------- tensors
def _tensor(t: torch.Tensor, name: str) -> TensorC:
    if t.dim() != 4:
        raise ShapeMismatch(f"{name}: expected a (B, H, L, D) tensor, got {tuple(t.shape)}")
    if not t.is_cuda:
        raise Unsupported(f"{name}: tensors must live on a CUDA device (no CPU path)")
    if not t.is_contiguous():
        raise ShapeMismatch(f"{name}: tensor must be contiguous")
    if t.dtype == torch.bfloat16:
        dt = FA_BF16
    elif t.dtype == torch.float32:
        dt = FA_F32
    else:
        raise Unsupported(f"{name}: dtype {t.dtype} (bf16 or fp32 only)")
    s = TensorC()
    s.data, s.dtype = t.data_ptr(), dt
    s.b, s.h, s.l, s.d = t.shape
    return s


def _scale(cfg: AttentionConfig) -> float:
    return float(cfg.scale) if cfg.scale is not None else 0.0


@dataclass
class OpCounters:
    """OpCounters (engine.hpp:21-32), computed on the device from the BlockMask and the mask:
    mask_evals and score_evals exactly as the reference counts them; madds without the
    data-dependent accumulator-rescale term (see fa_op_counters in include/flexattn_b200.h).
    Calls add into it, like the reference's ``*counters += worker counters``."""
    madds: int = 0
    mask_evals: int = 0
    score_evals: int = 0

    def _add(self, c: OpCountersC):
        self.madds += int(c.madds)
        self.mask_evals += int(c.mask_evals)
        self.score_evals += int(c.score_evals)


def check_finite(*named_tensors) -> None:
    """validate_inputs' finiteness scan (validate.hpp:36-38) on the device: raises NonFiniteInput
    naming the first tensor holding NaN/inf. ``named_tensors`` are (name, tensor) pairs."""
    n = len(named_tensors)
    arr = (TensorC * max(n, 1))()
    names = (C.c_char_p * max(n, 1))()
    for i, (name, t) in enumerate(named_tensors):
        arr[i] = _tensor(t, name)
        names[i] = name.encode()
    with torch.cuda.device(named_tensors[0][1].device if n else torch.cuda.current_device()):
        _check(_lib.load().fa_check_finite(arr, names, n, C.c_void_p(_stream())))


@dataclass
class AttentionOutput:
    """engine.hpp:38-46: out (B,H,L,D) and lse (B,H,L) natural log."""
    out: torch.Tensor
    lse: torch.Tensor


@dataclass
class Gradients:
    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor


def _prep_mods(smod: ScoreMod, bm: BlockMask, mask: Optional[MaskMod]):
    if smod is None:
        raise BlockMaskMismatch("forward: score modifier has no callable")
    m = mask if mask is not None else bm.mask
    if m is None:
        raise BlockMaskMismatch("forward: block mask has no runtime mask attached")
    return m


def forward(q, k, v, smod: ScoreMod, bm: BlockMask, cfg: Optional[AttentionConfig] = None,
            mask: Optional[MaskMod] = None, out: Optional[torch.Tensor] = None,
            lse: Optional[torch.Tensor] = None, counters: Optional[OpCounters] = None,
            validate: bool = False) -> AttentionOutput:
    """forward<Real> (engine.cpp:46-172) on the GPU: bf16 -> tcgen05 kernel (bs 128,
    D 64/128), otherwise the fp32 CUDA-core kernel. ``counters`` (OpCounters) and
    ``validate=True`` (the reference's NaN/inf scan of q/k/v -> NonFiniteInput) each cost a
    device pass and a stream synchronisation."""
    cfg = cfg or AttentionConfig()
    cfg.validate()
    m = _prep_mods(smod, bm, mask)
    if bm.bs_q != cfg.block_size_q or bm.bs_kv != cfg.block_size_kv:
        raise BlockMaskMismatch(f"block mask block sizes ({bm.bs_q},{bm.bs_kv}) disagree with config "
                                f"({cfg.block_size_q},{cfg.block_size_kv})")
    out = torch.empty_like(q) if out is None else out
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device) if lse is None else lse
    a = FwdArgs()
    a.q, a.k, a.v, a.out = _tensor(q, "q"), _tensor(k, "k"), _tensor(v, "v"), _tensor(out, "out")
    a.lse = lse.data_ptr()
    cbm = bm.c()
    a.bm = C.pointer(cbm)
    a.mask, a.score = m.desc(q.device), smod.desc(q.device)
    a.scale, a.gqa_group = _scale(cfg), cfg.gqa_group
    a.flags = FA_FLAG_VALIDATE if validate else 0
    cc = OpCountersC()
    if counters is not None:
        a.counters = C.pointer(cc)
    with torch.cuda.device(q.device):
        _check(_lib.load().fa_flex_fwd(C.byref(a), C.c_void_p(_stream())))
    if counters is not None:
        counters._add(cc)
    return AttentionOutput(out, lse)


def backward(q, k, v, fwd: AttentionOutput, d_out, smod: ScoreMod, bm: BlockMask,
             bm_t: Optional[BlockMask] = None, cfg: Optional[AttentionConfig] = None,
             mask: Optional[MaskMod] = None, counters: Optional[OpCounters] = None,
             validate: bool = False, deterministic: bool = False, phase_events=None) -> Gradients:
    """backward<Real> (engine.cpp:174-401): dQ/dK/dV through score_mod'. ``bm_t`` is
    accepted for signature parity; the q-side arrays live in ``bm``. ``deterministic=True``
    runs the split backward (dK/dV kernel + a dQ pass accumulating in TMEM in one fixed kv
    order, engine.cpp:237-305), so the gradients are bitwise reproducible run to run (the
    default fused tensor-core kernel adds fp32 dQ partial sums in arrival order; dK/dV are
    reproducible either way). Measured on B200 at 1.2-1.5x the default's time.
    ``phase_events``: optional 4 torch.cuda.Event recorded around the kernels (timing)."""
    cfg = cfg or AttentionConfig()
    cfg.validate()
    m = _prep_mods(smod, bm, mask)
    if bm.q_num_blocks is None:
        transpose(bm)
    if bm_t is not None and (bm_t.rows != bm.cols or bm_t.cols != bm.rows):
        raise BlockMaskMismatch("backward: bm_t is not the transpose of bm")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    lib = _lib.load()
    B, H, L, D = q.shape
    ws = lib.fa_bwd_workspace_size(B, H, L, D)
    work = _workspace(q.device, ws)
    a = BwdArgs()
    a.q, a.k, a.v = _tensor(q, "q"), _tensor(k, "k"), _tensor(v, "v")
    a.out, a.d_out = _tensor(fwd.out, "out"), _tensor(d_out, "d_out")
    if fwd.lse.numel() != B * H * L:
        raise StaleStatistics("backward: saved forward statistics do not match these tensors")
    a.lse = fwd.lse.data_ptr()
    a.dq, a.dk, a.dv = _tensor(dq, "dq"), _tensor(dk, "dk"), _tensor(dv, "dv")
    cbm = bm.c()
    a.bm = C.pointer(cbm)
    a.mask, a.score = m.desc(q.device), smod.desc(q.device)
    a.scale, a.gqa_group = _scale(cfg), cfg.gqa_group
    a.workspace, a.workspace_bytes = work.data_ptr(), ws
    a.flags = (FA_FLAG_VALIDATE if validate else 0) | (FA_FLAG_DETERMINISTIC if deterministic else 0)
    cc = OpCountersC()
    if counters is not None:
        a.counters = C.pointer(cc)
    if phase_events is not None:
        for i, ev in enumerate(phase_events):
            if not ev.cuda_event:  # torch creates its events lazily, on the first record
                ev.record()
            a.phase_events[i] = ev.cuda_event
    with torch.cuda.device(q.device):
        _check(lib.fa_flex_bwd(C.byref(a), C.c_void_p(_stream())))
    if counters is not None:
        counters._add(cc)
    return Gradients(dq, dk, dv)


_WS: dict = {}


def _workspace(device, nbytes) -> torch.Tensor:
    key = str(device)
    w = _WS.get(key)
    if w is None or w.numel() < nbytes:
        w = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = w
    return w


def decode(q_step, k_cache, v_cache, offset: int, mask: MaskMod, smod: ScoreMod, bm: BlockMask,
           cfg: Optional[AttentionConfig] = None, page_table: Optional["PageTable"] = None,
           num_splits: int = 0, counters: Optional[OpCounters] = None,
           validate: bool = False) -> AttentionOutput:
    """decode (engine.cpp:403-427): q_step rows sit at [offset, offset+n_new). ``mask``/``smod``
    speak absolute positions; ``bm`` describes the shifted mask at q_len = n_new (converted to
    physical pages when ``page_table`` is given)."""
    cfg = cfg or AttentionConfig()
    cfg.validate()
    if mask is None:
        raise BlockMaskMismatch("decode: mask has no callable")
    if smod is None:
        raise BlockMaskMismatch("decode: score modifier has no callable")
    out = torch.empty_like(q_step)
    B, H, n_new, D = q_step.shape
    lse = torch.empty((B, H, n_new), dtype=torch.float32, device=q_step.device)
    lib = _lib.load()
    ws = lib.fa_decode_workspace_size(B, H, n_new, D, num_splits)
    work = _workspace(q_step.device, ws)
    a = DecodeArgs()
    a.q, a.k_cache, a.v_cache = _tensor(q_step, "q"), _tensor(k_cache, "k_cache"), _tensor(v_cache, "v_cache")
    a.out = _tensor(out, "out")
    a.lse = lse.data_ptr()
    cbm = bm.c()
    a.bm = C.pointer(cbm)
    if page_table is not None:
        cpt = page_table.c()
        a.pt = C.pointer(cpt)
    a.offset = int(offset)
    a.mask, a.score = mask.desc(q_step.device), smod.desc(q_step.device)
    a.scale, a.gqa_group = _scale(cfg), cfg.gqa_group
    a.num_splits = int(num_splits)
    a.workspace, a.workspace_bytes = work.data_ptr(), ws
    a.flags = FA_FLAG_VALIDATE if validate else 0
    cc = OpCountersC()
    if counters is not None:
        a.counters = C.pointer(cc)
    with torch.cuda.device(q_step.device):
        _check(lib.fa_flex_decode(C.byref(a), C.c_void_p(_stream())))
    if counters is not None:
        counters._add(cc)
    return AttentionOutput(out, lse)


def flex_attention(query, key, value, score_mod: Optional[ScoreMod] = None,
                   block_mask: Optional[BlockMask] = None, scale: Optional[float] = None,
                   enable_gqa: bool = False, return_lse: bool = False):
    """FlexAttention-style entry point (the north-star signature): forward over a BlockMask."""
    if block_mask is None:
        block_mask = create_block_mask(noop_mask(), 1, 1, query.shape[2], key.shape[2],
                                       device=query.device)
    g = query.shape[1] // key.shape[1]
    if g != 1 and not enable_gqa:
        raise ShapeMismatch("flex_attention: q/kv head counts differ; pass enable_gqa=True")
    cfg = AttentionConfig(scale=scale, gqa_group=g, block_size_q=block_mask.bs_q,
                          block_size_kv=block_mask.bs_kv)
    res = forward(query, key, value, score_mod or noop_score(), block_mask, cfg)
    return (res.out, res.lse) if return_lse else res.out


# ---------------------------------------------------------------- synthetic inputs
def random_tensor(seed: int, shape, dtype=torch.bfloat16, device="cuda", first: int = 0) -> torch.Tensor:
    """random_tensor (random.hpp:41-46) generated on the device (bf16: RNE-rounded)."""
    t = torch.empty(shape, dtype=dtype, device=device)
    dt = FA_BF16 if dtype == torch.bfloat16 else FA_F32
    with torch.cuda.device(t.device):
        _check(_lib.load().fa_fill_uniform(C.c_void_p(t.data_ptr()), dt, C.c_uint64(seed & (2**64 - 1)),
                                           first, t.numel(), C.c_void_p(_stream())))
    return t


# ---------------------------------------------------------------- paged KV (paged_kv.hpp)
@dataclass
class PageTable:
    """PageTable (paged_kv.hpp:18-41), host copy plus device mirrors for the kernels."""
    batches: int
    max_logical_pages: int
    num_physical_pages: int
    page_size: int
    table: list
    phys_to_logical: list
    owner: list
    seq_len: list
    _dev: dict = field(default_factory=dict, repr=False)

    def lookup(self, b, logical_page):
        return self.table[b * self.max_logical_pages + logical_page]

    def device_arrays(self, device):
        key = str(device)
        if key not in self._dev:
            i32 = dict(dtype=torch.int32, device=device)
            self._dev[key] = (torch.tensor(self.table, **i32), torch.tensor(self.phys_to_logical, **i32),
                              torch.tensor(self.owner, **i32), torch.tensor(self.seq_len, **i32))
        return self._dev[key]

    def c(self, device="cuda") -> PageTableC:
        t, p2l, own, sl = self.device_arrays(torch.device(device))
        s = PageTableC()
        s.batches, s.max_logical_pages = self.batches, self.max_logical_pages
        s.num_physical_pages, s.page_size = self.num_physical_pages, self.page_size
        s.table, s.phys_to_logical, s.owner, s.seq_len = (t.data_ptr(), p2l.data_ptr(),
                                                           own.data_ptr(), sl.data_ptr())
        s.max_seq_len = max(self.seq_len) if self.seq_len else 0
        return s


class DevicePageTable:
    """Live view of a device page pool as a PageTable (paged_kv.hpp:18-41): the kernels read the
    pool's own arrays (no upload); the host lists are downloaded on access."""

    def __init__(self, cache: "PagedKVCache", max_seq_len: Optional[int] = None):
        self._cache = cache
        self._max_seq_len = max_seq_len
        self.batches = cache.batches
        self.max_logical_pages = cache.num_pages
        self.num_physical_pages = cache.num_pages
        self.page_size = cache.ps

    def _arr(self, name):
        return self._cache._view(name).cpu().tolist()

    @property
    def table(self):
        return self._arr("table")

    @property
    def phys_to_logical(self):
        return self._arr("phys_to_logical")

    @property
    def owner(self):
        return self._arr("owner")

    @property
    def seq_len(self):
        return self._arr("seq_len")

    def lookup(self, b, logical_page):
        return int(self._cache._view("table")[b * self.max_logical_pages + logical_page].item())

    def c(self, device=None) -> PageTableC:
        s = _lib.load().fa_page_pool_table(C.byref(self._cache._pool))
        s.max_seq_len = self._max_seq_len if self._max_seq_len is not None else self._cache._max_seq_len()
        return s


class PagedKVCache:
    """PagedKVCache (paged_kv.hpp:50-89) with the page allocator ON THE DEVICE (fa_page_pool:
    LIFO free stack with page 0 on top, deterministic shuffle, capacity-checked assign / append,
    erase; paged_kv.cpp:13-152) and device K/V of shape (1, kv_heads, num_pages * page_size, dim).
    Single-sequence calls mirror the reference; the ``*_batch`` calls apply many requests in
    order in one launch (one sequence per request), with ``sync=False`` for CUDA-graph serving
    loops (the outcome stays on the device until ``status()``)."""

    def __init__(self, batches, num_pages, page_size, kv_heads, dim, dtype=torch.bfloat16,
                 device="cuda"):
        if batches < 1 or num_pages < 1 or page_size < 1:
            raise ShapeMismatch("PagedKVCache: batches, num_pages and page_size must be >= 1")
        self.batches, self.num_pages, self.ps = batches, num_pages, page_size
        self.kv_heads, self.dim = kv_heads, dim
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        lib = _lib.load()
        nbytes = lib.fa_page_pool_bytes(batches, num_pages)
        self._mem = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self._pool = PagePoolC()
        with torch.cuda.device(self.device):
            _check(lib.fa_page_pool_init(C.byref(self._pool), C.c_void_p(self._mem.data_ptr()), nbytes,
                                         batches, num_pages, page_size, C.c_void_p(_stream())))
        self.k = torch.zeros((1, kv_heads, num_pages * page_size, dim), dtype=dtype, device=self.device)
        self.v = torch.zeros_like(self.k)
        self._seq_host = [0] * batches  # mirror kept by the synchronous calls
        self._host_valid = True

    # -- device state ------------------------------------------------------------------------
    def _view(self, name):
        ptr = getattr(self._pool, name)
        n = {"table": self.batches * self.num_pages, "phys_to_logical": self.num_pages,
             "owner": self.num_pages, "seq_len": self.batches, "free_stack": self.num_pages,
             "free_count": 1}[name]
        off = (ptr - self._mem.data_ptr()) // 4
        return self._mem.view(torch.int32)[off:off + n]

    def _max_seq_len(self):
        if not self._host_valid:
            self._seq_host = self._view("seq_len").cpu().tolist()
            self._host_valid = True
        return max(self._seq_host) if self._seq_host else 0

    def page_table(self, max_seq_len: Optional[int] = None) -> DevicePageTable:
        """The live device page table. ``max_seq_len`` (an upper bound of the sequence lengths,
        for the mask's range checks) avoids reading the lengths back after ``sync=False``
        updates."""
        return DevicePageTable(self, max_seq_len)

    def shuffle_free_pages(self, seed: int):
        """shuffle_free_pages (paged_kv.cpp:143-146) of the device free stack."""
        with torch.cuda.device(self.device):
            _check(_lib.load().fa_page_pool_shuffle(C.byref(self._pool), C.c_uint64(seed & (2**64 - 1)),
                                                    C.c_void_p(_stream())))

    def _check_tokens(self, k_t, v_t):
        if tuple(k_t.shape) != tuple(v_t.shape):
            raise ShapeMismatch("PagedKVCache: k and v tokens must agree")
        if k_t.dim() != 4 or k_t.shape[0] != 1 or k_t.shape[1] != self.kv_heads or k_t.shape[3] != self.dim:
            raise ShapeMismatch(f"PagedKVCache: token tensors must be (1,{self.kv_heads},n,{self.dim})")

    def _update(self, op, batch_ids, n_tokens=None, k_t=None, v_t=None, sync=True):
        lib = _lib.load()
        n = len(batch_ids) if not torch.is_tensor(batch_ids) else batch_ids.numel()
        i32 = dict(dtype=torch.int32, device=self.device)
        ids = batch_ids.to(**i32) if torch.is_tensor(batch_ids) else torch.tensor(list(batch_ids), **i32)
        nt = None
        if op != PAGE_ERASE:
            nt = n_tokens.to(**i32) if torch.is_tensor(n_tokens) else torch.tensor(list(n_tokens), **i32)
        tk = tv = ck = cv = None
        if k_t is not None:
            self._check_tokens(k_t, v_t)
            k_t = k_t.to(device=self.device, dtype=self.k.dtype).contiguous()
            v_t = v_t.to(device=self.device, dtype=self.k.dtype).contiguous()
            tk, tv = C.byref(_tensor(k_t, "k_tokens")), C.byref(_tensor(v_t, "v_tokens"))
            ck, cv = C.byref(_tensor(self.k, "k_cache")), C.byref(_tensor(self.v, "v_cache"))
        with torch.cuda.device(self.device):
            st = C.c_void_p(_stream())
            _check(lib.fa_page_pool_update(C.byref(self._pool), op, C.c_void_p(ids.data_ptr() if n else 0),
                                           C.c_void_p(nt.data_ptr() if nt is not None and n else 0), n,
                                           tk, tv, ck, cv, FA_FLAG_NO_SYNC, st))
            if not sync:
                self._host_valid = False
                self._keep = (ids, nt, k_t, v_t)  # alive until the stream has consumed them
                return None
            applied = C.c_int32(0)
            rc = lib.fa_page_pool_status(C.byref(self._pool), C.byref(applied), st)
        # host mirror of the applied prefix (requests run in order)
        ids_h = ids.cpu().tolist()
        nt_h = nt.cpu().tolist() if nt is not None else None
        if self._host_valid:
            for i in range(applied.value):
                b = ids_h[i]
                self._seq_host[b] = (nt_h[i] if op == PAGE_ASSIGN else
                                     self._seq_host[b] + nt_h[i] if op == PAGE_APPEND else 0)
        _check(rc)
        return applied.value

    def status(self):
        """Outcome of the last update (synchronises): raises its error, else the applied count."""
        applied = C.c_int32(0)
        lib = _lib.load()
        with torch.cuda.device(self.device):
            rc = lib.fa_page_pool_status(C.byref(self._pool), C.byref(applied), C.c_void_p(_stream()))
        _check(rc)
        return applied.value

    # -- the reference's calls ---------------------------------------------------------------
    def _check_batch(self, b):
        if b < 0 or b >= self.batches:
            raise IndexOutOfRange(f"PagedKVCache: batch {b} outside [0, {self.batches})")

    def erase(self, b):
        """erase (paged_kv.cpp:128-141)."""
        self._update(PAGE_ERASE, [b])

    def assign(self, b, k_tokens, v_tokens):
        """assign (paged_kv.cpp:72-98): tokens (1, kv_heads, n, dim)."""
        self._check_tokens(k_tokens, v_tokens)
        self._update(PAGE_ASSIGN, [b], [k_tokens.shape[2]], k_tokens, v_tokens)

    def append_tokens(self, b, k_new, v_new):
        """append_tokens (paged_kv.cpp:100-126)."""
        self._check_tokens(k_new, v_new)
        self._update(PAGE_APPEND, [b], [k_new.shape[2]], k_new, v_new)

    # -- batched (one launch for many sequences) ------------------------------------------------
    def assign_batch(self, batch_ids, n_tokens, k_tokens=None, v_tokens=None, sync=True):
        """assign for each (batch_ids[i], n_tokens[i]) in order; tokens packed along L."""
        return self._update(PAGE_ASSIGN, batch_ids, n_tokens, k_tokens, v_tokens, sync)

    def append_batch(self, batch_ids, n_tokens, k_new=None, v_new=None, sync=True):
        """append_tokens for each (batch_ids[i], n_tokens[i]) in order; tokens packed along L."""
        return self._update(PAGE_APPEND, batch_ids, n_tokens, k_new, v_new, sync)

    def erase_batch(self, batch_ids, sync=True):
        return self._update(PAGE_ERASE, batch_ids, None, None, None, sync)

    def k_phys(self):
        return self.k

    def v_phys(self):
        return self.v

    def seq_len(self, b):
        self._check_batch(b)
        return int(self._view("seq_len")[b].item())

    def free_pages(self):
        return int(self._view("free_count")[0].item())

    def free_list(self):
        """The free stack bottom to top (the reference's free_ vector)."""
        return self._view("free_stack")[:self.free_pages()].cpu().tolist()

    def max_tokens(self):
        return self.num_pages * self.ps


def convert_block_mask(bm: BlockMask, pt: PageTable, out: Optional[BlockMask] = None,
                       status: Optional[torch.Tensor] = None) -> BlockMask:
    """convert_block_mask (paged_kv.cpp:154-228) on the GPU: logical block columns -> pages.
    ``out`` reuses a converted mask of the same geometry; with a device int32 ``status`` tensor
    the call does not synchronise (UnmappedBlock is reported as status[0] == 1 instead), so a
    serving step can be captured in a CUDA graph."""
    dev = bm.device
    i32 = dict(dtype=torch.int32, device=dev)
    rows, cols = bm.rows, pt.num_physical_pages
    n = pt.batches * bm.h_dims
    if out is None:
        out = BlockMask(pt.batches, bm.h_dims, rows, cols, bm.bs_q, bm.bs_kv, bm.q_len,
                        pt.num_physical_pages * pt.page_size, torch.empty(n * rows, **i32),
                        torch.empty(n * rows * cols, **i32), torch.empty(n * rows, **i32),
                        torch.empty(n * rows * cols, **i32), mask=bm.mask)
    elif out.kv_indices.numel() != n * rows * cols or out.kv_num_blocks.numel() != n * rows:
        raise BlockMaskMismatch("convert_block_mask: `out` has another geometry")
    cl, co = bm.c(), out.c()
    cpt = pt.c(dev)
    lib = _lib.load()
    if status is None:
        _check(lib.fa_convert_block_mask(C.byref(cl), C.byref(cpt), C.byref(co), C.c_void_p(_stream())))
    else:
        if status.dtype != torch.int32 or not status.is_cuda:
            raise ShapeMismatch("convert_block_mask: status must be a device int32 tensor")
        _check(lib.fa_convert_block_mask_async(C.byref(cl), C.byref(cpt), C.byref(co),
                                               C.c_void_p(status.data_ptr()), C.c_void_p(_stream())))
    return out


def launch_count() -> int:
    """Kernel launches issued by libflexattn_b200 in this process."""
    return int(_lib.load().fa_launch_count())
