"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end of the CPU oracle.

Two checkers live behind this module:

* ``port``: ``oracle/libflex_oracle.so``, the C restatement of the reference
  algorithms (``oracle/flex_oracle.c``; every function cites the reference
  file:line it follows). Always available once ``make -C oracle`` ran.
* ``ref``: ``oracle/_ref/libblockattn_ref.so``, the UNMODIFIED reference
  library compiled from /root/reference sources plus a C shim
  (``oracle/ref_shim.cpp``). Available where it was built (it travels to the
  GPU box with the repo snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module. The product path (``paper_2412_05496_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "libflex_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libblockattn_ref.so")

MASK_CAUSAL, MASK_SLIDING, MASK_DOCUMENT, MASK_PREFIX, MASK_HASH, MASK_NEVER = 1, 2, 4, 8, 16, 32
MASK_NATTEN = 64
SCORE_ALIBI, SCORE_SOFTCAP = 1, 2


class _FoMask(C.Structure):
    _fields_ = [("terms", C.c_uint32), ("hash_density", C.c_int32), ("window", C.c_int64),
                ("prefix", C.c_int64), ("q_offset", C.c_int64), ("hash_seed", C.c_uint64),
                ("doc_ids", C.POINTER(C.c_int64)), ("doc_len", C.c_int64),
                ("bound_q", C.c_int64), ("bound_kv", C.c_int64),
                ("or_terms", C.c_uint32), ("na_kernel", C.c_int32), ("na_height", C.c_int64),
                ("na_width", C.c_int64), ("remap", C.POINTER(C.c_int64)), ("remap_len", C.c_int64)]


class _FoScore(C.Structure):
    _fields_ = [("terms", C.c_uint32), ("num_slopes", C.c_int32), ("cap", C.c_double),
                ("slopes", C.POINTER(C.c_double)), ("q_offset", C.c_int64)]


class _FoBm(C.Structure):
    _fields_ = [("b_dims", C.c_int64), ("h_dims", C.c_int64), ("rows", C.c_int64),
                ("cols", C.c_int64), ("bs_q", C.c_int64), ("bs_kv", C.c_int64),
                ("partial_num", C.POINTER(C.c_int64)), ("partial_idx", C.POINTER(C.c_int64)),
                ("full_num", C.POINTER(C.c_int64)), ("full_idx", C.POINTER(C.c_int64))]


@dataclass
class Mask:
    """AND of primitive mask terms, optionally ORed with a second group and remapped
    (same bits and meaning as fa_mask_desc)."""
    terms: int = 0
    window: int = 0
    prefix: int = 0
    q_offset: int = 0
    hash_seed: int = 0
    hash_density: int = 128
    doc_ids: Optional[np.ndarray] = None
    or_terms: int = 0
    na_height: int = 0
    na_width: int = 0
    na_kernel: int = 0
    remap: Optional[np.ndarray] = None

    def c(self, bound_q: int = 0, bound_kv: int = 0) -> _FoMask:
        m = _FoMask()
        m.terms = self.terms
        m.hash_density = self.hash_density
        m.window = self.window
        m.prefix = self.prefix
        m.q_offset = self.q_offset
        m.hash_seed = self.hash_seed
        if self.doc_ids is not None:
            self._ids = np.ascontiguousarray(self.doc_ids, dtype=np.int64)
            m.doc_ids = self._ids.ctypes.data_as(C.POINTER(C.c_int64))
            m.doc_len = len(self._ids)
        m.bound_q = bound_q
        m.bound_kv = bound_kv
        m.or_terms = self.or_terms
        m.na_height, m.na_width, m.na_kernel = self.na_height, self.na_width, self.na_kernel
        if self.remap is not None:
            self._remap = np.ascontiguousarray(self.remap, dtype=np.int64)
            m.remap = self._remap.ctypes.data_as(C.POINTER(C.c_int64))
            m.remap_len = len(self._remap)
        return m


@dataclass
class Score:
    terms: int = 0
    cap: float = 0.0
    slopes: Optional[np.ndarray] = None
    q_offset: int = 0

    def c(self) -> _FoScore:
        s = _FoScore()
        s.terms = self.terms
        s.cap = self.cap
        s.q_offset = self.q_offset
        if self.slopes is not None:
            self._sl = np.ascontiguousarray(self.slopes, dtype=np.float64)
            s.slopes = self._sl.ctypes.data_as(C.POINTER(C.c_double))
            s.num_slopes = len(self._sl)
        return s


def causal(offset: int = 0) -> Mask:
    return Mask(terms=MASK_CAUSAL, q_offset=offset)


def sliding_window(w: int) -> Mask:
    return Mask(terms=MASK_SLIDING, window=w)


def document(ids, and_causal: bool = False) -> Mask:
    return Mask(terms=MASK_DOCUMENT | (MASK_CAUSAL if and_causal else 0),
                doc_ids=np.asarray(ids, dtype=np.int64))


def na_naive(h: int, w: int, kernel: int) -> Mask:
    """na_naive(NAGeometry(h, w, kernel)) (mask_library.cpp:137-149)."""
    return Mask(terms=MASK_NATTEN, na_height=h, na_width=w, na_kernel=kernel)


def tile_permutation_np(h: int, w: int, tile: int) -> np.ndarray:
    """Restatement of tile_permutation (mask_library.cpp:164-181): tiles in row-major order,
    pixels row-major within a tile."""
    out = []
    for tr in range(0, h, tile):
        for tc in range(0, w, tile):
            for r in range(tr, tr + tile):
                for c in range(tc, tc + tile):
                    out.append(r * w + c)
    return np.asarray(out, dtype=np.int64)


def morton_permutation_np(n_side: int) -> np.ndarray:
    """Restatement of morton_permutation (mask_library.cpp:183-201): slot = bit interleave
    of (row, col), col bits in the even positions."""
    out = np.zeros(n_side * n_side, dtype=np.int64)
    bits = max(1, (n_side - 1).bit_length())
    for r in range(n_side):
        for c in range(n_side):
            slot = 0
            for b in range(bits):
                if (1 << b) >= n_side:
                    break
                slot |= ((c >> b) & 1) << (2 * b)
                slot |= ((r >> b) & 1) << (2 * b + 1)
            out[slot] = r * n_side + c
    return out


def ref_save_block_mask(mask: Mask, bd, hd, ql, kl, bsq, bskv, path: str):
    lib = ref()
    mc = mask.c()
    _check(lib.ref_save_block_mask(C.byref(mc), *_i64(bd, hd, ql, kl, bsq, bskv), path.encode()), lib)


def ref_load_block_mask(path: str, cap_rows: int = 1 << 16, cap_cells: int = 1 << 22):
    """(header[8], partial_num, partial_idx, full_num, full_idx) as read by the reference."""
    lib = ref()
    hdr = np.zeros(8, np.int64)
    pn, fn = np.zeros(cap_rows, np.int64), np.zeros(cap_rows, np.int64)
    pi, fi = np.zeros(cap_cells, np.int64), np.zeros(cap_cells, np.int64)
    _check(lib.ref_load_block_mask(path.encode(), *[_p(a, C.c_int64) for a in (hdr, pn, pi, fn, fi)],
                                   C.c_int64(cap_rows), C.c_int64(cap_cells)), lib)
    n = int(hdr[0] * hdr[1])
    rows, cols = int(hdr[2]), int(hdr[3])
    return hdr, pn[:n * rows], pi[:n * rows * cols], fn[:n * rows], fi[:n * rows * cols]


def ref_write_ppm(mask: Mask, ql, kl, bs, path: str):
    lib = ref()
    mc = mask.c()
    _check(lib.ref_write_ppm(C.byref(mc), *_i64(ql, kl, bs), path.encode()), lib)


def ref_save_tensor_f32(x: np.ndarray, path: str):
    lib = ref()
    x = np.ascontiguousarray(x, dtype=np.float32)
    _check(lib.ref_save_tensor_f32(_p(x, C.c_float), *_i64(*x.shape), path.encode()), lib)


def ref_load_tensor_f32(path: str, shape) -> np.ndarray:
    lib = ref()
    out = np.zeros(int(np.prod(shape)), np.float32)
    _check(lib.ref_load_tensor_f32(path.encode(), _p(out, C.c_float), C.c_int64(out.size)), lib)
    return out.reshape(shape)


def ref_tile_permutation(h: int, w: int, kernel: int, tile: int) -> np.ndarray:
    lib = ref()
    out = np.zeros(h * w, dtype=np.int64)
    _check(lib.ref_tile_permutation(C.c_int64(h), C.c_int64(w), C.c_int64(kernel), C.c_int64(tile),
                                    _p(out, C.c_int64)), lib)
    return out


def ref_morton_permutation(h: int, w: int, kernel: int) -> np.ndarray:
    lib = ref()
    out = np.zeros(h * w, dtype=np.int64)
    _check(lib.ref_morton_permutation(C.c_int64(h), C.c_int64(w), C.c_int64(kernel), _p(out, C.c_int64)), lib)
    return out


def alibi_slopes(heads: int) -> np.ndarray:
    """alibi_slopes (mask_library.cpp:71-81)."""
    return np.array([-(2.0 ** (-8.0 * (h + 1) / heads)) for h in range(heads)], dtype=np.float64)


# ---- SplitMix64 (random.hpp:15-46) --------------------------------------------------------
_M64 = (1 << 64) - 1
_GOLD = 0x9E3779B97F4A7C15


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & _M64

    def next_u64(self) -> int:
        self.state = (self.state + _GOLD) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def next_below(self, n: int) -> int:
        return self.next_u64() % n


def random_f32(seed: int, shape, first: int = 0) -> np.ndarray:
    """random_tensor<float>(seed, ...) (random.hpp:41-46), vectorised counter form."""
    n = int(np.prod(shape))
    i = np.arange(first, first + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (i + np.uint64(1)) * np.uint64(_GOLD)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    unit = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (unit * 2.0 - 1.0).astype(np.float32).reshape(shape)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 (round to nearest even) -> float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


def make_doc_ids(length: int, ndocs: int, seed: int) -> np.ndarray:
    """make_doc_ids (bench.cpp:115-129)."""
    ndocs = max(1, min(ndocs, length))
    rng = SplitMix64(seed)
    cuts = set()
    while len(cuts) < ndocs - 1:
        cuts.add(1 + rng.next_below(length - 1))
    ids = np.zeros(length, dtype=np.int64)
    doc = 0
    for t in range(length):
        if t in cuts:
            doc += 1
        ids[t] = doc
    return ids


def deterministic_shuffle(v: list, seed: int) -> list:
    """deterministic_shuffle (random.hpp:49-56)."""
    rng = SplitMix64(seed)
    v = list(v)
    for i in range(len(v), 1, -1):
        j = rng.next_below(i)
        v[i - 1], v[j] = v[j], v[i - 1]
    return v


# ---- library loading -------------------------------------------------------------------------
_port = None
_ref = None


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            raise RuntimeError(f"oracle port not built: {PORT_PATH} (run `make -C oracle`)")
        _port = C.CDLL(PORT_PATH)
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference library not built: {REF_PATH} (run `make -C oracle ref`)")
        _ref = C.CDLL(REF_PATH)
        _ref.ref_last_error.restype = C.c_char_p
    return _ref


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _i64(*xs):
    return [C.c_int64(int(x)) for x in xs]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


def _check(st: int, lib=None):
    if st != 0:
        msg = lib.ref_last_error().decode() if lib is not None and hasattr(lib, "ref_last_error") else ""
        raise OracleError(st, msg)


# ---- BlockMask -------------------------------------------------------------------------------
@dataclass
class BlockMaskNP:
    b_dims: int
    h_dims: int
    rows: int
    cols: int
    bs_q: int
    bs_kv: int
    q_len: int
    kv_len: int
    partial_num: np.ndarray
    partial_idx: np.ndarray
    full_num: np.ndarray
    full_idx: np.ndarray
    extra: dict = field(default_factory=dict)

    def c(self) -> _FoBm:
        b = _FoBm()
        b.b_dims, b.h_dims, b.rows, b.cols, b.bs_q, b.bs_kv = (
            self.b_dims, self.h_dims, self.rows, self.cols, self.bs_q, self.bs_kv)
        self._keep = [np.ascontiguousarray(a, dtype=np.int64) for a in
                      (self.partial_num, self.partial_idx, self.full_num, self.full_idx)]
        b.partial_num, b.partial_idx, b.full_num, b.full_idx = [_p(a, C.c_int64) for a in self._keep]
        return b

    def transposed(self) -> "BlockMaskNP":
        return transpose(self)


def _alloc_bm(bd, hd, rows, cols):
    return (np.zeros(bd * hd * rows, np.int64), np.zeros(bd * hd * rows * cols, np.int64),
            np.zeros(bd * hd * rows, np.int64), np.zeros(bd * hd * rows * cols, np.int64))


def create_block_mask(mask: Mask, b_dims, h_dims, q_len, kv_len, bs_q=128, bs_kv=128) -> BlockMaskNP:
    """Port of create_block_mask (block_mask.cpp:79-115)."""
    rows, cols = -(-q_len // bs_q), -(-kv_len // bs_kv)
    pn, pi, fn, fi = _alloc_bm(b_dims, h_dims, rows, cols)
    mc = mask.c()
    lib = port()
    st = lib.fo_create_block_mask(C.byref(mc), *_i64(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv),
                                  _p(pn, C.c_int64), _p(pi, C.c_int64), _p(fn, C.c_int64), _p(fi, C.c_int64))
    _check(st)
    return BlockMaskNP(b_dims, h_dims, rows, cols, bs_q, bs_kv, q_len, kv_len, pn, pi, fn, fi)


def transpose(bm: BlockMaskNP) -> BlockMaskNP:
    """Port of transpose (block_mask.cpp:161-178)."""
    tpn, tpi, tfn, tfi = _alloc_bm(bm.b_dims, bm.h_dims, bm.cols, bm.rows)
    port().fo_transpose(*_i64(bm.b_dims, bm.h_dims, bm.rows, bm.cols),
                        _p(bm.partial_num, C.c_int64), _p(bm.partial_idx, C.c_int64),
                        _p(bm.full_num, C.c_int64), _p(bm.full_idx, C.c_int64),
                        _p(tpn, C.c_int64), _p(tpi, C.c_int64), _p(tfn, C.c_int64), _p(tfi, C.c_int64))
    return BlockMaskNP(bm.b_dims, bm.h_dims, bm.cols, bm.rows, bm.bs_kv, bm.bs_q, bm.kv_len,
                       bm.q_len, tpn, tpi, tfn, tfi)


def ref_create_block_mask(mask: Mask, b_dims, h_dims, q_len, kv_len, bs_q=128, bs_kv=128):
    """The reference's own create_block_mask + transpose (oracle/_ref)."""
    rows, cols = -(-q_len // bs_q), -(-kv_len // bs_kv)
    pn, pi, fn, fi = _alloc_bm(b_dims, h_dims, rows, cols)
    vn = np.zeros_like(pn)
    vi = np.zeros_like(pi)
    vf = np.zeros(pi.shape, np.uint8)
    tpn, tpi, tfn, tfi = _alloc_bm(b_dims, h_dims, cols, rows)
    mc = mask.c()
    lib = ref()
    st = lib.ref_create_block_mask(C.byref(mc), *_i64(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv),
                                   *[_p(a, C.c_int64) for a in (pn, pi, fn, fi, vn, vi)], _p(vf, C.c_uint8),
                                   *[_p(a, C.c_int64) for a in (tpn, tpi, tfn, tfi)])
    _check(st, lib)
    bm = BlockMaskNP(b_dims, h_dims, rows, cols, bs_q, bs_kv, q_len, kv_len, pn, pi, fn, fi,
                     extra=dict(visit_num=vn, visit_idx=vi, visit_full=vf))
    bm_t = BlockMaskNP(b_dims, h_dims, cols, rows, bs_kv, bs_q, kv_len, q_len, tpn, tpi, tfn, tfi)
    return bm, bm_t


# ---- attention -------------------------------------------------------------------------------
def _dims(q, k, gqa):
    B, Hq, Lq, D = q.shape
    Bkv, Hkv, Lkv, _ = k.shape
    return B, Hq, Hkv, Bkv, Lq, Lkv, D


def _scale(scale, D):
    return float(scale) if scale and scale > 0 else 1.0 / np.sqrt(D)


def forward(q, k, v, mask: Mask, score: Score, bm: BlockMaskNP, scale=None, gqa=1):
    """Port of forward<Real> (engine.cpp:46-172); dtype from q (float32/float64)."""
    dt = q.dtype
    q, k, v = (np.ascontiguousarray(x, dtype=dt) for x in (q, k, v))
    B, Hq, Hkv, Bkv, Lq, Lkv, D = _dims(q, k, gqa)
    out = np.zeros_like(q)
    lse = np.zeros((B, Hq, Lq), dt)
    ct = C.c_float if dt == np.float32 else C.c_double
    fn = port().fo_forward_f32 if dt == np.float32 else port().fo_forward_f64
    mc, sc, bc = mask.c(bound_q=bm.q_len, bound_kv=bm.kv_len), score.c(), bm.c()
    st = fn(_p(q, ct), _p(k, ct), _p(v, ct), *_i64(B, Hq, Hkv, Bkv, Lq, Lkv, D),
            C.c_double(_scale(scale, D)), C.c_int64(gqa), C.byref(sc), C.byref(mc), C.byref(bc),
            _p(out, ct), _p(lse, ct))
    _check(st)
    return out, lse


def backward(q, k, v, out, lse, dout, mask: Mask, score: Score, bm: BlockMaskNP, scale=None, gqa=1):
    """Port of backward<Real> (engine.cpp:174-401)."""
    dt = q.dtype
    q, k, v, out, lse, dout = (np.ascontiguousarray(x, dtype=dt) for x in (q, k, v, out, lse, dout))
    B, Hq, Hkv, Bkv, Lq, Lkv, D = _dims(q, k, gqa)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    ct = C.c_float if dt == np.float32 else C.c_double
    fn = port().fo_backward_f32 if dt == np.float32 else port().fo_backward_f64
    bm_t = transpose(bm)
    mc, sc, bc, btc = mask.c(bound_q=bm.q_len, bound_kv=bm.kv_len), score.c(), bm.c(), bm_t.c()
    st = fn(*[_p(x, ct) for x in (q, k, v, out, lse, dout)], *_i64(B, Hq, Hkv, Bkv, Lq, Lkv, D),
            C.c_double(_scale(scale, D)), C.c_int64(gqa), C.byref(sc), C.byref(mc), C.byref(bc),
            C.byref(btc), _p(dq, ct), _p(dk, ct), _p(dv, ct))
    _check(st)
    return dq, dk, dv


def dense_forward64(q, k, v, mask: Mask, score: Score, scale=None, gqa=1):
    """Port of dense_forward (oracle.cpp:13-76) in double, bounds = tensor lengths."""
    q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
    B, Hq, Hkv, Bkv, Lq, Lkv, D = _dims(q, k, gqa)
    out = np.zeros_like(q)
    lse = np.zeros((B, Hq, Lq))
    mc, sc = mask.c(), score.c()
    ct = C.c_double
    st = port().fo_dense_forward_f64(_p(q, ct), _p(k, ct), _p(v, ct), *_i64(B, Hq, Hkv, Bkv, Lq, Lkv, D),
                                     C.c_double(_scale(scale, D)), C.c_int64(gqa), C.byref(sc),
                                     C.byref(mc), _p(out, ct), _p(lse, ct))
    _check(st)
    return out, lse


def convert_block_mask(bm: BlockMaskNP, table: np.ndarray, num_physical_pages: int) -> BlockMaskNP:
    """Port of convert_block_mask (paged_kv.cpp:154-228), kv side."""
    table = np.ascontiguousarray(table, dtype=np.int32)
    batches, mlp = table.shape
    pn, pi, fn, fi = _alloc_bm(batches, bm.h_dims, bm.rows, num_physical_pages)
    st = port().fo_convert_block_mask(*_i64(bm.b_dims, bm.h_dims, bm.rows, bm.cols),
                                      *[_p(np.ascontiguousarray(a, np.int64), C.c_int64) for a in
                                        (bm.partial_num, bm.partial_idx, bm.full_num, bm.full_idx)],
                                      *_i64(batches, mlp, num_physical_pages), _p(table, C.c_int32),
                                      *[_p(a, C.c_int64) for a in (pn, pi, fn, fi)])
    _check(st)
    return BlockMaskNP(batches, bm.h_dims, bm.rows, num_physical_pages, bm.bs_q, bm.bs_kv, bm.q_len,
                       num_physical_pages * bm.bs_kv, pn, pi, fn, fi)


# ---- reference library (oracle/_ref) ---------------------------------------------------------
def ref_forward(q, k, v, mask: Mask, score: Score, mask_dims=(1, 1), bs=128, scale=None, gqa=1):
    dt = q.dtype
    q, k, v = (np.ascontiguousarray(x, dtype=dt) for x in (q, k, v))
    B, Hq, Hkv, Bkv, Lq, Lkv, D = _dims(q, k, gqa)
    out = np.zeros_like(q)
    lse = np.zeros((B, Hq, Lq), dt)
    ct = C.c_float if dt == np.float32 else C.c_double
    lib = ref()
    fn = lib.ref_forward_f32 if dt == np.float32 else lib.ref_forward_f64
    mc, sc = mask.c(), score.c()
    st = fn(_p(q, ct), _p(k, ct), _p(v, ct), *_i64(B, Hq, Hkv, Bkv, Lq, Lkv, D),
            C.c_double(scale or 0.0), C.c_int64(gqa), C.byref(sc), C.byref(mc),
            *_i64(mask_dims[0], mask_dims[1], bs), _p(out, ct), _p(lse, ct))
    _check(st, lib)
    return out, lse


def ref_backward(q, k, v, dout, mask: Mask, score: Score, mask_dims=(1, 1), bs=128, scale=None, gqa=1):
    dt = q.dtype
    q, k, v, dout = (np.ascontiguousarray(x, dtype=dt) for x in (q, k, v, dout))
    B, Hq, Hkv, Bkv, Lq, Lkv, D = _dims(q, k, gqa)
    out, dq = np.zeros_like(q), np.zeros_like(q)
    dk, dv = np.zeros_like(k), np.zeros_like(v)
    lse = np.zeros((B, Hq, Lq), dt)
    ct = C.c_float if dt == np.float32 else C.c_double
    lib = ref()
    fn = lib.ref_backward_f32 if dt == np.float32 else lib.ref_backward_f64
    mc, sc = mask.c(), score.c()
    st = fn(*[_p(x, ct) for x in (q, k, v, dout)], *_i64(B, Hq, Hkv, Bkv, Lq, Lkv, D),
            C.c_double(scale or 0.0), C.c_int64(gqa), C.byref(sc), C.byref(mc),
            *_i64(mask_dims[0], mask_dims[1], bs), *[_p(x, ct) for x in (out, lse, dq, dk, dv)])
    _check(st, lib)
    return out, lse, dq, dk, dv


def ref_decode(q_step, k, v, offset, mask: Mask, score: Score, bs=128, scale=None, gqa=1):
    q_step, k, v = (np.ascontiguousarray(x, dtype=np.float32) for x in (q_step, k, v))
    B, Hq, Hkv, Bkv, n_new, Lkv, D = _dims(q_step, k, gqa)
    out = np.zeros_like(q_step)
    lse = np.zeros((B, Hq, n_new), np.float32)
    lib = ref()
    mc, sc = mask.c(), score.c()
    ct = C.c_float
    st = lib.ref_decode_f32(_p(q_step, ct), _p(k, ct), _p(v, ct), *_i64(B, Hq, Hkv, Bkv, n_new, Lkv, D, offset),
                            C.c_double(scale or 0.0), C.c_int64(gqa), C.byref(sc), C.byref(mc),
                            C.c_int64(bs), _p(out, ct), _p(lse, ct))
    _check(st, lib)
    return out, lse


def ref_paged_decode(q_step, k, v, offset, mask: Mask, score: Score, page_size=128,
                     shuffle_seed=0, scale=None, gqa=1):
    q_step, k, v = (np.ascontiguousarray(x, dtype=np.float32) for x in (q_step, k, v))
    B, Hq, Hkv, Bkv, n_new, Lkv, D = _dims(q_step, k, gqa)
    out = np.zeros_like(q_step)
    lse = np.zeros((B, Hq, n_new), np.float32)
    pages_per_seq = -(-Lkv // page_size)
    num_pages = B * pages_per_seq + B
    table = np.zeros((B, num_pages), np.int32)
    npages = C.c_int64(0)
    lib = ref()
    mc, sc = mask.c(), score.c()
    ct = C.c_float
    st = lib.ref_paged_decode_f32(_p(q_step, ct), _p(k, ct), _p(v, ct), *_i64(B, Hq, Hkv, n_new, Lkv, D, offset),
                                  C.c_double(scale or 0.0), C.c_int64(gqa), C.byref(sc), C.byref(mc),
                                  C.c_int64(page_size), C.c_uint64(shuffle_seed), _p(out, ct), _p(lse, ct),
                                  _p(table, C.c_int32), C.byref(npages))
    _check(st, lib)
    return out, lse, table


def ref_paged_layout(B, num_pages, page_size, shuffle_seed, tokens_per_batch):
    """Page table of a reference PagedKVCache after shuffle + assign (paged_kv.cpp:14-98)."""
    table = np.zeros((B, num_pages), np.int32)
    p2l = np.zeros(num_pages, np.int32)
    owner = np.zeros(num_pages, np.int32)
    lib = ref()
    st = lib.ref_paged_layout(*_i64(B, num_pages, page_size), C.c_uint64(shuffle_seed),
                              C.c_int64(tokens_per_batch), _p(table, C.c_int32), _p(p2l, C.c_int32),
                              _p(owner, C.c_int32))
    _check(st, lib)
    return table, p2l, owner


def ref_paged_script(B, num_pages, page_size, heads, dim, ops, tok):
    """Run a script of PagedKVCache calls on the reference (ref_shim.cpp ref_paged_script):
    ops = [(kind, b, n, seed)], kind 0 assign / 1 append / 2 erase / 3 shuffle. Returns
    (status per op, table, p2l, owner, seq_len, free_pages, k_phys, v_phys)."""
    m = len(ops)
    op = np.array([o[0] for o in ops], np.int32)
    bat = np.array([o[1] for o in ops], np.int64)
    nn = np.array([o[2] for o in ops], np.int64)
    seed = np.array([o[3] & (2**64 - 1) for o in ops], np.uint64)
    tok = np.ascontiguousarray(tok, np.float32)
    status = np.zeros(m, np.int32)
    table = np.zeros((B, num_pages), np.int32)
    p2l = np.zeros(num_pages, np.int32)
    owner = np.zeros(num_pages, np.int32)
    seq = np.zeros(B, np.int64)
    free = C.c_int64(0)
    kp = np.zeros((1, heads, num_pages * page_size, dim), np.float32)
    vp = np.zeros_like(kp)
    lib = ref()
    st = lib.ref_paged_script(*_i64(B, num_pages, page_size, heads, dim, m), _p(op, C.c_int32),
                              _p(bat, C.c_int64), _p(nn, C.c_int64), _p(seed, C.c_uint64),
                              _p(tok, C.c_float), _p(status, C.c_int32), _p(table, C.c_int32),
                              _p(p2l, C.c_int32), _p(owner, C.c_int32), _p(seq, C.c_int64),
                              C.byref(free), _p(kp, C.c_float), _p(vp, C.c_float))
    _check(st, lib)
    return status, table, p2l, owner, seq, free.value, kp, vp


def ref_convert_block_mask(mask: Mask, bd, hd, ql, kl, bs, table: np.ndarray, num_physical_pages: int):
    table = np.ascontiguousarray(table, dtype=np.int32)
    batches, mlp = table.shape
    rows = -(-ql // bs)
    pn, pi, fn, fi = _alloc_bm(batches, hd, rows, num_physical_pages)
    lib = ref()
    mc = mask.c()
    st = lib.ref_convert_block_mask(C.byref(mc), *_i64(bd, hd, ql, kl, bs, batches, mlp, num_physical_pages),
                                    _p(table, C.c_int32), *[_p(a, C.c_int64) for a in (pn, pi, fn, fi)])
    _check(st, lib)
    return pn, pi, fn, fi


def ref_time_fwd_bwd(q, k, v, dout, mask: Mask, score: Score, bs=128, scale=None, gqa=1,
                     do_bwd=True, workers=None):
    """Wall time (s) of the reference forward<float> and backward<float> on prebuilt masks."""
    if workers is not None:
        os.environ["BLOCKATTN_WORKERS"] = str(int(workers))  # read per call (parallel.cpp:10-15)
    q, k, v, dout = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v, dout))
    B, Hq, Hkv, Bkv, Lq, Lkv, D = _dims(q, k, gqa)
    f, b = C.c_double(0.0), C.c_double(0.0)
    lib = ref()
    mc, sc = mask.c(), score.c()
    ct = C.c_float
    st = lib.ref_time_fwd_bwd_f32(*[_p(x, ct) for x in (q, k, v, dout)], *_i64(B, Hq, Hkv, Bkv, Lq, Lkv, D),
                                  C.c_double(scale or 0.0), C.c_int64(gqa), C.byref(sc), C.byref(mc),
                                  C.c_int64(bs), C.c_int(1 if do_bwd else 0), C.byref(f), C.byref(b))
    _check(st, lib)
    return f.value, b.value


def ref_counters(q, k, v, dout, mask: Mask, score: Score, bs=128, scale=None, gqa=1):
    """OpCounters of the reference forward<float> and backward<float> (engine.hpp:21-32):
    ((madds, mask_evals, score_evals) forward, (...) backward)."""
    q, k, v, dout = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v, dout))
    B, Hq, Hkv, Bkv, Lq, Lkv, D = _dims(q, k, gqa)
    out = np.zeros(6, np.uint64)
    lib = ref()
    mc, sc = mask.c(), score.c()
    ct = C.c_float
    st = lib.ref_counters_f32(*[_p(x, ct) for x in (q, k, v, dout)], *_i64(B, Hq, Hkv, Bkv, Lq, Lkv, D),
                              C.c_double(scale or 0.0), C.c_int64(gqa), C.byref(sc), C.byref(mc),
                              C.c_int64(bs), _p(out, C.c_uint64))
    _check(st, lib)
    return tuple(int(x) for x in out[:3]), tuple(int(x) for x in out[3:])
