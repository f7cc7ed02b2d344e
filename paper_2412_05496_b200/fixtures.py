"""BlockMask / tensor fixture I/O and the block-grid test aids of the reference, over device
BlockMasks.

File formats are the reference's, byte for byte, so masks and tensors move between this
library and the CPU reference (``blockattn``):

* BlockMask (block_mask.cpp:225-237): 8 u64le header fields (b_dims, h_dims, rows, cols,
  bs_q, bs_kv, q_len, kv_len), then partial_num, partial_idx, full_num, full_idx as u64le.
  The merged visit list is not stored (it is the ascending merge, rebuilt on load,
  block_mask.cpp:239-277); the q-side arrays are rebuilt on the GPU (transpose).
* Tensor4 (tensor.hpp:144-203): u64le rank (4), u64le dims[4], u64le precision tag (32|64),
  then little-endian IEEE values row-major. bf16 tensors are written widened to float32.

Host-side code: the arrays are small (O(rows * cols)); the device work stays in the kernels.
"""
from __future__ import annotations

import struct
from typing import Optional

import numpy as np
import torch

from .api import (BlockMask, Error, IndexOutOfRange, MaskMod, BlockMaskMismatch, _geometry,
                  transpose)

KIND_EMPTY, KIND_PARTIAL, KIND_FULL = 0, 1, 2


def _host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().astype(np.int64)


def _upload(arrs, bm_geom, device, mask) -> BlockMask:
    b_dims, h_dims, rows, cols, bs_q, bs_kv, q_len, kv_len = bm_geom
    dev = torch.device(device)
    t = [torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=dev) for a in arrs]
    bm = BlockMask(b_dims, h_dims, rows, cols, bs_q, bs_kv, q_len, kv_len, t[0], t[1], t[2], t[3],
                   mask=mask)
    if dev.type == "cuda":
        transpose(bm)  # q-side arrays, on the GPU
    return bm


# ---- BlockMask files ------------------------------------------------------------------------
def save_block_mask(path: str, bm: BlockMask) -> None:
    """save_block_mask (block_mask.cpp:225-237)."""
    hdr = (bm.b_dims, bm.h_dims, bm.rows, bm.cols, bm.bs_q, bm.bs_kv, bm.q_len, bm.kv_len)
    try:
        with open(path, "wb") as f:
            f.write(struct.pack("<8Q", *hdr))
            for t in (bm.kv_num_blocks, bm.kv_indices, bm.full_kv_num_blocks, bm.full_kv_indices):
                f.write(_host(t).astype("<u8").tobytes())
    except OSError as e:
        raise Error(f"save_block_mask: cannot write {path}: {e}") from None


def load_block_mask(path: str, device="cuda", mask: Optional[MaskMod] = None) -> BlockMask:
    """load_block_mask (block_mask.cpp:239-277): the runtime mask is not stored; pass ``mask``
    (or use ``with_mask``) before running attention, as with the reference's ``with_mask``."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise Error(f"load_block_mask: cannot open {path}") from None
    if len(data) < 64:
        raise Error("unexpected end of file while reading u64")
    b_dims, h_dims, rows, cols, bs_q, bs_kv, q_len, kv_len = struct.unpack_from("<8q", data, 0)
    r, c, _ = _geometry(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv)
    if (r, c) != (rows, cols):
        raise Error(f"load_block_mask: header rows/cols inconsistent with lengths in {path}")
    n = b_dims * h_dims
    sizes = (n * rows, n * rows * cols, n * rows, n * rows * cols)
    if len(data) < 64 + 8 * sum(sizes):
        raise Error("unexpected end of file while reading u64")
    arrs, off = [], 64
    for sz in sizes:
        arrs.append(np.frombuffer(data, dtype="<i8", count=sz, offset=off).copy())
        off += 8 * sz
    return _upload(arrs, (b_dims, h_dims, rows, cols, bs_q, bs_kv, q_len, kv_len), device, mask)


# ---- dense block grid, test aids --------------------------------------------------------------
def to_dense(bm: BlockMask) -> np.ndarray:
    """to_dense (block_mask.cpp:117-138): (b_dims, h_dims, rows, cols) of KIND_* values."""
    g = np.full((bm.b_dims, bm.h_dims, bm.rows, bm.cols), KIND_EMPTY, dtype=np.int8)
    pn, pi = _host(bm.kv_num_blocks), _host(bm.kv_indices).reshape(-1, bm.cols)
    fn, fi = _host(bm.full_kv_num_blocks), _host(bm.full_kv_indices).reshape(-1, bm.cols)
    flat = g.reshape(-1, bm.cols)
    for row in range(flat.shape[0]):
        flat[row, pi[row, :pn[row]]] = KIND_PARTIAL
        flat[row, fi[row, :fn[row]]] = KIND_FULL
    return g


def block_mask_from_grid(grid: np.ndarray, bs_q: int, bs_kv: int, q_len: int, kv_len: int,
                         mask: Optional[MaskMod] = None, device="cuda") -> BlockMask:
    """block_mask_from_grid (block_mask.cpp:140-159): ascending compacted lists, zero tails."""
    grid = np.asarray(grid)
    if grid.ndim != 4:
        raise BlockMaskMismatch("block_mask_from_grid: grid must be (b_dims, h_dims, rows, cols)")
    b_dims, h_dims, rows, cols = grid.shape
    r, c, _ = _geometry(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv)
    if (r, c) != (rows, cols):
        raise BlockMaskMismatch(f"block_mask_from_grid: grid is {rows}x{cols} blocks but lengths give {r}x{c}")
    flat = grid.reshape(-1, cols)
    pn = np.zeros(flat.shape[0], np.int64)
    fn = np.zeros_like(pn)
    pi = np.zeros(flat.shape, np.int64)
    fi = np.zeros_like(pi)
    for row in range(flat.shape[0]):
        p = np.nonzero(flat[row] == KIND_PARTIAL)[0]
        f = np.nonzero(flat[row] == KIND_FULL)[0]
        pn[row], fn[row] = len(p), len(f)
        pi[row, :len(p)], fi[row, :len(f)] = p, f
    return _upload((pn, pi.reshape(-1), fn, fi.reshape(-1)),
                   (b_dims, h_dims, rows, cols, bs_q, bs_kv, q_len, kv_len), device, mask)


def demote_full_to_partial(bm: BlockMask) -> BlockMask:
    """demote_full_to_partial (block_mask.cpp:193-206): the merged visit list becomes the
    partial list, no full blocks — every visited block then evaluates mask_mod (the
    metamorphic check of the full-block fast path, acceptance.cpp:280-309)."""
    g = to_dense(bm)
    vis = np.where(g != KIND_EMPTY, KIND_PARTIAL, KIND_EMPTY).astype(np.int8)
    return block_mask_from_grid(vis, bm.bs_q, bm.bs_kv, bm.q_len, bm.kv_len, bm.mask, bm.device)


def promote_empty_to_partial(bm: BlockMask) -> BlockMask:
    """promote_empty_to_partial (block_mask.cpp:208-223): empty tiles become partial, so the
    kernels visit every tile (the mask must then zero them; test_engine.cpp:103-122)."""
    g = to_dense(bm)
    out = np.where(g == KIND_FULL, KIND_FULL, KIND_PARTIAL).astype(np.int8)
    return block_mask_from_grid(out, bm.bs_q, bm.bs_kv, bm.q_len, bm.kv_len, bm.mask, bm.device)


def _check_bh(bm: BlockMask, b: int, h: int):
    if b < 0 or b >= bm.b_dims or h < 0 or h >= bm.h_dims:
        raise IndexOutOfRange(f"BlockMask: (b,h)=({b},{h}) outside mask dims ({bm.b_dims},{bm.h_dims})")


def render_ascii(bm: BlockMask, b: int = 0, h: int = 0) -> str:
    """render_ascii (block_mask.cpp:279-295): white square / shade / full block per tile."""
    _check_bh(bm, b, h)
    sym = {KIND_EMPTY: "□", KIND_PARTIAL: "▒", KIND_FULL: "█"}
    g = to_dense(bm)[b, h]
    return "".join("".join(sym[int(k)] for k in row) + "\n" for row in g)


def render_ppm(bm: BlockMask, b: int = 0, h: int = 0) -> bytes:
    """render_ppm (block_mask.cpp:297-316): P6, empty 255 / partial 128 / full 0."""
    _check_bh(bm, b, h)
    g = to_dense(bm)[b, h]
    lut = np.array([255, 128, 0], np.uint8)
    px = np.repeat(lut[g.astype(np.int64)].reshape(-1, 1), 3, axis=1)
    return f"P6\n{bm.cols} {bm.rows}\n255\n".encode() + px.tobytes()


def write_ppm(path: str, bm: BlockMask, b: int = 0, h: int = 0) -> None:
    data = render_ppm(bm, b, h)
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:
        raise Error(f"write_ppm: cannot open {path}: {e}") from None


# ---- Tensor4 files ------------------------------------------------------------------------------
def save_tensor(path: str, t: torch.Tensor) -> None:
    """save_tensor (tensor.hpp:144-170): float64 keeps tag 64, everything else is written as
    float32 (tag 32; bf16 widens exactly)."""
    if t.dim() != 4:
        raise Error(f"save_tensor: expected a rank-4 tensor, got rank {t.dim()}")
    x = t.detach().cpu()
    x = x.to(torch.float64) if x.dtype == torch.float64 else x.to(torch.float32)
    tag = 64 if x.dtype == torch.float64 else 32
    try:
        with open(path, "wb") as f:
            f.write(struct.pack("<5Q", 4, *x.shape))
            f.write(struct.pack("<Q", tag))
            f.write(x.contiguous().numpy().astype("<f8" if tag == 64 else "<f4").tobytes())
    except OSError as e:
        raise Error(f"save_tensor: cannot open {path}: {e}") from None


def load_tensor(path: str, dtype: torch.dtype = torch.float32, device="cpu") -> torch.Tensor:
    """load_tensor (tensor.hpp:172-203): the file's precision tag must match ``dtype`` (float32
    <-> 32, float64 <-> 64); bf16 loads a 32-bit file and rounds."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise Error(f"load_tensor: cannot open {path}") from None
    if len(data) < 48:
        raise Error("unexpected end of file while reading u64")
    rank = struct.unpack_from("<Q", data, 0)[0]
    if rank != 4:
        raise Error(f"load_tensor: expected rank 4, got {rank}")
    dims = struct.unpack_from("<4q", data, 8)
    tag = struct.unpack_from("<Q", data, 40)[0]
    want = 64 if dtype == torch.float64 else 32
    if tag != want:
        raise Error(f"load_tensor: precision tag {tag} does not match requested {want}-bit load")
    n = int(np.prod(dims))
    if len(data) < 48 + n * tag // 8:
        raise Error(f"load_tensor: truncated payload in {path}")
    arr = np.frombuffer(data, dtype="<f8" if tag == 64 else "<f4", count=n, offset=48).reshape(dims)
    return torch.from_numpy(arr.copy()).to(dtype=dtype, device=device)
