"""ctypes binding of the C ABI in include/flexattn_b200.h.

The library is built in-tree (``make -C paper_2412_05496_b200``) as
``paper_2412_05496_b200/libflexattn_b200.so``. There is no fallback: if the
library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FA_LIB_PATH: developer override (e.g. an instrumented build); the product path is in-tree
LIB_PATH = os.environ.get("FA_LIB_PATH") or os.path.join(HERE, "libflexattn_b200.so")

FA_F32, FA_BF16 = 0, 1


class MaskDesc(C.Structure):
    _fields_ = [("terms", C.c_uint32), ("hash_density", C.c_int32), ("window", C.c_int64),
                ("prefix", C.c_int64), ("q_offset", C.c_int64), ("hash_seed", C.c_uint64),
                ("doc_ids", C.c_void_p), ("doc_len", C.c_int64),
                ("or_terms", C.c_uint32), ("na_kernel", C.c_int32), ("na_height", C.c_int64),
                ("na_width", C.c_int64), ("remap", C.c_void_p), ("remap_len", C.c_int64),
                ("remap_rc", C.c_void_p)]


class ScoreDesc(C.Structure):
    _fields_ = [("terms", C.c_uint32), ("num_slopes", C.c_int32), ("cap", C.c_double),
                ("slopes", C.c_void_p), ("q_offset", C.c_int64)]


class BlockMaskC(C.Structure):
    _fields_ = [("b_dims", C.c_int64), ("h_dims", C.c_int64), ("rows", C.c_int64),
                ("cols", C.c_int64), ("bs_q", C.c_int64), ("bs_kv", C.c_int64),
                ("q_len", C.c_int64), ("kv_len", C.c_int64),
                ("kv_num_blocks", C.c_void_p), ("kv_indices", C.c_void_p),
                ("full_kv_num_blocks", C.c_void_p), ("full_kv_indices", C.c_void_p),
                ("q_num_blocks", C.c_void_p), ("q_indices", C.c_void_p),
                ("full_q_num_blocks", C.c_void_p), ("full_q_indices", C.c_void_p)]


class TensorC(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int32), ("_pad", C.c_int32),
                ("b", C.c_int64), ("h", C.c_int64), ("l", C.c_int64), ("d", C.c_int64)]


class PageTableC(C.Structure):
    _fields_ = [("batches", C.c_int64), ("max_logical_pages", C.c_int64),
                ("num_physical_pages", C.c_int64), ("page_size", C.c_int64),
                ("table", C.c_void_p), ("phys_to_logical", C.c_void_p), ("owner", C.c_void_p),
                ("seq_len", C.c_void_p), ("max_seq_len", C.c_int64)]


class OpCountersC(C.Structure):
    _fields_ = [("madds", C.c_uint64), ("mask_evals", C.c_uint64), ("score_evals", C.c_uint64)]


FA_FLAG_VALIDATE, FA_FLAG_DETERMINISTIC, FA_FLAG_NO_SYNC = 1, 2, 4
PAGE_ASSIGN, PAGE_APPEND, PAGE_ERASE = 0, 1, 2


class PagePoolC(C.Structure):
    _fields_ = [("batches", C.c_int64), ("num_pages", C.c_int64), ("page_size", C.c_int64),
                ("table", C.c_void_p), ("phys_to_logical", C.c_void_p), ("owner", C.c_void_p),
                ("seq_len", C.c_void_p), ("free_stack", C.c_void_p), ("free_count", C.c_void_p),
                ("status", C.c_void_p), ("scratch", C.c_void_p)]


class FwdArgs(C.Structure):
    _fields_ = [("q", TensorC), ("k", TensorC), ("v", TensorC), ("out", TensorC),
                ("lse", C.c_void_p), ("bm", C.POINTER(BlockMaskC)), ("mask", MaskDesc),
                ("score", ScoreDesc), ("scale", C.c_double), ("gqa_group", C.c_int64),
                ("flags", C.c_uint32), ("_pad1", C.c_int32), ("counters", C.POINTER(OpCountersC))]


class BwdArgs(C.Structure):
    _fields_ = [("q", TensorC), ("k", TensorC), ("v", TensorC), ("out", TensorC),
                ("d_out", TensorC), ("lse", C.c_void_p), ("dq", TensorC), ("dk", TensorC),
                ("dv", TensorC), ("bm", C.POINTER(BlockMaskC)), ("mask", MaskDesc),
                ("score", ScoreDesc), ("scale", C.c_double), ("gqa_group", C.c_int64),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("flags", C.c_uint32), ("_pad1", C.c_int32), ("counters", C.POINTER(OpCountersC)),
                ("phase_events", C.c_void_p * 4)]


class DecodeArgs(C.Structure):
    _fields_ = [("q", TensorC), ("k_cache", TensorC), ("v_cache", TensorC), ("out", TensorC),
                ("lse", C.c_void_p), ("bm", C.POINTER(BlockMaskC)), ("pt", C.POINTER(PageTableC)),
                ("offset", C.c_int64), ("mask", MaskDesc), ("score", ScoreDesc),
                ("scale", C.c_double), ("gqa_group", C.c_int64), ("num_splits", C.c_int32),
                ("_pad", C.c_int32), ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("flags", C.c_uint32), ("_pad2", C.c_int32), ("counters", C.POINTER(OpCountersC))]


# Every symbol include/flexattn_b200.h declares (checked by tests/test_boundary.py).
EXPORTS = [
    "fa_last_error", "fa_status_name", "fa_abi_version", "fa_launch_count",
    "fa_block_mask_geometry", "fa_create_block_mask", "fa_transpose_block_mask",
    "fa_convert_block_mask", "fa_flex_fwd", "fa_bwd_workspace_size", "fa_flex_bwd",
    "fa_decode_workspace_size", "fa_flex_decode", "fa_fill_uniform", "fa_paged_write",
    "fa_check_finite", "fa_page_pool_bytes", "fa_page_pool_init", "fa_page_pool_shuffle",
    "fa_page_pool_update", "fa_page_pool_status", "fa_page_pool_table", "fa_convert_block_mask_async",
]

_lib = None


def load():
    """Load libflexattn_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `make -C paper_2412_05496_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    lib.fa_last_error.restype = C.c_char_p
    lib.fa_status_name.restype = C.c_char_p
    lib.fa_status_name.argtypes = [C.c_int32]
    lib.fa_abi_version.restype = C.c_int32
    lib.fa_launch_count.restype = C.c_uint64
    lib.fa_block_mask_geometry.argtypes = [C.c_int64] * 6 + [C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                                             C.POINTER(C.c_size_t)]
    lib.fa_create_block_mask.argtypes = [C.POINTER(MaskDesc)] + [C.c_int64] * 6 + [
        C.POINTER(BlockMaskC), C.c_void_p, C.c_size_t, C.c_void_p]
    lib.fa_transpose_block_mask.argtypes = [C.POINTER(BlockMaskC), C.c_void_p, C.c_size_t, C.c_void_p]
    lib.fa_convert_block_mask.argtypes = [C.POINTER(BlockMaskC), C.POINTER(PageTableC),
                                          C.POINTER(BlockMaskC), C.c_void_p]
    lib.fa_convert_block_mask_async.argtypes = [C.POINTER(BlockMaskC), C.POINTER(PageTableC),
                                                C.POINTER(BlockMaskC), C.c_void_p, C.c_void_p]
    lib.fa_flex_fwd.argtypes = [C.POINTER(FwdArgs), C.c_void_p]
    lib.fa_bwd_workspace_size.restype = C.c_size_t
    lib.fa_bwd_workspace_size.argtypes = [C.c_int64] * 4
    lib.fa_flex_bwd.argtypes = [C.POINTER(BwdArgs), C.c_void_p]
    lib.fa_decode_workspace_size.restype = C.c_size_t
    lib.fa_decode_workspace_size.argtypes = [C.c_int64] * 4 + [C.c_int32]
    lib.fa_flex_decode.argtypes = [C.POINTER(DecodeArgs), C.c_void_p]
    lib.fa_fill_uniform.argtypes = [C.c_void_p, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_void_p]
    lib.fa_paged_write.argtypes = [C.POINTER(TensorC), C.POINTER(PageTableC), C.POINTER(TensorC),
                                   C.c_void_p]
    lib.fa_check_finite.argtypes = [C.POINTER(TensorC), C.POINTER(C.c_char_p), C.c_int32, C.c_void_p]
    lib.fa_page_pool_bytes.restype = C.c_size_t
    lib.fa_page_pool_bytes.argtypes = [C.c_int64, C.c_int64]
    lib.fa_page_pool_init.argtypes = [C.POINTER(PagePoolC), C.c_void_p, C.c_size_t, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_void_p]
    lib.fa_page_pool_shuffle.argtypes = [C.POINTER(PagePoolC), C.c_uint64, C.c_void_p]
    lib.fa_page_pool_update.argtypes = [C.POINTER(PagePoolC), C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                                        C.POINTER(TensorC), C.POINTER(TensorC), C.POINTER(TensorC),
                                        C.POINTER(TensorC), C.c_uint32, C.c_void_p]
    lib.fa_page_pool_status.argtypes = [C.POINTER(PagePoolC), C.POINTER(C.c_int32), C.c_void_p]
    lib.fa_page_pool_table.restype = PageTableC
    lib.fa_page_pool_table.argtypes = [C.POINTER(PagePoolC)]
    for fn in ("fa_convert_block_mask_async", "fa_page_pool_init", "fa_page_pool_shuffle", "fa_page_pool_update", "fa_page_pool_status",
               "fa_create_block_mask", "fa_transpose_block_mask", "fa_convert_block_mask",
               "fa_flex_fwd", "fa_flex_bwd", "fa_flex_decode", "fa_fill_uniform", "fa_paged_write",
               "fa_block_mask_geometry", "fa_check_finite"):
        getattr(lib, fn).restype = C.c_int32
    _lib = lib
    return lib
