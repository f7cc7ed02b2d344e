"""CPU: the C-ABI boundary. The library loads without a GPU, exports exactly what
include/flexattn_b200.h declares, the ctypes mirror matches the C struct layouts, and the
host-side argument validation returns the reference's error taxonomy (errors.hpp) before
any device work."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flexattn_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"FA_API\s+[\w\s\*]*?\b(fa_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    assert sorted(_lib.EXPORTS) == syms
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r" T (fa_\w+)", out)))
    assert exported == syms  # nothing else leaks across the boundary


def test_ctypes_layout_matches_header(tmp_path):
    from paper_2412_05496_b200 import _lib
    structs = {"fa_mask_desc": _lib.MaskDesc, "fa_score_desc": _lib.ScoreDesc,
               "fa_block_mask": _lib.BlockMaskC, "fa_tensor": _lib.TensorC,
               "fa_page_table": _lib.PageTableC, "fa_fwd_args": _lib.FwdArgs,
               "fa_bwd_args": _lib.BwdArgs, "fa_decode_args": _lib.DecodeArgs,
               "fa_page_pool": _lib.PagePoolC}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", str(src), "-o", str(exe)], check=True)
    got = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, got):
        cname, field, val = line.split()
        py = structs[cname]
        want = C.sizeof(py) if field == "size" else getattr(py, field).offset
        assert int(val) == want, line


def test_status_names():
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    names = {i: lib.fa_status_name(i).decode() for i in (0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 100, 101)}
    assert names[1] == "ShapeMismatch" and names[6] == "BlockMaskMismatch" and names[10] == "UnmappedBlock"
    assert lib.fa_abi_version() == 6  # v3 flags/counters/events/check_finite; v4 page pool; v5 remap_rc; v6 async convert


def test_geometry_validation():
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    r, c, w = C.c_int64(), C.c_int64(), C.c_size_t()
    assert lib.fa_block_mask_geometry(1, 1, 1000, 777, 128, 64, C.byref(r), C.byref(c), C.byref(w)) == 0
    assert (r.value, c.value, w.value) == (8, 13, 104)
    assert lib.fa_block_mask_geometry(0, 1, 10, 10, 16, 16, None, None, None) == 1  # make_empty :30-32
    assert lib.fa_block_mask_geometry(1, 1, 0, 10, 16, 16, None, None, None) == 1   # :33-35
    assert b"lengths" in lib.fa_last_error()


def _tensor(b, h, l, d, dtype=1):
    from paper_2412_05496_b200 import _lib
    t = _lib.TensorC()
    t.data, t.dtype, t.b, t.h, t.l, t.d = 0x1000, dtype, b, h, l, d
    return t


def _fwd_args(**kw):
    from paper_2412_05496_b200 import _lib
    a = _lib.FwdArgs()
    a.q, a.k, a.v, a.out = _tensor(1, 4, 256, 128), _tensor(1, 4, 256, 128), _tensor(1, 4, 256, 128), _tensor(1, 4, 256, 128)
    a.lse = 0x2000
    bm = _lib.BlockMaskC()
    bm.b_dims = bm.h_dims = 1
    bm.rows = bm.cols = 2
    bm.bs_q = bm.bs_kv = 128
    bm.q_len = bm.kv_len = 256
    bm.kv_num_blocks = bm.kv_indices = bm.full_kv_num_blocks = bm.full_kv_indices = 0x3000
    a._bm = bm
    a.bm = C.pointer(bm)
    a.gqa_group = 1
    for k, v in kw.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize("mutate,status", [
    (lambda a: setattr(a, "k", _tensor(1, 4, 256, 64)), 1),                   # validate_shapes
    (lambda a: setattr(a, "gqa_group", 3), 1),                                # H_q != G * H_kv
    (lambda a: setattr(a._bm, "q_len", 512), 6),                              # check_block_mask
    (lambda a: setattr(a._bm, "b_dims", 3), 6),
    (lambda a: (setattr(a.score, "terms", 2), setattr(a.score, "cap", 0.0)), 4),   # soft_cap cap <= 0
    (lambda a: (setattr(a.score, "terms", 1), setattr(a.score, "slopes", 0x10), setattr(a.score, "num_slopes", 2)), 3),
    (lambda a: (setattr(a.mask, "terms", 4), setattr(a.mask, "doc_ids", 0x10), setattr(a.mask, "doc_len", 100)), 3),
    (lambda a: (setattr(a.mask, "terms", 2), setattr(a.mask, "window", -1)), 3),
    (lambda a: setattr(a.q, "dtype", 7), 101),
])
def test_forward_validation_errors(mutate, status):
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    a = _fwd_args()
    mutate(a)
    assert lib.fa_flex_fwd(C.byref(a), None) == status
    assert lib.fa_last_error()  # message set


def test_null_args():
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    assert lib.fa_flex_fwd(None, None) == 1
    assert lib.fa_flex_bwd(None, None) == 1
    assert lib.fa_flex_decode(None, None) == 1


def test_python_api_errors():
    import paper_2412_05496_b200 as fa
    with pytest.raises(fa.IndexOutOfRange):
        fa.sliding_window(-1)
    with pytest.raises(fa.NonPositiveCap):
        fa.soft_cap(0.0)
    with pytest.raises(fa.IndexOutOfRange):
        fa.alibi_slopes(0)
    with pytest.raises(fa.Unsupported):
        fa.compose(fa.alibi([1.0]), fa.soft_cap(2.0))
    m = fa.and_mask(fa.causal(), fa.sliding_window(9))
    assert m.terms == fa.MASK_CAUSAL | fa.MASK_SLIDING and m.window == 9
    s = fa.compose(fa.soft_cap(5.0), fa.alibi([0.5]))
    assert s.terms == 3 and s.cap == 5.0
    assert fa.offset_mask(fa.causal(), 7).q_offset == 7


def test_no_cpu_path():
    import torch

    import paper_2412_05496_b200 as fa
    x = torch.zeros((1, 1, 128, 128), dtype=torch.bfloat16)
    with pytest.raises((fa.Unsupported, fa.CudaError, RuntimeError)):
        fa.forward(x, x, x, fa.noop_score(), None or fa.BlockMask(1, 1, 1, 1, 128, 128, 128, 128, x, x, x, x,
                                                                   mask=fa.causal()))


def test_forward_unknown_flags():
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    a = _fwd_args()
    a.flags = 0x80
    assert lib.fa_flex_fwd(C.byref(a), None) == 1
    assert b"flags" in lib.fa_last_error()


def _bwd_args():
    from paper_2412_05496_b200 import _lib
    a = _lib.BwdArgs()
    t = lambda: _tensor(1, 4, 256, 128)  # noqa: E731
    a.q, a.k, a.v, a.out, a.d_out, a.dq, a.dk, a.dv = t(), t(), t(), t(), t(), t(), t(), t()
    a.lse = 0x2000
    bm = _lib.BlockMaskC()
    bm.b_dims = bm.h_dims = 1
    bm.rows = bm.cols = 2
    bm.bs_q = bm.bs_kv = 128
    bm.q_len = bm.kv_len = 256
    for f in ("kv_num_blocks", "kv_indices", "full_kv_num_blocks", "full_kv_indices", "q_num_blocks",
              "q_indices", "full_q_num_blocks", "full_q_indices"):
        setattr(bm, f, 0x3000)
    a._bm = bm
    a.bm = C.pointer(bm)
    a.gqa_group = 1
    a.workspace = 0x4000
    a.workspace_bytes = 1 << 30
    return a


@pytest.mark.parametrize("mutate,status", [
    (lambda a: setattr(a, "dq", _tensor(1, 4, 128, 128)), 1),           # dq must match q
    (lambda a: setattr(a, "dk", _tensor(1, 4, 256, 64)), 1),            # dk must match k
    (lambda a: setattr(a, "dv", _tensor(1, 4, 256, 128, dtype=0)), 1),  # dtype of dv
    (lambda a: setattr(a, "d_out", _tensor(1, 4, 256, 128, dtype=0)), 1),
    (lambda a: setattr(a, "out", _tensor(1, 4, 255, 128)), 7),          # StaleStatistics
    (lambda a: setattr(a._bm, "q_indices", None), 6),                    # q side required
    (lambda a: setattr(a, "workspace_bytes", 16), 1),
    (lambda a: setattr(a, "flags", 0x40), 1),
])
def test_backward_validation_errors(mutate, status):
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    a = _bwd_args()
    mutate(a)
    assert lib.fa_flex_bwd(C.byref(a), None) == status
    assert lib.fa_last_error()


def _decode_args(paged=False):
    from paper_2412_05496_b200 import _lib
    a = _lib.DecodeArgs()
    a.q, a.out = _tensor(2, 4, 1, 128), _tensor(2, 4, 1, 128)
    a.k_cache = a.v_cache = _tensor(1 if paged else 2, 4, 1024, 128)
    a.lse = 0x2000
    bm = _lib.BlockMaskC()
    bm.b_dims, bm.h_dims, bm.rows, bm.cols = (2 if paged else 1), 1, 1, 8
    bm.bs_q = bm.bs_kv = 128
    bm.q_len, bm.kv_len = 1, 1024
    bm.kv_num_blocks = bm.kv_indices = bm.full_kv_num_blocks = bm.full_kv_indices = 0x3000
    a._bm = bm
    a.bm = C.pointer(bm)
    if paged:
        pt = _lib.PageTableC()
        pt.batches, pt.max_logical_pages, pt.num_physical_pages, pt.page_size = 2, 8, 8, 128
        pt.table = pt.phys_to_logical = pt.owner = pt.seq_len = 0x5000
        a._pt = pt
        a.pt = C.pointer(pt)
    a.offset = 1023
    a.gqa_group = 1
    a.workspace = 0x4000
    a.workspace_bytes = 1 << 30
    return a


@pytest.mark.parametrize("paged", [False, True])
@pytest.mark.parametrize("mutate,status", [
    (lambda a: setattr(a, "bm", None), 6),                              # NULL mask checked first
    (lambda a: setattr(a, "out", _tensor(2, 4, 2, 128)), 1),            # out must match q
    (lambda a: setattr(a, "out", _tensor(2, 4, 1, 128, dtype=0)), 1),
    (lambda a: setattr(a, "offset", 1024), 8),                          # OffsetOutOfRange
    (lambda a: (setattr(a.mask, "remap", 0x10), setattr(a.mask, "remap_len", 512)), 3),  # kv range
    (lambda a: (setattr(a.mask, "terms", 4), setattr(a.mask, "doc_ids", 0x10),
                setattr(a.mask, "doc_len", 1000)), 3),
    (lambda a: setattr(a._bm, "h_dims", 3), 6),
])
def test_decode_validation_errors(paged, mutate, status):
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    a = _decode_args(paged)
    mutate(a)
    assert lib.fa_flex_decode(C.byref(a), None) == status, lib.fa_last_error()
    assert lib.fa_last_error()


def test_paged_decode_mask_range_uses_max_seq_len():
    # the mask is evaluated only below the sequences' lengths: a table spanning max_seq_len is
    # enough even when the page table has room for more logical pages
    from paper_2412_05496_b200 import _lib
    lib = _lib.load()
    a = _decode_args(paged=True)
    a.offset = 299
    a.mask.remap, a.mask.remap_len = 0x10, 300
    a._pt.max_seq_len = 300
    a.flags = 0x80  # stop right after argument validation (unknown flag)
    assert lib.fa_flex_decode(C.byref(a), None) == 1
    assert b"flags" in lib.fa_last_error()
    a._pt.max_seq_len = 0  # unknown: the whole logical page range must be covered
    assert lib.fa_flex_decode(C.byref(a), None) == 3


def test_user_functor_library_built():
    """tests/cpp/custom_mods.cu instantiates the kernels with user functors through the public
    templated header (include/flexattn_b200_device.cuh); build() compiles it for sm_100a."""
    so = os.path.join(ROOT, "tests", "cpp", "libcustom_mods.so")
    assert os.path.exists(so), "run __graft_entry__.build()"
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    for sym in ("cm_create_block_mask", "cm_forward", "cm_backward", "cm_decode"):
        assert f" T {sym}" in out
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass  # the tcgen05 / TMA kernels, not a CUDA-core stand-in
