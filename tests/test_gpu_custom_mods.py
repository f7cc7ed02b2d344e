"""GPU: user-defined mask_mod / score_mod functors (the reference's any-callable modifiers,
modifiers.hpp:17-40) instantiating the sm100a kernels from a user translation unit through
include/flexattn_b200_device.cuh (tests/cpp/custom_mods.cu -> tests/cpp/libcustom_mods.so).

Checked against a dense fp32 restatement of the same functors: the BlockMask bit for bit
(create_block_mask semantics, block_mask.cpp:79-115: EMPTY / FULL only when every position is
live and the tile is not ragged / PARTIAL, ascending lists, zero tails, q side = transpose), the
forward (O, lse) and, through torch autograd of the restatement, dQ/dK/dV — which exercise the
user score's derivative (score_mod', modifiers.hpp:25-28) — and decode rows."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tests", "cpp", "libcustom_mods.so")
WINDOW, STRIDE, R = 200, 96, 300


@pytest.fixture(scope="module")
def cm():
    if not os.path.exists(SO):
        pytest.fail(f"{SO} not built (__graft_entry__.build())")
    lib = C.CDLL(SO)
    lib.cm_last_error.restype = C.c_char_p
    return lib


def _check(lib, st):
    assert st == 0, (st, lib.cm_last_error())


def dense_mask(Lq, Lkv, off=0):
    q = np.arange(Lq)[:, None] + off
    kv = np.arange(Lkv)[None, :]
    return (q >= kv) & ((q - kv < WINDOW) | (kv % STRIDE == 0))


def expected_lists(M, bs):
    Lq, Lkv = M.shape
    rows, cols = -(-Lq // bs), -(-Lkv // bs)
    kind = np.zeros((rows, cols), np.int8)
    for r in range(rows):
        for c in range(cols):
            t = M[r * bs:(r + 1) * bs, c * bs:(c + 1) * bs]
            ragged = t.shape != (bs, bs)
            kind[r, c] = 0 if not t.any() else (2 if t.all() and not ragged else 1)

    def lists(K):
        n, m = K.shape
        pn, pi = np.zeros(n, np.int32), np.zeros((n, m), np.int32)
        fn, fi = np.zeros(n, np.int32), np.zeros((n, m), np.int32)
        for i in range(n):
            p, f = np.nonzero(K[i] == 1)[0], np.nonzero(K[i] == 2)[0]
            pn[i], fn[i] = len(p), len(f)
            pi[i, :len(p)], fi[i, :len(f)] = p, f
        return pn, pi.ravel(), fn, fi.ravel()
    return lists(kind), lists(kind.T)


def build_mask(fa, cm, Lq, Lkv, dev, bs=128):
    bm = fa.create_block_mask(fa.noop_mask(), 1, 1, Lq, Lkv, bs, bs, device=dev)  # allocation
    rows, cols = bm.rows, bm.cols
    work = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
    for t in (bm.kv_num_blocks, bm.kv_indices, bm.full_kv_num_blocks, bm.full_kv_indices,
              bm.q_num_blocks, bm.q_indices, bm.full_q_num_blocks, bm.full_q_indices):
        t.fill_(-7)  # the user build must overwrite every element (tails included)
    cbm = bm.c()
    _check(cm, cm.cm_create_block_mask(WINDOW, STRIDE, C.c_int64(Lq), C.c_int64(Lkv), C.c_int64(bs), C.byref(cbm),
                                       C.c_void_p(work.data_ptr()), C.c_size_t(rows * cols),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return bm


def tables(H, dev):
    g = torch.Generator().manual_seed(5)
    bias = (torch.rand(R + 1, generator=g) * 2 - 1).to(dev)
    cap = (torch.rand(H, generator=g) * 10 + 5).to(dev)
    return bias, cap


def reference(q, k, v, bias, cap, G, unit, off=0, scale=None):
    """dense fp32 restatement of the user functors (autograd gives score_mod')."""
    B, Hq, Lq, D = q.shape
    Lkv = k.shape[2]
    scale = scale or 1.0 / np.sqrt(D)
    kk = k.repeat_interleave(G, dim=1)
    vv = v.repeat_interleave(G, dim=1)
    s = torch.einsum("bhqd,bhkd->bhqk", q, kk) * scale
    qi = torch.arange(Lq, device=q.device)[:, None] + off
    ki = torch.arange(Lkv, device=q.device)[None, :]
    x = s + bias[(qi - ki).clamp(0, R)]
    if not unit:
        c = cap.view(1, Hq, 1, 1)
        x = c * torch.tanh(x / c)
    M = torch.from_numpy(dense_mask(Lq, Lkv, off)).to(q.device)
    x = x.masked_fill(~M, float("-inf"))
    lse = torch.logsumexp(x, dim=-1)
    o = torch.einsum("bhqk,bhkd->bhqd", torch.softmax(x, dim=-1), vv)
    return o, lse


def _fwd_args(fa, q, k, v, out, lse, bm, G):
    from paper_2412_05496_b200 import _lib
    from paper_2412_05496_b200.api import _tensor
    a = _lib.FwdArgs()
    a.q, a.k, a.v, a.out = _tensor(q, "q"), _tensor(k, "k"), _tensor(v, "v"), _tensor(out, "out")
    a.lse = lse.data_ptr()
    a._bm = bm.c()
    a.bm = C.pointer(a._bm)
    a.gqa_group = G
    return a


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("Lq,Lkv", [(640, 640), (1000, 1000), (300, 777)])
def test_block_mask_bit_exact(fa, cm, dev, Lq, Lkv):
    bm = build_mask(fa, cm, Lq, Lkv, dev)
    (pn, pi, fn, fi), (tpn, tpi, tfn, tfi) = expected_lists(dense_mask(Lq, Lkv), 128)
    for got, want in ((bm.kv_num_blocks, pn), (bm.kv_indices, pi), (bm.full_kv_num_blocks, fn),
                      (bm.full_kv_indices, fi), (bm.q_num_blocks, tpn), (bm.q_indices, tpi),
                      (bm.full_q_num_blocks, tfn), (bm.full_q_indices, tfi)):
        assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("unit", [0, 1])
@pytest.mark.parametrize("dtype,L,D,G,tol", [(torch.bfloat16, 640, 128, 2, 2e-2), (torch.bfloat16, 384, 64, 1, 2e-2),
                                             (torch.float32, 200, 64, 1, 1e-4)])
def test_forward_backward_vs_dense(fa, cm, dev, unit, dtype, L, D, G, tol):
    B, Hkv = 1, 2
    Hq = Hkv * G
    bs = 128 if dtype == torch.bfloat16 else 64
    q = fa.random_tensor(71, (B, Hq, L, D), dtype=dtype, device=dev)
    k = fa.random_tensor(72, (B, Hkv, L, D), dtype=dtype, device=dev)
    v = fa.random_tensor(73, (B, Hkv, L, D), dtype=dtype, device=dev)
    do = fa.random_tensor(74, (B, Hq, L, D), dtype=dtype, device=dev)
    bias, cap = tables(Hq, dev)
    bm = build_mask(fa, cm, L, L, dev, bs)
    out, lse = torch.empty_like(q), torch.empty((B, Hq, L), dtype=torch.float32, device=dev)
    a = _fwd_args(fa, q, k, v, out, lse, bm, G)
    _check(cm, cm.cm_forward(C.byref(a), WINDOW, STRIDE, C.c_void_p(bias.data_ptr()), C.c_void_p(cap.data_ptr()),
                             R, unit, _stream()))
    # backward through the C-ABI argument struct
    from paper_2412_05496_b200 import _lib
    from paper_2412_05496_b200.api import _tensor
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = _lib.load().fa_bwd_workspace_size(B, Hq, L, D)
    work = torch.empty(ws, dtype=torch.uint8, device=dev)
    b = _lib.BwdArgs()
    b.q, b.k, b.v, b.out, b.d_out = (_tensor(x, n) for x, n in ((q, "q"), (k, "k"), (v, "v"), (out, "out"), (do, "do")))
    b.lse = lse.data_ptr()
    b.dq, b.dk, b.dv = _tensor(dq, "dq"), _tensor(dk, "dk"), _tensor(dv, "dv")
    b._bm = bm.c()
    b.bm = C.pointer(b._bm)
    b.gqa_group = G
    b.workspace, b.workspace_bytes = work.data_ptr(), ws
    _check(cm, cm.cm_backward(C.byref(b), WINDOW, STRIDE, C.c_void_p(bias.data_ptr()), C.c_void_p(cap.data_ptr()),
                              R, unit, _stream()))
    torch.cuda.synchronize()
    qf, kf, vf = (x.float().clone().requires_grad_(True) for x in (q, k, v))
    o_ref, l_ref = reference(qf, kf, vf, bias, cap, G, unit)
    assert (out.float() - o_ref).abs().max().item() <= tol
    assert (lse - l_ref).abs().max().item() <= tol
    o_ref.backward(do.float())
    for got, want in ((dq, qf.grad), (dk, kf.grad), (dv, vf.grad)):
        rel = (got.float() - want).abs().max().item() / max(1.0, want.abs().max().item())
        assert rel <= tol, rel


def test_decode_rows_vs_dense(fa, cm, dev):
    B, H, L, D, n, off = 2, 2, 900, 128, 3, 600
    q = fa.random_tensor(81, (B, H, L, D), device=dev)
    k = fa.random_tensor(82, (B, H, L, D), device=dev)
    v = fa.random_tensor(83, (B, H, L, D), device=dev)
    bias, cap = tables(H, dev)
    # the BlockMask of the shifted mask at q_len = n (offset_mask, engine.cpp:421-424), built
    # from the dense restatement's tiles (same layout the builder emits)
    (pn, pi, fn, fi), _ = expected_lists(dense_mask(n, L, off), 128)
    bm = fa.create_block_mask(fa.noop_mask(), 1, 1, n, L, device=dev)
    for t, w in ((bm.kv_num_blocks, pn), (bm.kv_indices, pi), (bm.full_kv_num_blocks, fn), (bm.full_kv_indices, fi)):
        t.copy_(torch.from_numpy(w))
    from paper_2412_05496_b200 import _lib
    from paper_2412_05496_b200.api import _tensor
    qs = q[:, :, off:off + n].contiguous()
    out, lse = torch.empty_like(qs), torch.empty((B, H, n), dtype=torch.float32, device=dev)
    ws = _lib.load().fa_decode_workspace_size(B, H, n, D, 0)
    work = torch.empty(ws, dtype=torch.uint8, device=dev)
    a = _lib.DecodeArgs()
    a.q, a.k_cache, a.v_cache, a.out = _tensor(qs, "q"), _tensor(k, "k"), _tensor(v, "v"), _tensor(out, "out")
    a.lse = lse.data_ptr()
    a._bm = bm.c()
    a.bm = C.pointer(a._bm)
    a.offset, a.gqa_group = off, 1
    a.workspace, a.workspace_bytes = work.data_ptr(), ws
    _check(cm, cm.cm_decode(C.byref(a), WINDOW, STRIDE, C.c_void_p(bias.data_ptr()), C.c_void_p(cap.data_ptr()), R,
                            _stream()))
    torch.cuda.synchronize()
    o_ref, l_ref = reference(qs.float(), k.float(), v.float(), bias, cap, 1, 0, off=off)
    assert (out.float() - o_ref).abs().max().item() <= 2e-2
    assert (lse - l_ref).abs().max().item() <= 2e-2
