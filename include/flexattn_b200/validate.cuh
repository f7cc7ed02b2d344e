// validate.cuh — data-dependent checks and work counters of the reference, on the device.
//
//  * finite_scan_kernel: the NaN/inf scans of validate_inputs (validate.hpp:36-38) and of the
//    backward's d_out (engine.cpp:196), several tensors in one grid-stride pass with 16-byte
//    loads (exponent-field test per element: bf16 0x7f80, fp32 0x7f800000). HBM-bound.
//  * counters_kernel: OpCounters (engine.hpp:21-32) computed from the BlockMask and the mask
//    instead of by instrumenting the attention kernels: one warp per query row walks the row's
//    visited tiles; partial tiles count their in-bounds positions (mask evaluations) and the
//    popcount of the mask words (live positions); full tiles count bs_kv live positions.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "host.cuh"
#include "mods.cuh"

namespace fa {
namespace {  // internal linkage: every including translation unit has its own copy

constexpr int kMaxScan = 8;
struct ScanList {
  const void* ptr[kMaxScan];
  long long n[kMaxScan];   // elements
  int dtype[kMaxScan];
  int count;
};

__device__ __forceinline__ bool nonfinite_bf16x2(uint32_t w) {
  const uint32_t t = w & 0x7f807f80u;
  return (t & 0xffffu) == 0x7f80u || (t >> 16) == 0x7f80u;
}
__device__ __forceinline__ bool nonfinite_f32(uint32_t w) { return (w & 0x7f800000u) == 0x7f800000u; }

__global__ void __launch_bounds__(256) finite_scan_kernel(ScanList L, int* __restrict__ flags) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  for (int t = 0; t < L.count; ++t) {
    const int esz = L.dtype[t] == FA_F32 ? 4 : 2;
    const long long n = L.n[t];
    const uintptr_t base = reinterpret_cast<uintptr_t>(L.ptr[t]);
    const bool aligned = (base & 15u) == 0;
    const long long per16 = 16 / esz;
    const long long nvec = aligned ? n / per16 : 0;
    bool bad = false;
    const uint4* v = reinterpret_cast<const uint4*>(L.ptr[t]);
    for (long long i = tid; i < nvec; i += nthreads) {
      const uint4 x = __ldg(v + i);
      if (esz == 2) {
        bad |= nonfinite_bf16x2(x.x) | nonfinite_bf16x2(x.y) | nonfinite_bf16x2(x.z) | nonfinite_bf16x2(x.w);
      } else {
        bad |= nonfinite_f32(x.x) | nonfinite_f32(x.y) | nonfinite_f32(x.z) | nonfinite_f32(x.w);
      }
    }
    for (long long i = nvec * per16 + tid; i < n; i += nthreads) {  // tail / unaligned
      if (esz == 2) {
        const uint32_t h = reinterpret_cast<const uint16_t*>(L.ptr[t])[i];
        bad |= (h & 0x7f80u) == 0x7f80u;
      } else {
        bad |= nonfinite_f32(reinterpret_cast<const uint32_t*>(L.ptr[t])[i]);
      }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags + t, 1);
  }
}

struct CountGeom {
  int B, Hq, Lq, Lkv, bm_b, bm_h, rows, cols, bs_q, bs_kv;
  int paged, page_size, logical_kv;
  const int32_t* p2l;
  const int32_t* owner;
  const int32_t* seq_len;
};

// sums: [0] live, [1] partial-tile positions, [2] partial-tile positions of rows with >= 1 live
template <class MaskT>
__global__ void __launch_bounds__(256) counters_kernel(CountGeom g, BmView bm, MaskT mask,
                                                       unsigned long long* __restrict__ sums) {
  __shared__ unsigned long long red[3][8];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nrows = (long long)g.B * g.Hq * g.Lq;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned long long s_live = 0, s_part = 0, s_part_live = 0;
  for (long long row = w0; row < nrows; row += nw) {
    const int iq = (int)(row % g.Lq);
    const int h = (int)((row / g.Lq) % g.Hq);
    const int b = (int)(row / ((long long)g.Lq * g.Hq));
    const int r = iq / g.bs_q;
    const int mb = g.bm_b == 1 ? 0 : b, mh = g.bm_h == 1 ? 0 : h;
    const long long slot = ((long long)mb * g.bm_h + mh) * g.rows + r;
    const int np = __ldg(bm.kv_num + slot), nf = __ldg(bm.full_num + slot);
    unsigned long long live = 0, part = 0;
    for (int t = lane; t < np + nf; t += 32) {
      const bool full = t >= np;
      const int c = full ? __ldg(bm.full_idx + slot * g.cols + (t - np)) : __ldg(bm.kv_idx + slot * g.cols + t);
      const int j0 = c * g.bs_kv, j1 = min(j0 + g.bs_kv, g.Lkv);
      if (!g.paged) {
        if (full) {
          live += (unsigned)(j1 - j0);
        } else {
          part += (unsigned)(j1 - j0);
          for (int kv0 = j0; kv0 < j1; kv0 += 32) live += __popc(mask.bits32(b, h, iq, kv0, j1) & range_bits32(kv0, kv0, j1 - 1));
        }
      } else {
        // physical page c of the converted mask: logical positions of its owner (convert_mods)
        if (!full) part += (unsigned)(j1 - j0);
        const int lp = __ldg(g.p2l + c), own = __ldg(g.owner + c);
        if (lp < 0 || own != b) continue;  // foreign: the validated decode rejects it
        const int seq = min(__ldg(g.seq_len + b), g.logical_kv);
        const int l0 = lp * g.page_size, l1 = min(l0 + (j1 - j0), seq);
        for (int kv0 = l0; kv0 < l1; kv0 += 32) {
          const uint32_t in = range_bits32(kv0, kv0, l1 - 1);
          live += __popc(full ? in : (mask.bits32(b, h, iq, kv0, l1) & in));
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      live += __shfl_xor_sync(0xffffffffu, live, o);
      part += __shfl_xor_sync(0xffffffffu, part, o);
    }
    s_live += live;
    s_part += part;
    if (live > 0) s_part_live += part;
  }
  if (lane == 0) {
    red[0][wib] = s_live;
    red[1][wib] = s_part;
    red[2][wib] = s_part_live;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    unsigned long long a = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[threadIdx.x][w];
    if (a) atomicAdd(sums + threadIdx.x, a);
  }
}

template <class MaskT>
fa_status launch_counts(const CountGeom& g, const BmView& bm, MaskT m, unsigned long long* sums,
                        cudaStream_t st) {
  const long long rows = (long long)g.B * g.Hq * g.Lq;
  const int blocks = (int)std::max<long long>(1, std::min<long long>((rows + 7) / 8, 148LL * 8));
  counters_kernel<MaskT><<<blocks, 256, 0, st>>>(g, bm, m, sums);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

// OpCounters of one call (engine.hpp:21-32) from the BlockMask and the mask; synchronises `st`.
template <class MaskT>
fa_status compute_counters(const AttnGeom& a, const BmView& bm, MaskT mask, const PageView* pv, int logical_kv,
                           int pass, fa_op_counters* out, cudaStream_t st) {
  unsigned long long* sums = reinterpret_cast<unsigned long long*>(scheduler_counter(kSlotCounters, st));
  FA_REQUIRE(sums != nullptr, FA_CUDA_ERROR, "counters: cannot allocate the device sums");
  FA_CHECK_CUDA(cudaMemsetAsync(sums, 0, 3 * sizeof(unsigned long long), st));
  CountGeom g{};
  g.B = a.B; g.Hq = a.Hq; g.Lq = a.Lq; g.Lkv = a.Lkv; g.bm_b = a.bm_b; g.bm_h = a.bm_h;
  g.rows = a.rows; g.cols = a.cols; g.bs_q = a.bs_q; g.bs_kv = a.bs_kv;
  g.logical_kv = logical_kv;
  if (pv != nullptr && pv->enabled) {
    g.paged = 1;
    g.page_size = pv->page_size;
    g.p2l = pv->phys_to_logical;
    g.owner = pv->owner;
    g.seq_len = pv->seq_len;
  }
  const fa_status s = launch_counts(g, bm, mask, sums, st);
  if (s != FA_OK) return s;
  unsigned long long h[3] = {0, 0, 0};
  FA_CHECK_CUDA(cudaMemcpyAsync(h, sums, sizeof(h), cudaMemcpyDeviceToHost, st));
  FA_CHECK_CUDA(cudaStreamSynchronize(st));
  const unsigned long long D = static_cast<unsigned long long>(a.D);
  if (pass == kPassBackward) {
    // dq pass + dk/dv pass each evaluate the mask and the score once per position of rows with
    // a finite lse (engine.cpp:257-260, 344); madds: Δ (D per row, :218-235), dq pass 3D per
    // live score (q.k, dO.v, dq += coeff k), dk/dv pass 4D (q.k, dv, dO.v, dk)
    out->mask_evals = 2 * h[2];
    out->score_evals = 2 * h[0];
    out->madds = D * static_cast<unsigned long long>(a.B) * a.Hq * a.Lq + 7 * D * h[0];
  } else {
    out->mask_evals = h[1];
    out->score_evals = h[0];
    out->madds = 2 * D * h[0];  // q.k dot + p.v per live score (rescales not counted)
  }
  return FA_OK;
}

// NaN/inf scan of n tensors (validate.hpp:36-38); synchronises `st`.
inline fa_status check_finite_list(const fa_tensor* ts, const char* const* names, int n, cudaStream_t st) {
  FA_REQUIRE(n >= 0 && n <= kMaxScan, FA_SHAPE_MISMATCH, "check_finite: at most 8 tensors");
  if (n == 0) return FA_OK;
  int* flags = scheduler_counter(kSlotFiniteErr, st);
  FA_REQUIRE(flags != nullptr, FA_CUDA_ERROR, "check_finite: cannot allocate the status words");
  FA_CHECK_CUDA(cudaMemsetAsync(flags, 0, kMaxScan * sizeof(int), st));
  ScanList L{};
  long long total = 0;
  for (int i = 0; i < n; ++i) {
    FA_REQUIRE(ts[i].data != nullptr && (ts[i].dtype == FA_F32 || ts[i].dtype == FA_BF16),
               FA_SHAPE_MISMATCH, "check_finite: bad tensor");
    L.ptr[i] = ts[i].data;
    L.n[i] = ts[i].b * ts[i].h * ts[i].l * ts[i].d;
    L.dtype[i] = ts[i].dtype;
    total += L.n[i];
  }
  L.count = n;
  const int blocks = (int)std::max<long long>(1, std::min<long long>((total / 8 + 255) / 256, 148LL * 8));
  finite_scan_kernel<<<blocks, 256, 0, st>>>(L, flags);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  int h[kMaxScan] = {0};
  FA_CHECK_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, st));
  FA_CHECK_CUDA(cudaStreamSynchronize(st));
  for (int i = 0; i < n; ++i)
    if (h[i])
      return set_error(FA_NON_FINITE_INPUT,
                       std::string("validate_inputs: ") + (names && names[i] ? names[i] : std::to_string(i).c_str()) +
                           " contains NaN or inf");
  return FA_OK;
}
}  // namespace
}  // namespace fa
