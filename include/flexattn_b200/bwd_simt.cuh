// bwd_simt.cuh — recomputation backward on CUDA cores, the exact-arithmetic
// path for fp32 tensors and for geometries the tensor-core backward is not
// instantiated for. Mirrors backward (engine.cpp:174-401) pass for pass:
//   delta  : Δ_i = Σ_d dO·O                         (engine.cpp:218-235)
//   dq     : warp per query row over the kv-side visit list (:237-305)
//   dk/dv  : warp per kv row over the q-side (transposed) visit list, looping
//            the kv-batch broadcast and the G query heads of the group (:307-395)
// Lanes split the head dim; dot products reduce with warp shuffles.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "host.cuh"
#include "mods.cuh"

namespace fa {
namespace bsimt {
namespace {  // internal linkage: every including translation unit has its own copy

template <typename T>
__device__ __forceinline__ float ld(const T* p);
template <>
__device__ __forceinline__ float ld<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <typename T>
__device__ __forceinline__ void st(T* p, float v);
template <>
__device__ __forceinline__ void st<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void st<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <typename T>
__global__ void delta_kernel(const T* __restrict__ o, const T* __restrict__ dout, int rows, int D,
                             float* __restrict__ delta) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float a = 0.f;
  for (int d = lane; d < D; d += 32)
    a += ld(o + static_cast<long long>(row) * D + d) * ld(dout + static_cast<long long>(row) * D + d);
  a = warp_sum(a);
  if (lane == 0) delta[row] = a;
}

template <typename T, int MAXP, class MaskT, class ScoreT>
__global__ void dq_kernel(AttnGeom g, const T* __restrict__ q, const T* __restrict__ k,
                          const T* __restrict__ v, const float* __restrict__ lse,
                          const T* __restrict__ dout, const float* __restrict__ delta,
                          T* __restrict__ dq, BmView bm, MaskT mask, ScoreT score) {
  const int lane = threadIdx.x & 31;
  const long long row = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= (long long)g.B * g.Hq * g.Lq) return;
  const int qi = (int)(row % g.Lq);
  const int h = (int)((row / g.Lq) % g.Hq);
  const int b = (int)(row / ((long long)g.Lq * g.Hq));
  const int D = g.D;
  float qv[MAXP], dov[MAXP], acc[MAXP];
#pragma unroll
  for (int e = 0; e < MAXP; ++e) {
    const int d = lane + 32 * e;
    qv[e] = d < D ? ld(q + row * D + d) : 0.f;
    dov[e] = d < D ? ld(dout + row * D + d) : 0.f;
    acc[e] = 0.f;
  }
  const float lse_i = lse[row];
  if (lse_i != -INFINITY) {
    const float di = delta[row];
    const int r = qi / g.bs_q;
    const int kb = g.Bkv == 1 ? 0 : b, kh = h / g.G;
    const int mb = g.bm_b == 1 ? 0 : b, mh = g.bm_h == 1 ? 0 : h;
    const long long slot = ((long long)mb * g.bm_h + mh) * g.rows + r;
    const int np = bm.kv_num[slot], nf = bm.full_num[slot];
    const int32_t* pi = bm.kv_idx + slot * g.cols;
    const int32_t* fi = bm.full_idx + slot * g.cols;
    const T* kbase = k + ((long long)kb * g.Hkv + kh) * g.Lkv * D;
    const T* vbase = v + ((long long)kb * g.Hkv + kh) * g.Lkv * D;
    int ip = 0, jf = 0;
    while (ip < np || jf < nf) {
      const bool full = ip >= np || (jf < nf && fi[jf] < pi[ip]);
      const int c = full ? fi[jf++] : pi[ip++];
      const int j1 = min((c + 1) * g.bs_kv, g.Lkv);
      for (int j = c * g.bs_kv; j < j1; ++j) {
        if (!full && !mask(b, h, qi, j)) continue;
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < MAXP; ++e) {
          const int d = lane + 32 * e;
          if (d < D) {
            s += qv[e] * ld(kbase + (long long)j * D + d);
            dp += dov[e] * ld(vbase + (long long)j * D + d);
          }
        }
        s = warp_sum(s) * g.scale;
        dp = warp_sum(dp);
        const float x = score.apply(s, b, h, qi, j);
        const float p = expf(x - lse_i);
        const float coeff = p * (dp - di) * score.grad(s, b, h, qi, j) * g.scale;
#pragma unroll
        for (int e = 0; e < MAXP; ++e) {
          const int d = lane + 32 * e;
          if (d < D) acc[e] = fmaf(coeff, ld(kbase + (long long)j * D + d), acc[e]);
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < MAXP; ++e) {
    const int d = lane + 32 * e;
    if (d < D) st(dq + row * D + d, acc[e]);
  }
}

template <typename T, int MAXP, class MaskT, class ScoreT>
__global__ void dkdv_kernel(AttnGeom g, const T* __restrict__ q, const T* __restrict__ k,
                            const T* __restrict__ v, const float* __restrict__ lse,
                            const T* __restrict__ dout, const float* __restrict__ delta,
                            T* __restrict__ dk, T* __restrict__ dv, BmView bmt, MaskT mask,
                            ScoreT score) {
  const int lane = threadIdx.x & 31;
  const long long krow = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (krow >= (long long)g.Bkv * g.Hkv * g.Lkv) return;
  const int j = (int)(krow % g.Lkv);
  const int kh = (int)((krow / g.Lkv) % g.Hkv);
  const int ob = (int)(krow / ((long long)g.Lkv * g.Hkv));
  const int D = g.D;
  float kv_[MAXP], vv[MAXP], dka[MAXP], dva[MAXP];
#pragma unroll
  for (int e = 0; e < MAXP; ++e) {
    const int d = lane + 32 * e;
    kv_[e] = d < D ? ld(k + krow * D + d) : 0.f;
    vv[e] = d < D ? ld(v + krow * D + d) : 0.f;
    dka[e] = dva[e] = 0.f;
  }
  const int c = j / g.bs_kv;
  const int b_begin = g.Bkv == 1 ? 0 : ob, b_end = g.Bkv == 1 ? g.B : ob + 1;
  for (int b = b_begin; b < b_end; ++b) {
    for (int gi = 0; gi < g.G; ++gi) {
      const int h = kh * g.G + gi;
      const int mb = g.bm_b == 1 ? 0 : b, mh = g.bm_h == 1 ? 0 : h;
      const long long slot = ((long long)mb * g.bm_h + mh) * g.cols + c;  // q-side row = kv column
      const int np = bmt.kv_num[slot], nf = bmt.full_num[slot];
      const int32_t* pi = bmt.kv_idx + slot * g.rows;
      const int32_t* fi = bmt.full_idx + slot * g.rows;
      int ip = 0, jf = 0;
      while (ip < np || jf < nf) {
        const bool full = ip >= np || (jf < nf && fi[jf] < pi[ip]);
        const int r = full ? fi[jf++] : pi[ip++];
        const int i1 = min((r + 1) * g.bs_q, g.Lq);
        for (int qi = r * g.bs_q; qi < i1; ++qi) {
          const long long qrow = ((long long)b * g.Hq + h) * g.Lq + qi;
          const float lse_i = lse[qrow];
          if (lse_i == -INFINITY) continue;
          if (!full && !mask(b, h, qi, j)) continue;
          float s = 0.f, dp = 0.f;
          float qq[MAXP], dd[MAXP];
#pragma unroll
          for (int e = 0; e < MAXP; ++e) {
            const int d = lane + 32 * e;
            qq[e] = d < D ? ld(q + qrow * D + d) : 0.f;
            dd[e] = d < D ? ld(dout + qrow * D + d) : 0.f;
            s += qq[e] * kv_[e];
            dp += dd[e] * vv[e];
          }
          s = warp_sum(s) * g.scale;
          dp = warp_sum(dp);
          const float x = score.apply(s, b, h, qi, j);
          const float p = expf(x - lse_i);
          const float coeff = p * (dp - delta[qrow]) * score.grad(s, b, h, qi, j) * g.scale;
#pragma unroll
          for (int e = 0; e < MAXP; ++e) {
            dva[e] = fmaf(p, dd[e], dva[e]);
            dka[e] = fmaf(coeff, qq[e], dka[e]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < MAXP; ++e) {
    const int d = lane + 32 * e;
    if (d < D) {
      st(dk + krow * D + d, dka[e]);
      st(dv + krow * D + d, dva[e]);
    }
  }
}

template <typename T, int MAXP, class MaskT, class ScoreT>
fa_status run(const AttnGeom& g, const void* q, const void* k, const void* v, const void* o,
              const float* lse, const void* dout, void* dq, void* dk, void* dv, const BmView& bm,
              const BmView& bmt, MaskT mask, ScoreT score, float* delta, cudaStream_t s) {
  const long long qrows = (long long)g.B * g.Hq * g.Lq;
  delta_kernel<T><<<(unsigned)((qrows + 7) / 8), 256, 0, s>>>(static_cast<const T*>(o),
                                                              static_cast<const T*>(dout),
                                                              (int)qrows, g.D, delta);
  dq_kernel<T, MAXP><<<(unsigned)((qrows + 7) / 8), 256, 0, s>>>(
      g, static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v), lse,
      static_cast<const T*>(dout), delta, static_cast<T*>(dq), bm, mask, score);
  const long long krows = (long long)g.Bkv * g.Hkv * g.Lkv;
  dkdv_kernel<T, MAXP><<<(unsigned)((krows + 7) / 8), 256, 0, s>>>(
      g, static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v), lse,
      static_cast<const T*>(dout), delta, static_cast<T*>(dk), static_cast<T*>(dv), bmt, mask, score);
  count_launch(3);
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

// The CUDA-core passes for any dtype / head dim <= 128 (deterministic by construction: separate
// dq pass, no atomics). Workspace layout (fa_bwd_workspace_size): [dq_acc | delta | lse2]; only
// delta is used here.
template <class MaskT, class ScoreT>
fa_status run_any(const AttnGeom& g, const void* q, const void* k, const void* v, const void* o,
                  const float* lse, const void* dout, void* dq, void* dk, void* dv, int dtype, const BmView& bm,
                  const BmView& bmt, MaskT mask, ScoreT score, void* workspace, cudaStream_t st) {
  const size_t rows = (size_t)g.B * g.Hq * g.Lq;
  const size_t off = ((rows * g.D * 4) + 255) & ~size_t(255);
  float* delta = reinterpret_cast<float*>(static_cast<char*>(workspace) + off);
  FA_REQUIRE(g.D <= 128, FA_UNSUPPORTED, "backward: head dim > 128 not compiled");
  if (dtype == FA_F32) {
    if (g.D <= 32) return run<float, 1>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mask, score, delta, st);
    return run<float, 4>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mask, score, delta, st);
  }
  if (g.D <= 32) return run<__nv_bfloat16, 1>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mask, score, delta, st);
  return run<__nv_bfloat16, 4>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mask, score, delta, st);
}

}  // namespace
}  // namespace bsimt
}  // namespace fa
