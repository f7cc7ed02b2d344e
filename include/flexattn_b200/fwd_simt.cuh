// fwd_simt.cuh — exact-arithmetic (fp32 FFMA) block-sparse forward.
//
// Serves the fp32 configuration (BASELINE config C1, gate 1e-4 vs the
// reference forward<float>) and every geometry the tensor-core kernel is not
// instantiated for (block sizes other than 128, head dims other than 64/128,
// fp32 I/O). Same traversal as forward_impl (engine.cpp:46-163): per query row,
// visited blocks in ascending merged order, mask only in partial blocks,
// score_mod on every live score, online max/sum, lse = m + ln l, empty rows
// give O = 0 / lse = -inf.
//
// One CTA = min(bs_q, 128) consecutive query rows of one (b, h) inside one
// block row (so all threads share a visit list); K/V blocks are staged through
// shared memory 32 rows at a time and reused by every row of the CTA.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "host.cuh"
#include "mods.cuh"

namespace fa {
namespace fsimt {
namespace {  // internal linkage: every including translation unit has its own copy

constexpr int kChunk = 32;

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

template <typename T, int MAXD, class MaskT, class ScoreT>
__global__ void __launch_bounds__(128) fwd_simt_kernel(AttnGeom g, const T* __restrict__ q,
                                                       const T* __restrict__ k,
                                                       const T* __restrict__ v, T* __restrict__ o,
                                                       float* __restrict__ lse, BmView bm,
                                                       MaskT mask, ScoreT score) {
  __shared__ float ks[kChunk][MAXD + 1];
  __shared__ float vs[kChunk][MAXD];
  const int rows_per_cta = min(g.bs_q, 128);
  const int ctas_per_row = (g.bs_q + rows_per_cta - 1) / rows_per_cta;
  const int r = blockIdx.x / ctas_per_row;
  const int sub = blockIdx.x % ctas_per_row;
  const int bh = blockIdx.y;
  const int b = bh / g.Hq, h = bh % g.Hq;
  const int tid = threadIdx.x;
  const int qi = r * g.bs_q + sub * rows_per_cta + tid;
  const bool active = tid < rows_per_cta && (sub * rows_per_cta + tid) < g.bs_q && qi < g.Lq;
  const int D = g.D;
  const int kb = g.Bkv == 1 ? 0 : b, kh = h / g.G;
  const int mb = g.bm_b == 1 ? 0 : b, mh = g.bm_h == 1 ? 0 : h;
  const long long row_slot = (static_cast<long long>(mb) * g.bm_h + mh) * g.rows + r;
  const int np = bm.kv_num[row_slot], nf = bm.full_num[row_slot];
  const int32_t* pidx = bm.kv_idx + row_slot * g.cols;
  const int32_t* fidx = bm.full_idx + row_slot * g.cols;

  float qr[MAXD], acc[MAXD];
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    qr[d] = (active && d < D) ? to_f(q[((static_cast<long long>(b) * g.Hq + h) * g.Lq + qi) * D + d]) : 0.f;
    acc[d] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const T* kbase = k + (static_cast<long long>(kb) * g.Hkv + kh) * g.Lkv * D;
  const T* vbase = v + (static_cast<long long>(kb) * g.Hkv + kh) * g.Lkv * D;

  int ip = 0, jf = 0;
  while (ip < np || jf < nf) {  // ascending merge = reference visit order
    const bool take_full = ip >= np || (jf < nf && fidx[jf] < pidx[ip]);
    const int c = take_full ? fidx[jf++] : pidx[ip++];
    const int j0 = c * g.bs_kv, j1 = min(j0 + g.bs_kv, g.Lkv);
    for (int jc = j0; jc < j1; jc += kChunk) {
      const int n = min(kChunk, j1 - jc);
      __syncthreads();
      for (int e = tid; e < kChunk * D; e += blockDim.x) {
        const int jj = e / D, d = e % D;
        const bool in = jj < n;
        ks[jj][d] = in ? to_f(kbase[static_cast<long long>(jc + jj) * D + d]) : 0.f;
        vs[jj][d] = in ? to_f(vbase[static_cast<long long>(jc + jj) * D + d]) : 0.f;
      }
      __syncthreads();
      if (!active) continue;
      for (int jj = 0; jj < n; ++jj) {
        const int kv = jc + jj;
        if (!take_full && !(kv < g.Lkv && mask(b, h, qi, kv))) continue;  // bounds + mask_mod
        float dot = 0.f;
#pragma unroll
        for (int d = 0; d < MAXD; ++d) dot = fmaf(qr[d], ks[jj][d], dot);
        const float s = score.apply(dot * g.scale, b, h, qi, kv);
        if (s > m) {  // rescale when the running max grows (engine.cpp:124-134)
          const float alpha = (m == -INFINITY) ? 0.f : expf(m - s);
          l *= alpha;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) acc[d] *= alpha;
          m = s;
        }
        const float p = expf(s - m);
        l += p;
#pragma unroll
        for (int d = 0; d < MAXD; ++d) acc[d] = fmaf(p, vs[jj][d], acc[d]);
      }
    }
  }
  if (!active) return;
  const long long slot = (static_cast<long long>(b) * g.Hq + h) * g.Lq + qi;
  T* orow = o + slot * D;
  if (l > 0.f) {
    const float inv = 1.f / l;
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < D) orow[d] = from_f<T>(acc[d] * inv);
    lse[slot] = m + logf(l);
  } else {
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < D) orow[d] = from_f<T>(0.f);
    lse[slot] = -INFINITY;
  }
}

template <typename T, int MAXD, class MaskT, class ScoreT>
fa_status run(const AttnGeom& g, const void* q, const void* k, const void* v, void* o, float* lse,
              const BmView& bm, MaskT m, ScoreT s, cudaStream_t st) {
  const int rows_per_cta = g.bs_q < 128 ? g.bs_q : 128;
  const int ctas_per_row = (g.bs_q + rows_per_cta - 1) / rows_per_cta;
  dim3 grid(g.rows * ctas_per_row, g.B * g.Hq);
  fwd_simt_kernel<T, MAXD, MaskT, ScoreT><<<grid, 128, 0, st>>>(
      g, static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v),
      static_cast<T*>(o), lse, bm, m, s);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

// run with the smallest compiled head-dim bound >= D
template <typename T, class MaskT, class ScoreT>
fa_status run_any_dim(const AttnGeom& g, const void* q, const void* k, const void* v, void* o, float* lse,
                      const BmView& bm, MaskT m, ScoreT s, cudaStream_t st) {
  if (g.D <= 16) return run<T, 16>(g, q, k, v, o, lse, bm, m, s, st);
  if (g.D <= 64) return run<T, 64>(g, q, k, v, o, lse, bm, m, s, st);
  if (g.D <= 128) return run<T, 128>(g, q, k, v, o, lse, bm, m, s, st);
  return set_error(FA_UNSUPPORTED, "forward: head dim > 128 not compiled");
}

}  // namespace
}  // namespace fsimt
}  // namespace fa
