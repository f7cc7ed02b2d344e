// decode.cuh — split-KV (paged) decode for short query steps, the HBM-bound
// replacement of decode (engine.cpp:403-427) composed with the paged-KV index
// rewrite (convert_block_mask, paged_kv.cpp:154-228) and the logical-position
// recovery of convert_mods (paged_kv.cpp:230-310).
//
// One CTA (4 warps) = one query row x one split of its visit list. The list
// (partial blocks, then full blocks, in stored order — identical for the
// logical and the page-converted mask, so paged == unpaged bit for bit) names
// the K/V tiles; a single thread streams each (K, V) tile pair into a 3-stage
// shared-memory ring with 1-D cp.async.bulk (a page is contiguous: bs_kv rows
// of D bf16 per head), completion tracked by mbarrier transaction counts.
// Warps split the tile's rows in 32-key chunks; lanes split D (conflict-free 8-byte smem
// reads); per chunk a 31-shuffle transposed butterfly turns 32 partial dots into one score
// per lane, one online-softmax update, then P V with broadcast weights; each warp keeps its
// own online-softmax state; states are merged in smem and,
// with more than one split, across splits by a combine kernel.
//
// Paged mode: physical page c -> logical page phys_to_logical[c] of owner[c];
// positions past seq_len (slack) or on a foreign page are masked (the
// reference treats slack as masked and throws on foreign pages; foreign pages
// cannot occur in a mask produced by fa_convert_block_mask).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "host.cuh"
#include "mods.cuh"
#include "sm100_ptx.cuh"

namespace fa {
namespace dec {
namespace {  // internal linkage: every including translation unit has its own copy

constexpr int kStagesDec = 3;
constexpr int kMaxTileBytes = 32768;  // bs_kv * D * 2 <= 32 KiB (page 128 x D 128)
constexpr float kLog2eD = 1.4426950408889634f;

struct DecParams {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  __nv_bfloat16* out;
  float* lse;
  float* part;  // (rows_total, splits, D + 2)
  int B, Hq, Hkv, Bkv, n_new, Lc, D, G;
  int bm_b, bm_h, rows, cols, bs_q, bs_kv;
  const int32_t* kv_num;
  const int32_t* kv_idx;
  const int32_t* full_num;
  const int32_t* full_idx;
  const int32_t* p2l;
  const int32_t* owner;
  const int32_t* seq_len;
  int* foreign;  // optional: set when a visited page is foreign to the row's batch element
  int paged, logical_kv;
  int splits;
  float scale;
};

template <int D>
struct alignas(128) DecSmem {
  uint8_t kv[kStagesDec][2][kMaxTileBytes];
  float q[D];
  float wm[4], wl[4];
  float wacc[4][D];
  uint64_t full[kStagesDec];
};

template <int D, class MaskT, class ScoreT>
__global__ void __launch_bounds__(128, 1) decode_kernel(DecParams p, MaskT mask, ScoreT score) {
  extern __shared__ __align__(128) uint8_t dsm_raw[];
  DecSmem<D>& sm = *reinterpret_cast<DecSmem<D>*>(dsm_raw);
  const int split = blockIdx.x;
  const int qrow = blockIdx.y;
  const int bh = blockIdx.z;
  const int b = bh / p.Hq, h = bh % p.Hq;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kb = p.Bkv == 1 ? 0 : b, kh = h / p.G;
  const int r = qrow / p.bs_q;
  const int mb = p.bm_b == 1 ? 0 : b, mh = p.bm_h == 1 ? 0 : h;
  const long long row_slot = (static_cast<long long>(mb) * p.bm_h + mh) * p.rows + r;
  const int np = __ldg(p.kv_num + row_slot), nf = __ldg(p.full_num + row_slot);
  const int nt = np + nf;
  const int per = (nt + p.splits - 1) / p.splits;
  const int t0 = split * per, t1 = min(nt, t0 + per);
  const int ntiles = max(0, t1 - t0);
  const int32_t* pidx = p.kv_idx + row_slot * p.cols;
  const int32_t* fidx = p.full_idx + row_slot * p.cols;
  const long long head_base = (static_cast<long long>(kb) * p.Hkv + kh) * p.Lc;
  const int tile_rows = p.bs_kv;

  const long long qslot = (static_cast<long long>(b) * p.Hq + h) * p.n_new + qrow;
  for (int d = tid; d < D; d += 128) sm.q[d] = __bfloat162float(p.q[qslot * D + d]);
  if (tid == 0) {
    for (int s = 0; s < kStagesDec; ++s) mbar_init(&sm.full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  auto tile_col = [&](int t) { return t < np ? __ldg(pidx + t) : __ldg(fidx + t - np); };
  auto issue = [&](int i) {  // tile i of this split -> stage i % S
    const int c = tile_col(t0 + i);
    const int valid_rows = min(tile_rows, p.Lc - c * tile_rows);
    const uint32_t bytes = static_cast<uint32_t>(valid_rows) * D * 2;
    const int s = i % kStagesDec;
    mbar_expect_tx(&sm.full[s], 2 * bytes);
    const long long off = (head_base + static_cast<long long>(c) * tile_rows) * D;
    bulk_load(sm.kv[s][0], p.k + off, bytes, &sm.full[s]);
    bulk_load(sm.kv[s][1], p.v + off, bytes, &sm.full[s]);
  };
  if (tid == 0)
    for (int i = 0; i < min(kStagesDec, ntiles); ++i) issue(i);

  // lane owns dims [4*lane, 4*lane+4) (D=128) or [2*lane, 2*lane+2) (D=64)
  constexpr int kPer = D / 32;
  float qv[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) qv[e] = sm.q[lane * kPer + e];
  float m = -INFINITY, l = 0.f, acc[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) acc[e] = 0.f;

  for (int i = 0; i < ntiles; ++i) {
    const int s = i % kStagesDec;
    mbar_wait(&sm.full[s], (i / kStagesDec) & 1);
    const int t = t0 + i;
    const bool full_blk = t >= np;
    const int c = tile_col(t);
    const int valid_rows = min(tile_rows, p.Lc - c * tile_rows);
    int lpage = c, own = b, seq = p.logical_kv;
    if (p.paged) {
      lpage = __ldg(p.p2l + c);
      own = __ldg(p.owner + c);
      seq = min(__ldg(p.seq_len + b), p.logical_kv);
      // convert_mods throws UnmappedPhysicalIndex on such a page (paged_kv.cpp:265-269); here
      // it is masked and reported through the status word when the caller validates
      if (p.foreign != nullptr && tid == 0 && (own != b || lpage < 0)) atomicOr(p.foreign, 1);
    }
    const __nv_bfloat16* ks = reinterpret_cast<const __nv_bfloat16*>(sm.kv[s][0]);
    const __nv_bfloat16* vs = reinterpret_cast<const __nv_bfloat16*>(sm.kv[s][1]);
    for (int jb = warp * 32; jb < valid_rows; jb += 128) {
      // 1) partial dots of this lane's D-slice against the chunk's 32 keys
      float v[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const int j = min(jb + t, valid_rows - 1);  // rows past the page end are masked below
        if constexpr (kPer == 4) {
          const uint2 kw = *reinterpret_cast<const uint2*>(ks + j * D + lane * 4);
          const __nv_bfloat162 k01 = *reinterpret_cast<const __nv_bfloat162*>(&kw.x);
          const __nv_bfloat162 k23 = *reinterpret_cast<const __nv_bfloat162*>(&kw.y);
          v[t] = qv[0] * __low2float(k01) + qv[1] * __high2float(k01) + qv[2] * __low2float(k23) +
                 qv[3] * __high2float(k23);
        } else {
          const __nv_bfloat162 k01 = *reinterpret_cast<const __nv_bfloat162*>(ks + j * D + lane * 2);
          v[t] = qv[0] * __low2float(k01) + qv[1] * __high2float(k01);
        }
      }
      // 2) transposed butterfly: 31 shuffles leave lane l with the full dot of key jb + l
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
          const float send = upper ? v[i] : v[i + off];
          const float keep = upper ? v[i + off] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      // 3) score_mod / mask_mod for this lane's key, one online-softmax update per chunk
      const int j = jb + lane;
      const int phys = c * tile_rows + j;
      int logical = phys;
      bool live = j < valid_rows;
      if (p.paged) {
        logical = lpage * tile_rows + j;
        live = live && own == b && lpage >= 0 && logical < seq;
      }
      float x = -INFINITY;
      if (live && (full_blk || (qrow < p.n_new && logical < p.logical_kv && mask(b, h, qrow, logical))))
        x = score.apply(v[0] * p.scale, b, h, qrow, logical) * kLog2eD;
      float mx = x;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (mx == -INFINITY) continue;  // the whole chunk is masked: exact no-op (warp-uniform)
      const float m_new = fmaxf(m, mx);
      const float alpha = ex2(m - m_new);  // m == -inf -> 0
      const float pw = ex2(x - m_new);     // masked -> 0
      float ps = pw;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      l = l * alpha + ps;
      m = m_new;
#pragma unroll
      for (int e = 0; e < kPer; ++e) acc[e] *= alpha;
      // 4) P V: broadcast each key's weight, lanes accumulate their D-slice
      const int nj = min(32, valid_rows - jb);
#pragma unroll 8
      for (int t = 0; t < nj; ++t) {
        const float pj = __shfl_sync(0xffffffffu, pw, t);
        const int jj = jb + t;
        if constexpr (kPer == 4) {
          const uint2 vw = *reinterpret_cast<const uint2*>(vs + jj * D + lane * 4);
          const __nv_bfloat162 v01 = *reinterpret_cast<const __nv_bfloat162*>(&vw.x);
          const __nv_bfloat162 v23 = *reinterpret_cast<const __nv_bfloat162*>(&vw.y);
          acc[0] = fmaf(pj, __low2float(v01), acc[0]);
          acc[1] = fmaf(pj, __high2float(v01), acc[1]);
          acc[2] = fmaf(pj, __low2float(v23), acc[2]);
          acc[3] = fmaf(pj, __high2float(v23), acc[3]);
        } else {
          const __nv_bfloat162 v01 = *reinterpret_cast<const __nv_bfloat162*>(vs + jj * D + lane * 2);
          acc[0] = fmaf(pj, __low2float(v01), acc[0]);
          acc[1] = fmaf(pj, __high2float(v01), acc[1]);
        }
      }
    }
    __syncthreads();  // every warp is done with stage s
    if (tid == 0 && i + kStagesDec < ntiles) issue(i + kStagesDec);
  }

  // merge the 4 warp states
  if (lane == 0) {
    sm.wm[warp] = m;
    sm.wl[warp] = l;
  }
#pragma unroll
  for (int e = 0; e < kPer; ++e) sm.wacc[warp][lane * kPer + e] = acc[e];
  __syncthreads();
  if (warp == 0) {
    float M = fmaxf(fmaxf(sm.wm[0], sm.wm[1]), fmaxf(sm.wm[2], sm.wm[3]));
    const float Ms = M == -INFINITY ? 0.f : M;
    float L = 0.f, A[kPer];
#pragma unroll
    for (int e = 0; e < kPer; ++e) A[e] = 0.f;
    for (int w = 0; w < 4; ++w) {
      const float f = ex2(sm.wm[w] - Ms);
      L += sm.wl[w] * f;
#pragma unroll
      for (int e = 0; e < kPer; ++e) A[e] += sm.wacc[w][lane * kPer + e] * f;
    }
    if (p.splits == 1) {
      const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
      for (int e = 0; e < kPer; ++e) p.out[qslot * D + lane * kPer + e] = __float2bfloat16_rn(A[e] * inv);
      if (lane == 0) p.lse[qslot] = L > 0.f ? (M + __log2f(L)) * 0.6931471805599453f : -INFINITY;
    } else {
      float* dst = p.part + (qslot * p.splits + split) * (D + 2);
#pragma unroll
      for (int e = 0; e < kPer; ++e) dst[2 + lane * kPer + e] = A[e];
      if (lane == 0) {
        dst[0] = M;
        dst[1] = L;
      }
    }
  }
}

// Merge per-split (m, l, acc) states: one warp per query row.
template <int D>
__global__ void decode_combine_kernel(const float* __restrict__ part, int rows_total, int splits,
                                      __nv_bfloat16* __restrict__ out, float* __restrict__ lse) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows_total) return;
  constexpr int kPer = D / 32;
  const float* base = part + static_cast<long long>(row) * splits * (D + 2);
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, base[s * (D + 2)]);
  const float Ms = M == -INFINITY ? 0.f : M;
  float L = 0.f, A[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) A[e] = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float* ps = base + s * (D + 2);
    const float f = ex2(ps[0] - Ms);
    L += ps[1] * f;
#pragma unroll
    for (int e = 0; e < kPer; ++e) A[e] += ps[2 + lane * kPer + e] * f;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
  for (int e = 0; e < kPer; ++e)
    out[static_cast<long long>(row) * D + lane * kPer + e] = __float2bfloat16_rn(A[e] * inv);
  if (lane == 0) lse[row] = L > 0.f ? (M + __log2f(L)) * 0.6931471805599453f : -INFINITY;
}

template <int D, class MaskT, class ScoreT>
fa_status run(const DecParams& p, MaskT mask, ScoreT score, cudaStream_t st) {
  const size_t smem = sizeof(DecSmem<D>);
  auto kern = decode_kernel<D, MaskT, ScoreT>;
  FA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(p.splits, p.n_new, p.B * p.Hq);
  kern<<<grid, 128, smem, st>>>(p, mask, score);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  if (p.splits > 1) {
    const int rows_total = p.B * p.Hq * p.n_new;
    decode_combine_kernel<D><<<(rows_total + 3) / 4, 128, 0, st>>>(p.part, rows_total, p.splits,
                                                                 p.out, p.lse);
    count_launch();
    FA_CHECK_CUDA(cudaGetLastError());
  }
  return FA_OK;
}

// Kernel parameters of one decode call (geometry, views, workspace).
inline fa_status make_params(const DecodeGeom& g, const void* q, const void* k, const void* v, void* o,
                             float* lse, const BmView& bm, const PageView& pv, void* workspace, DecParams* out) {
  const AttnGeom& a = g.a;
  FA_REQUIRE(a.D == 128 || a.D == 64, FA_UNSUPPORTED, "decode: head dim must be 64 or 128");
  FA_REQUIRE(static_cast<long long>(a.bs_kv) * a.D * 2 <= kMaxTileBytes, FA_UNSUPPORTED,
             "decode: bs_kv * D * 2 must be <= 32 KiB");
  DecParams p{};
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.k = static_cast<const __nv_bfloat16*>(k);
  p.v = static_cast<const __nv_bfloat16*>(v);
  p.out = static_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.part = static_cast<float*>(workspace);
  p.B = a.B; p.Hq = a.Hq; p.Hkv = a.Hkv; p.Bkv = a.Bkv; p.n_new = a.Lq; p.Lc = a.Lkv; p.D = a.D;
  p.G = a.G; p.bm_b = a.bm_b; p.bm_h = a.bm_h; p.rows = a.rows; p.cols = a.cols;
  p.bs_q = a.bs_q; p.bs_kv = a.bs_kv;
  p.kv_num = bm.kv_num; p.kv_idx = bm.kv_idx; p.full_num = bm.full_num; p.full_idx = bm.full_idx;
  p.p2l = pv.phys_to_logical; p.owner = pv.owner; p.seq_len = pv.seq_len; p.paged = pv.enabled;
  p.foreign = pv.foreign;
  p.logical_kv = g.logical_kv;
  p.splits = g.num_splits;
  p.scale = a.scale;
  FA_REQUIRE(p.splits == 1 || workspace != nullptr, FA_SHAPE_MISMATCH,
             "decode: workspace required when num_splits > 1");
  *out = p;
  return FA_OK;
}

template <class MaskT, class ScoreT>
fa_status run_any_dim(const DecParams& p, MaskT mask, ScoreT score, cudaStream_t st) {
  if (p.D == 128) return run<128>(p, mask, score, st);
  return run<64>(p, mask, score, st);
}

}  // namespace
}  // namespace dec
}  // namespace fa
