// bwd_dq.cuh — the dQ pass of the backward as its own tensor-core kernel (sm_100a): the
// reference's separate dq pass (engine.cpp:237-305) over the kv-side lists, with dQ
// accumulated in TMEM across the row's kv blocks in one fixed order, so it is bitwise
// reproducible and needs no fp32 accumulator, no zeroing and no conversion pass. Paired with
// the dK/dV-only variant of the main backward kernel (bwd_sm100.cuh, kMode == kModeNoDQ).
//
// Persistent, warp-specialised CTA (384 threads, 1 CTA/SM; setmaxnreg 224 for the compute
// warpgroups, 56 for the rest). A work item is one 128-row q tile
// r of one (b, h); it walks the tile's kv-side list (partial blocks, then full blocks) and per
// kv block j runs
//     S_j  = Q K_j^T        (SS, fp32 in TMEM, double-buffered)
//     dP_j = dO V_j^T       (SS, fp32 in TMEM)
//     compute warps (thread = q row; two warpgroups, 64 kv columns each):
//        P·scale = exp2(score_mod(S_j)·log2e + log2(scale) - lse·log2e)   (mask_mod in partial
//        blocks), dS = P·scale·mod'(s)·(dP_j - Δ) as bf16 over S_j's columns
//     dQ  += dS K_j          (TS: dS from TMEM, K_j from smem, MN-major)
// issued  S(j+1) | dQ(j) | dP(j+1) so the next block's scores are ready when the compute warps
// finish a block. Warps 0-7 compute, warp 8 TMA producer, warp 9 MMA issuer, 10-11 idle.
// TMEM (512 columns): S0 [0,128), S1 [128,256), dP [256,384), dQ [384, 384 + D).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <string>
#include <type_traits>

#include "host.cuh"
#include "mods.cuh"
#include "sm100_ptx.cuh"

namespace fa {
namespace bdq {
namespace {  // internal linkage: every including translation unit has its own copy

constexpr int kThreads = 384;  // 2 compute warpgroups + (producer, MMA, 2 idle) warpgroup
constexpr int kTile = 128;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kKStages = 3;  // K_j is read by S(j) and, a block later, by dQ(j)
constexpr int kVStages = 2;

template <int D>
struct Cfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = kTile * D * 2;
  static constexpr int kChunkBytes = kTile * 128;
};

template <int D>
struct alignas(1024) Smem {
  uint8_t q[Cfg<D>::kTileBytes];
  uint8_t dO[Cfg<D>::kTileBytes];
  uint8_t k[kKStages][Cfg<D>::kTileBytes];
  uint8_t v[kVStages][Cfg<D>::kTileBytes];
  uint64_t q_full, q_free, do_full, do_free;
  uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[2], dp_full, ds_full, dq_done, dq_free;
  uint64_t item_full[2], item_empty[2];
  int32_t uitem[2];
  uint32_t tmem_base;
};

struct Params {
  int B, Hq, Hkv, Bkv, Lq, Lkv, G, Lq_pad;
  int bm_b, bm_h, rows, cols;
  const int32_t* kv_num;
  const int32_t* kv_idx;
  const int32_t* full_num;
  const int32_t* full_idx;
  const float* lse;    // (B*Hq, Lq) natural log, from the forward
  const float* delta;  // (B*Hq, Lq_pad) Δ = rowsum(dO·O), from the preprocess
  __nv_bfloat16* dq;   // (B*Hq, Lq, D)
  float scale, log2_scale;
  int num_items;
  int* work_counter;
};

struct Item {
  int b, h, r;
};
__device__ __forceinline__ Item decode_item(const Params& p, int item) {
  // the longest q rows (causal-like masks) first across all heads: a cheap LPT order
  const int bh_count = p.B * p.Hq;
  const int r = p.rows - 1 - item / bh_count;
  const int bh = item % bh_count;
  return Item{bh / p.Hq, bh % p.Hq, r};
}

// The kv blocks of q tile r: the partial list then the full list (one fixed order).
struct RowList {
  const int32_t* pidx;
  const int32_t* fidx;
  int np, nf;
  __device__ __forceinline__ void init(const Params& p, const Item& it) {
    const int mb = p.bm_b == 1 ? 0 : it.b, mh = p.bm_h == 1 ? 0 : it.h;
    const long long slot = (static_cast<long long>(mb) * p.bm_h + mh) * p.rows + it.r;
    np = __ldg(p.kv_num + slot);
    nf = __ldg(p.full_num + slot);
    pidx = p.kv_idx + slot * p.cols;
    fidx = p.full_idx + slot * p.cols;
  }
  __device__ __forceinline__ int len() const { return np + nf; }
  __device__ __forceinline__ int col(int j) const { return j < np ? __ldg(pidx + j) : __ldg(fidx + j - np); }
};

template <int D, class MaskT, class ScoreT>
__global__ void __launch_bounds__(kThreads, 1)
    flex_bwd_dq_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                       const Params p, MaskT mask, ScoreT score) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();  // SWIZZLE_128B operands need 1 KiB alignment

  if (threadIdx.x == 0) {
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_free, 1);
    mbar_init(&sm.do_full, 1);
    mbar_init(&sm.do_free, 1);
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    mbar_init(&sm.s_full[0], 1);
    mbar_init(&sm.s_full[1], 1);
    mbar_init(&sm.dp_full, 1);
    mbar_init(&sm.ds_full, 8);
    mbar_init(&sm.dq_done, 1);
    mbar_init(&sm.dq_free, 8);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.item_full[s], 1);
      mbar_init(&sm.item_empty[s], 1 + 8);
    }
    fence_barrier_init();
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
  }
  if (warp == 9) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  constexpr uint32_t kS = 0, kDP = 256, kDQ = 384;

#define FA_BDQ_TEARDOWN()      \
  do {                         \
    tc_fence_before();         \
    __syncthreads();           \
    if (warp == 9) {           \
      tc_fence_after();        \
      tmem_dealloc(tmem, 512); \
    }                          \
    return;                    \
  } while (0)

  if (warp >= 8) reg_dealloc<56>();
  if (warp >= 10) {
    FA_BDQ_TEARDOWN();
  } else if (warp == 8) {
    if (lane == 0) {
      // ===================== TMA producer =====================
      int gb = 0;  // blocks streamed so far (K/V ring positions)
      for (int n = 0;; ++n) {
        const int item = n == 0 ? static_cast<int>(blockIdx.x)
                                : static_cast<int>(gridDim.x) + atomicAdd(p.work_counter, 1);
        const int buf = n & 1;
        mbar_wait(&sm.item_empty[buf], ((n >> 1) & 1) ^ 1);
        sm.uitem[buf] = item < p.num_items ? item : -1;
        mbar_arrive(&sm.item_full[buf]);
        if (item >= p.num_items) break;
        const Item it = decode_item(p, item);
        RowList rl;
        rl.init(p, it);
        const int len = rl.len();
        const int kb = p.Bkv == 1 ? 0 : it.b, kh = it.h / p.G;
        mbar_wait(&sm.q_free, (n & 1) ^ 1);
        mbar_expect_tx(&sm.q_full, C::kTileBytes);
        for (int ch = 0; ch < C::kChunks; ++ch)
          tma_load_3d(sm.q + ch * C::kChunkBytes, &tmQ, &sm.q_full, ch * 64, it.r * kTile, it.b * p.Hq + it.h);
        mbar_wait(&sm.do_free, (n & 1) ^ 1);
        mbar_expect_tx(&sm.do_full, C::kTileBytes);
        for (int ch = 0; ch < C::kChunks; ++ch)
          tma_load_3d(sm.dO + ch * C::kChunkBytes, &tmDO, &sm.do_full, ch * 64, it.r * kTile, it.b * p.Hq + it.h);
        int col = len > 0 ? rl.col(0) : 0;
        for (int j = 0; j < len; ++j, ++gb) {
          const int col_next = j + 1 < len ? rl.col(j + 1) : 0;  // index load ahead of the waits
          const int ks = gb % kKStages, vs = gb % kVStages;
          mbar_wait(&sm.k_empty[ks], ((gb / kKStages) & 1) ^ 1);
          mbar_expect_tx(&sm.k_full[ks], C::kTileBytes);
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_3d(sm.k[ks] + ch * C::kChunkBytes, &tmK, &sm.k_full[ks], ch * 64, col * kTile, kb * p.Hkv + kh);
          mbar_wait(&sm.v_empty[vs], ((gb / kVStages) & 1) ^ 1);
          mbar_expect_tx(&sm.v_full[vs], C::kTileBytes);
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_3d(sm.v[vs] + ch * C::kChunkBytes, &tmV, &sm.v_full[vs], ch * 64, col * kTile, kb * p.Hkv + kh);
          col = col_next;
        }
      }
    }
    FA_BDQ_TEARDOWN();
  } else if (warp == 9) {
    // ===================== MMA issuer (whole warp, one elected lane issues) =====================
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);  // S = Q K^T, dP = dO V^T
    constexpr uint32_t idesc_dq = make_idesc_bf16(128, D, 0, 1);   // dQ += dS K (K MN-major)
    const uint32_t q_addr = smem_u32(sm.q), do_addr = smem_u32(sm.dO);
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) umma_commit(bar);
      __syncwarp();
    };
    auto gemm_kmajor = [&](uint32_t d_col, uint32_t a_addr, uint32_t b_addr) {
      if (elect_one()) {
        const uint64_t a0 = make_sdesc_sw128(a_addr, 16, 1024);
        const uint64_t b0 = make_sdesc_sw128(b_addr, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * C::kChunkBytes + (kk & 3) * 32) >> 4;
          umma_ss(tm + d_col, a0 + off, b0 + off, idesc_s, kk > 0 ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    auto issue_s = [&](int g) {
      const int ks = g % kKStages;
      mbar_wait(&sm.k_full[ks], (g / kKStages) & 1);
      tc_fence_after();
      gemm_kmajor(kS + (g & 1) * 128, q_addr, smem_u32(sm.k[ks]));
      commit(&sm.s_full[g & 1]);
    };
    auto issue_dp = [&](int g) {
      const int vs = g % kVStages;
      mbar_wait(&sm.v_full[vs], (g / kVStages) & 1);
      tc_fence_after();
      gemm_kmajor(kDP, do_addr, smem_u32(sm.v[vs]));
      commit(&sm.dp_full);
      commit(&sm.v_empty[vs]);  // V_j's only reader
    };
    auto issue_dq = [&](int g, bool acc) {
      const int ks = g % kKStages;
      if (elect_one()) {
        const uint64_t b0 = make_sdesc_sw128(smem_u32(sm.k[ks]), C::kChunkBytes, 1024);
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk) {
          // dS of warpgroup w (kv 64w..64w+63) sits in columns [64w, 64w + 32) of S_g
          const uint32_t a_col = kS + (g & 1) * 128 + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8);
          umma_ts(tm + kDQ, tm + a_col, b0 + kk * (2048 >> 4), idesc_dq, (acc || kk > 0) ? 1u : 0u);
        }
        umma_commit(&sm.k_empty[ks]);  // K_j's last reader
      }
      __syncwarp();
    };
    int gb = 0, ndq = 0;
    for (int n = 0;; ++n) {
      const int buf = n & 1;
      mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
      const int item = sm.uitem[buf];
      if (lane == 0) mbar_arrive(&sm.item_empty[buf]);
      if (item < 0) break;
      const Item it = decode_item(p, item);
      RowList rl;
      rl.init(p, it);
      const int len = rl.len();
      mbar_wait(&sm.q_full, n & 1);
      mbar_wait(&sm.do_full, n & 1);
      tc_fence_after();
      if (len == 0) {
        commit(&sm.q_free);
        commit(&sm.do_free);
        continue;
      }
      issue_s(gb);
      if (len == 1) commit(&sm.q_free);
      issue_dp(gb);
      if (len == 1) commit(&sm.do_free);
      mbar_wait(&sm.dq_free, (ndq & 1) ^ 1);  // the previous item's dQ was read out
      for (int j = 0; j < len; ++j) {
        const int g = gb + j;
        if (j + 1 < len) {
          issue_s(g + 1);
          if (j + 2 == len) commit(&sm.q_free);
        }
        mbar_wait(&sm.ds_full, g & 1);
        tc_fence_after();
        issue_dq(g, j > 0);
        if (j + 1 == len) commit(&sm.dq_done);
        if (j + 1 < len) {
          issue_dp(g + 1);
          if (j + 2 == len) commit(&sm.do_free);
        }
      }
      gb += len;
      ++ndq;
    }
    FA_BDQ_TEARDOWN();
  } else {
    // ===================== compute warpgroups: P, dS (thread = q row) =====================
    reg_alloc<224>();
    const int wg = warp >> 2;        // which 64 kv columns of a block
    const int wq = warp & 3;         // TMEM lane quarter
    const int row = wq * 32 + lane;  // q row within the tile
    const uint32_t tm = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    int gb = 0, ndq = 0;
    for (int n = 0;; ++n) {
      const int buf = n & 1;
      mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
      const int item = sm.uitem[buf];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.item_empty[buf]);
      if (item < 0) break;
      const Item it = decode_item(p, item);
      RowList rl;
      rl.init(p, it);
      const int len = rl.len();
      const int qi = it.r * kTile + row;
      const bool q_ok = qi < p.Lq;
      const long long bh = static_cast<long long>(it.b) * p.Hq + it.h;
      const float lse = q_ok ? __ldg(p.lse + bh * p.Lq + qi) : -INFINITY;
      // log2-domain column term: P·scale = exp2(x + ct); rows with lse = -inf contribute nothing
      const float ct = lse == -INFINITY ? -INFINITY : p.log2_scale - lse * kLog2e;
      const float dlt = q_ok ? __ldg(p.delta + bh * p.Lq_pad + qi) : 0.f;
      __nv_bfloat16* dq_row = p.dq + (bh * p.Lq + qi) * D + wg * (D / 2);
      if (len == 0) {  // no visited block: dQ = 0
        if (q_ok)
          for (int u = 0; u < D / 16; ++u) reinterpret_cast<uint4*>(dq_row)[u] = make_uint4(0, 0, 0, 0);
        continue;
      }
      int col = rl.col(0);
      for (int j = 0; j < len; ++j) {
        const int g = gb + j;
        const bool full = j >= rl.np;
        const int col_next = j + 1 < len ? rl.col(j + 1) : 0;
        const int kv0 = col * kTile + wg * 64;
        const uint32_t s_col = kS + (g & 1) * 128 + wg * 64;
        uint32_t bits0 = ~0u, bits1 = ~0u;
        if (!full) {
          bits0 = q_ok ? mask.bits32(it.b, it.h, qi, kv0, p.Lkv) : 0u;
          bits1 = q_ok ? mask.bits32(it.b, it.h, qi, kv0 + 32, p.Lkv) : 0u;
        }
        const auto rowc = score.row(it.b, it.h, qi, kv0, p.scale);
        mbar_wait(&sm.s_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        uint32_t sr[64];
        tmem_ld32(tm + s_col, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        tmem_ld32(tm + s_col + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_wait_ld();
        // P·scale·mod'(s), in place over the scores
        auto exps = [&](auto masked) {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const float sv = __uint_as_float(sr[i]);
            float x, gr = 1.f;
            if constexpr (ScoreT::kIdentity) {
              x = sv * rowc.c;
            } else if constexpr (ScoreT::kUnitGrad) {
              x = rowc.shifted(i & ~31).log2(sv, i & 31);
            } else {
              x = rowc.shifted(i & ~31).log2_grad(sv, i & 31, gr);
            }
            float pv = ex2(x + ct);
            if constexpr (decltype(masked)::value) pv = ((((i < 32) ? bits0 : bits1) >> (i & 31)) & 1u) ? pv : 0.f;
            sr[i] = __float_as_uint(ScoreT::kUnitGrad ? pv : pv * gr);
          }
        };
        if (full) exps(std::false_type{});
        else exps(std::true_type{});
        // dS = P·scale·mod'·(dP - Δ) -> bf16 over this warpgroup's first 32 S columns
        mbar_wait(&sm.dp_full, g & 1);
        tc_fence_after();
        uint32_t dpr[2][32];
        tmem_ld32(tm + kDP + wg * 64, dpr[0]);
        tmem_wait_ld();
        tmem_ld32(tm + kDP + wg * 64 + 32, dpr[1]);  // overlaps the first half's math
        uint32_t dsp[32];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (hh == 1) tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a0 = __uint_as_float(sr[hh * 32 + 2 * i]) * (__uint_as_float(dpr[hh][2 * i]) - dlt);
            const float a1 = __uint_as_float(sr[hh * 32 + 2 * i + 1]) * (__uint_as_float(dpr[hh][2 * i + 1]) - dlt);
            dsp[hh * 16 + i] = pack_bf16(a0, a1);
          }
        }
        tmem_st32(tm + s_col, dsp);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.ds_full);
        col = col_next;
      }
      gb += len;
      // ---- epilogue: dQ row (this warpgroup's half of the head dim) -> bf16 ----
      mbar_wait(&sm.dq_done, ndq & 1);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < D / 64; ++cc) {
        uint32_t a[32];
        tmem_ld32(tm + kDQ + wg * (D / 2) + cc * 32, a);
        tmem_wait_ld();
        if (q_ok) {
          uint4* d4 = reinterpret_cast<uint4*>(dq_row + cc * 32);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            d4[u] = make_uint4(pack_bf16(__uint_as_float(a[8 * u]), __uint_as_float(a[8 * u + 1])),
                               pack_bf16(__uint_as_float(a[8 * u + 2]), __uint_as_float(a[8 * u + 3])),
                               pack_bf16(__uint_as_float(a[8 * u + 4]), __uint_as_float(a[8 * u + 5])),
                               pack_bf16(__uint_as_float(a[8 * u + 6]), __uint_as_float(a[8 * u + 7])));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.dq_free);
      ++ndq;
    }
    FA_BDQ_TEARDOWN();
  }
#undef FA_BDQ_TEARDOWN
}

// Launch of the dQ pass; `lse` natural log from the forward, `delta` the preprocess's Δ
// (layout (B*Hq, Lq_pad)).
template <int D, class MaskT, class ScoreT>
fa_status run(const AttnGeom& g, const void* q, const void* k, const void* v, const void* dout, const float* lse,
              const float* delta, void* dq, const BmView& bm, MaskT mask, ScoreT score, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mdo;
  fa_status s;
  if ((s = make_map(&mq, q, g.B * g.Hq, g.Lq, D)) != FA_OK) return s;
  if ((s = make_map(&mk, k, g.Bkv * g.Hkv, g.Lkv, D)) != FA_OK) return s;
  if ((s = make_map(&mv, v, g.Bkv * g.Hkv, g.Lkv, D)) != FA_OK) return s;
  if ((s = make_map(&mdo, dout, g.B * g.Hq, g.Lq, D)) != FA_OK) return s;
  Params p{};
  p.B = g.B; p.Hq = g.Hq; p.Hkv = g.Hkv; p.Bkv = g.Bkv; p.Lq = g.Lq; p.Lkv = g.Lkv; p.G = g.G;
  p.Lq_pad = (g.Lq + kTile - 1) / kTile * kTile;
  p.bm_b = g.bm_b; p.bm_h = g.bm_h; p.rows = g.rows; p.cols = g.cols;
  p.kv_num = bm.kv_num; p.kv_idx = bm.kv_idx; p.full_num = bm.full_num; p.full_idx = bm.full_idx;
  p.lse = lse;
  p.delta = delta;
  p.dq = static_cast<__nv_bfloat16*>(dq);
  p.scale = g.scale;
  p.log2_scale = log2f(g.scale);
  p.num_items = g.B * g.Hq * g.rows;
  p.work_counter = scheduler_counter(kSlotDqSched, st);
  FA_REQUIRE(p.work_counter != nullptr, FA_CUDA_ERROR, "backward dQ pass: cannot allocate the scheduler counter");
  FA_CHECK_CUDA(cudaMemsetAsync(p.work_counter, 0, sizeof(int), st));
  const size_t smem = sizeof(Smem<D>);
  auto kern = flex_bwd_dq_kernel<D, MaskT, ScoreT>;
  FA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = p.num_items < num_sms() ? p.num_items : num_sms();
  if (grid <= 0) return FA_OK;
  kern<<<grid, kThreads, smem, st>>>(mq, mk, mv, mdo, p, mask, score);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

}  // namespace
}  // namespace bdq
}  // namespace fa
