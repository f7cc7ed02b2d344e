// dec_tc.cuh — tensor-core (paged) decode for steps with several query rows per kv head: the
// G query heads of a GQA group and the n_new rows of a multi-token step are packed into one
// 128-row tile, so every K/V page is streamed once per (batch element, kv head) instead of
// once per query row (decode, engine.cpp:403-427, over a convert_block_mask'ed BlockMask,
// paged_kv.cpp:154-228, with the logical positions of convert_mods, :230-310).
//
// The structure is fwd1t.cuh's (one tile per item, scores double-buffered in TMEM, the two
// softmax warpgroups splitting each page's 128 columns), with
//   * Q rows gathered by the softmax threads from (b, h_kv·G + g, i) into the swizzled tile
//     (row ρ = g·n_new + i; rows past G·n_new are zero and masked);
//   * K/V pages by TMA from the physical cache (1, H_kv, pages·page_size, D) (or the logical
//     cache when unpaged), positions for mask_mod / score_mod recovered per page
//     (phys -> logical, owner, seq_len; slack and foreign pages masked, foreign ones reported);
//   * split-KV over each row's page list, partial (m, l, acc) states merged by the decode
//     combine kernel (decode.cuh).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <type_traits>

#include "decode.cuh"
#include "host.cuh"
#include "mods.cuh"
#include "sm100_ptx.cuh"

namespace fa {
namespace dectc {
namespace {  // internal linkage: every including translation unit has its own copy

#ifndef FA_DEC_TC_MIN_ROWS
#define FA_DEC_TC_MIN_ROWS 2  // rows per kv head from which the tensor-core decode serves a step
#endif
constexpr int kThreads = 384;
constexpr int kTile = 128;
constexpr float kRescaleThreshold = 8.0f;
constexpr int kKStages = 2, kVStages = 2;

template <int D>
struct Cfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = kTile * D * 2;
  static constexpr int kChunkBytes = kTile * 128;
};

template <int D>
struct alignas(1024) Smem {
  uint8_t q[2][Cfg<D>::kTileBytes];
  uint8_t k[kKStages][Cfg<D>::kTileBytes];
  uint8_t v[kVStages][Cfg<D>::kTileBytes];
  float red[2][2][kTile];
  float lred[2][kTile];
  uint64_t q_full[2], q_free[2];
  uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[2], p_full, pv_done, o_full, o_free;
  uint64_t item_full[2], item_empty[2];
  int32_t uitem[2];
  uint32_t tmem_base;
};

struct Params {
  const __nv_bfloat16* q;  // (B, Hq, n_new, D)
  __nv_bfloat16* out;      // (B, Hq, n_new, D)
  float* lse;              // (B, Hq, n_new)
  float* part;             // (B·Hq·n_new, splits, D + 2) when splits > 1
  int B, Hq, Hkv, Bkv, G, n_new, rows_per_item, chunks, splits;
  int bm_b, bm_h, rows, cols, Lc;
  const int32_t* kv_num;
  const int32_t* kv_idx;
  const int32_t* full_num;
  const int32_t* full_idx;
  const int32_t* p2l;
  const int32_t* owner;
  const int32_t* seq_len;
  int* foreign;
  int paged, logical_kv;
  float scale;
  int num_items;
  int* work_counter;
};

struct Item {
  int b, hk, chunk, split;
};
__device__ __forceinline__ Item decode_item(const Params& p, int item) {
  Item it;
  it.split = item % p.splits;
  int rest = item / p.splits;
  it.chunk = rest % p.chunks;
  rest /= p.chunks;
  it.hk = rest % p.Hkv;
  it.b = rest / p.Hkv;
  return it;
}

// the page list of the item's rows (one BlockMask row: n_new <= bs_q), this split's share
struct PageList {
  const int32_t* pidx;
  const int32_t* fidx;
  int np, t0, t1;
  __device__ __forceinline__ void init(const Params& p, const Item& it) {
    const int mb = p.bm_b == 1 ? 0 : it.b;
    const int mh = p.bm_h == 1 ? 0 : it.hk * p.G;  // bm_h > 1 only with G == 1 (host check)
    const long long slot = (static_cast<long long>(mb) * p.bm_h + mh) * p.rows;
    np = __ldg(p.kv_num + slot);
    const int nt = np + __ldg(p.full_num + slot);
    const int per = (nt + p.splits - 1) / p.splits;
    t0 = it.split * per;
    t1 = min(nt, t0 + per);
    if (t1 < t0) t1 = t0;
    pidx = p.kv_idx + slot * p.cols;
    fidx = p.full_idx + slot * p.cols;
  }
  __device__ __forceinline__ int len() const { return t1 - t0; }
  __device__ __forceinline__ int col(int j) const {
    const int t = t0 + j;
    return t < np ? __ldg(pidx + t) : __ldg(fidx + t - np);
  }
};

template <int D, class MaskT, class ScoreT>
__global__ void __launch_bounds__(kThreads, 1)
    decode_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, const Params p,
                     MaskT mask, ScoreT score) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.q_full[s], 8);  // the softmax warps gather Q
      mbar_init(&sm.q_free[s], 1);
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.item_full[s], 1);
      mbar_init(&sm.item_empty[s], 1 + 8);
    }
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    mbar_init(&sm.p_full, 8);
    mbar_init(&sm.pv_done, 1);
    mbar_init(&sm.o_full, 1);
    mbar_init(&sm.o_free, 8);
    fence_barrier_init();
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 9) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  constexpr uint32_t kS = 0, kO = 256;

#define FA_DTC_TEARDOWN()      \
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
    FA_DTC_TEARDOWN();
  } else if (warp == 8) {
    if (lane == 0) {
      // ===================== TMA producer: K/V pages =====================
      int gb = 0;
      for (int n = 0;; ++n) {
        const int item = n == 0 ? static_cast<int>(blockIdx.x)
                                : static_cast<int>(gridDim.x) + atomicAdd(p.work_counter, 1);
        const int buf = n & 1;
        mbar_wait(&sm.item_empty[buf], ((n >> 1) & 1) ^ 1);
        sm.uitem[buf] = item < p.num_items ? item : -1;
        mbar_arrive(&sm.item_full[buf]);
        if (item >= p.num_items) break;
        const Item it = decode_item(p, item);
        PageList pl;
        pl.init(p, it);
        const int len = pl.len();
        const int kb = p.Bkv == 1 ? 0 : it.b;
        int col = len > 0 ? pl.col(0) : 0;
        for (int j = 0; j < len; ++j, ++gb) {
          const int col_next = j + 1 < len ? pl.col(j + 1) : 0;
          const int ks = gb % kKStages, vs = gb % kVStages;
          mbar_wait(&sm.k_empty[ks], ((gb / kKStages) & 1) ^ 1);
          mbar_expect_tx(&sm.k_full[ks], C::kTileBytes);
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_3d(sm.k[ks] + ch * C::kChunkBytes, &tmK, &sm.k_full[ks], ch * 64, col * kTile, kb * p.Hkv + it.hk);
          mbar_wait(&sm.v_empty[vs], ((gb / kVStages) & 1) ^ 1);
          mbar_expect_tx(&sm.v_full[vs], C::kTileBytes);
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_3d(sm.v[vs] + ch * C::kChunkBytes, &tmV, &sm.v_full[vs], ch * 64, col * kTile, kb * p.Hkv + it.hk);
          col = col_next;
        }
      }
    }
    FA_DTC_TEARDOWN();
  } else if (warp == 9) {
    // ===================== MMA issuer =====================
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idesc_pv = make_idesc_bf16(128, D, 0, 1);
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) umma_commit(bar);
      __syncwarp();
    };
    auto issue_qk = [&](int g, uint32_t q_addr) {
      const int ks = g % kKStages;
      mbar_wait(&sm.k_full[ks], (g / kKStages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t a0 = make_sdesc_sw128(q_addr, 16, 1024);
        const uint64_t b0 = make_sdesc_sw128(smem_u32(sm.k[ks]), 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * C::kChunkBytes + (kk & 3) * 32) >> 4;
          umma_ss(tm + kS + (g & 1) * 128, a0 + off, b0 + off, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&sm.s_full[g & 1]);
        umma_commit(&sm.k_empty[ks]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int g, bool acc) {
      const int vs = g % kVStages;
      mbar_wait(&sm.v_full[vs], (g / kVStages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t b0 = make_sdesc_sw128(smem_u32(sm.v[vs]), C::kChunkBytes, 1024);
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk) {
          const uint32_t a_col = kS + (g & 1) * 128 + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8);
          umma_ts(tm + kO, tm + a_col, b0 + kk * (2048 >> 4), idesc_pv, (acc || kk > 0) ? 1u : 0u);
        }
        umma_commit(&sm.v_empty[vs]);
        umma_commit(&sm.pv_done);
      }
      __syncwarp();
    };
    int gb = 0, no = 0;
    for (int n = 0;; ++n) {
      const int buf = n & 1;
      mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
      const int item = sm.uitem[buf];
      if (lane == 0) mbar_arrive(&sm.item_empty[buf]);
      if (item < 0) break;
      const Item it = decode_item(p, item);
      PageList pl;
      pl.init(p, it);
      const int len = pl.len();
      mbar_wait(&sm.q_full[buf], (n >> 1) & 1);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sm.q[buf]);
      if (len == 0) {
        commit(&sm.q_free[buf]);
        continue;
      }
      issue_qk(gb, q_addr);
      if (len == 1) commit(&sm.q_free[buf]);
      mbar_wait(&sm.o_free, (no & 1) ^ 1);
      for (int j = 0; j < len; ++j) {
        const int g = gb + j;
        if (j + 1 < len) {
          issue_qk(g + 1, q_addr);
          if (j + 2 == len) commit(&sm.q_free[buf]);
        }
        mbar_wait(&sm.p_full, g & 1);
        tc_fence_after();
        issue_pv(g, j > 0);
      }
      commit(&sm.o_full);
      gb += len;
      ++no;
    }
    FA_DTC_TEARDOWN();
  } else {
    // ===================== Q gather + softmax (thread = packed row, half a page each) =====================
    reg_alloc<224>();
    const int wg = warp >> 2;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const int tid = threadIdx.x;  // 0..255
    const uint32_t tm = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const uint32_t o_col = kO + wg * (D / 2);
    int gb = 0, no = 0;
    for (int n = 0;; ++n) {
      const int buf = n & 1;
      mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
      const int item = sm.uitem[buf];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.item_empty[buf]);
      if (item < 0) break;
      const Item it = decode_item(p, item);
      PageList pl;
      pl.init(p, it);
      const int len = pl.len();
      // ---- gather Q: packed row ρ = chunk·128 + r -> (g, i) = divmod(ρ, n_new) ----
      mbar_wait(&sm.q_free[buf], ((n >> 1) & 1) ^ 1);
      {
        constexpr int kUnits = D / 8;  // 16-byte units per row
        uint8_t* qs = sm.q[buf];
        for (int u = tid; u < kTile * kUnits; u += 256) {
          const int r = u / kUnits, c16 = u % kUnits;
          const int rho = it.chunk * kTile + r;
          uint4 val = make_uint4(0, 0, 0, 0);
          if (r < p.rows_per_item && rho < p.G * p.n_new) {
            const int g = rho / p.n_new, i = rho % p.n_new;
            const long long qslot = (static_cast<long long>(it.b) * p.Hq + it.hk * p.G + g) * p.n_new + i;
            val = __ldg(reinterpret_cast<const uint4*>(p.q + qslot * D) + c16);
          }
          // K-major SWIZZLE_128B: 64-column chunks of 128 rows x 128 B, 16-byte unit u ^ (row & 7)
          const int ch = c16 >> 3, u8 = c16 & 7;
          *reinterpret_cast<uint4*>(qs + ch * C::kChunkBytes + r * 128 + ((u8 ^ (r & 7)) << 4)) = val;
        }
        fence_proxy_async();  // generic-proxy stores -> the tensor core's async proxy
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.q_full[buf]);
      }
      const int rho = it.chunk * kTile + row;
      const bool row_ok = row < p.rows_per_item && rho < p.G * p.n_new;
      const int g_row = row_ok ? rho / p.n_new : 0, i_row = row_ok ? rho % p.n_new : 0;
      const int h = it.hk * p.G + g_row;
      const long long slot = (static_cast<long long>(it.b) * p.Hq + h) * p.n_new + i_row;
      const int seq = p.paged ? min(__ldg(p.seq_len + it.b), p.logical_kv) : p.logical_kv;
      float m = -INFINITY, l = 0.f;
      if (len > 0) {
        int col = pl.col(0);
        for (int j = 0; j < len; ++j) {
          const int gg = gb + j;
          const int col_next = j + 1 < len ? pl.col(j + 1) : 0;
          // logical position of the page (convert_mods, paged_kv.cpp:240-272)
          int lpage = col;
          bool page_ok = true;
          if (p.paged) {
            lpage = __ldg(p.p2l + col);
            const int own = __ldg(p.owner + col);
            page_ok = own == it.b && lpage >= 0;
            if (!page_ok && p.foreign != nullptr && tid == 0) atomicOr(p.foreign, 1);
          }
          const int kv0 = lpage * kTile + wg * 64;
          const uint32_t s_col = kS + (gg & 1) * 128 + wg * 64;
          uint32_t bits0 = 0u, bits1 = 0u;
          if (row_ok && page_ok) {  // every decode tile is partial: mask + bounds always (block_mask.cpp:94)
            bits0 = mask.bits32(it.b, h, i_row, kv0, seq);
            bits1 = mask.bits32(it.b, h, i_row, kv0 + 32, seq);
          }
          constexpr bool kPlain = ScoreT::kIdentity;
          const auto rowc = score.row(it.b, h, i_row, kv0, p.scale);
          mbar_wait(&sm.s_full[gg & 1], (gg >> 1) & 1);
          tc_fence_after();
          uint32_t r[64];
          tmem_ld32(tm + s_col, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld32(tm + s_col + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          tmem_wait_ld();
          float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < 64; i += 2) {
            float v0 = __uint_as_float(r[i]), v1 = __uint_as_float(r[i + 1]);
            if constexpr (!kPlain) {
              const auto rc = rowc.shifted(i & ~31);
              v0 = rc.log2(v0, i & 31);
              v1 = rc.log2(v1, (i + 1) & 31);
            }
            const uint32_t bw = i < 32 ? bits0 : bits1;
            v0 = ((bw >> (i & 31)) & 1u) ? v0 : -INFINITY;
            v1 = ((bw >> ((i + 1) & 31)) & 1u) ? v1 : -INFINITY;
            r[i] = __float_as_uint(v0);
            r[i + 1] = __float_as_uint(v1);
            mx4[(i >> 1) & 3] = fmax3(mx4[(i >> 1) & 3], v0, v1);
          }
          float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
          if constexpr (kPlain) mx *= rowc.c;
          sm.red[gg & 1][wg][row] = mx;
          named_bar_sync(1, 256);
          mx = fmaxf(mx, sm.red[gg & 1][wg ^ 1][row]);
          const float m_new = fmaxf(m, mx);
          const bool need = (m != -INFINITY) && (m_new > m + kRescaleThreshold);
          if (__any_sync(0xffffffffu, need)) {
            mbar_wait(&sm.pv_done, (gg - 1) & 1);
            tc_fence_after();
            const float alpha = need ? ex2(m - m_new) : 1.f;
#pragma unroll 1
            for (int cc = 0; cc < D / 64; ++cc) {
              uint32_t o[32];
              tmem_ld32(tm + o_col + cc * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st32(tm + o_col + cc * 32, o);
            }
            tmem_wait_st();
            l *= alpha;
          }
          if (need || m == -INFINITY) m = m_new;
          const float msub = (m == -INFINITY) ? 0.f : m;
          const float2 xs2 = make_float2(kPlain ? rowc.c : 1.f, kPlain ? rowc.c : 1.f);
          const float2 nm2 = make_float2(-msub, -msub);
          float2 ls[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), xs2, nm2);
            const float2 pv = make_float2(ex2(x.x), ex2(x.y));
            ls[i & 3] = __fadd2_rn(ls[i & 3], pv);
            pk[i] = pack_bf16(pv.x, pv.y);
          }
          tmem_st32(tm + s_col, pk);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.p_full);
          const float2 l01 = __fadd2_rn(ls[0], ls[1]), l23 = __fadd2_rn(ls[2], ls[3]);
          const float2 lt = __fadd2_rn(l01, l23);
          l += lt.x + lt.y;
          col = col_next;
        }
        gb += len;
      }
      // ---- epilogue: combine the halves' row sums; O / l (one split) or the partial state ----
      sm.lred[wg][row] = l;
      named_bar_sync(1, 256);
      l += sm.lred[wg ^ 1][row];
      uint32_t a[D / 2];
      if (len > 0) {
        mbar_wait(&sm.o_full, no & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < D / 64; ++cc)
          tmem_ld32(tm + o_col + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&a[cc * 32]));
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < D / 2; ++e) a[e] = 0u;
      }
      if (row_ok) {
        if (p.splits == 1) {
          const float inv = l > 0.f ? 1.f / l : 0.f;
          uint4* d4 = reinterpret_cast<uint4*>(p.out + slot * D + wg * (D / 2));
#pragma unroll
          for (int u = 0; u < D / 16; ++u)
            d4[u] = make_uint4(pack_bf16(__uint_as_float(a[8 * u]) * inv, __uint_as_float(a[8 * u + 1]) * inv),
                               pack_bf16(__uint_as_float(a[8 * u + 2]) * inv, __uint_as_float(a[8 * u + 3]) * inv),
                               pack_bf16(__uint_as_float(a[8 * u + 4]) * inv, __uint_as_float(a[8 * u + 5]) * inv),
                               pack_bf16(__uint_as_float(a[8 * u + 6]) * inv, __uint_as_float(a[8 * u + 7]) * inv));
          if (wg == 0) p.lse[slot] = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
        } else {
          // the decode combine kernel's layout: (m [log2 domain], l, acc[D]) per (row, split)
          float* dst = p.part + (slot * p.splits + it.split) * (D + 2);
#pragma unroll
          for (int e = 0; e < D / 2; ++e) dst[2 + wg * (D / 2) + e] = __uint_as_float(a[e]);
          if (wg == 0) {
            dst[0] = m;
            dst[1] = l;
          }
        }
      }
      tc_fence_before();
      named_bar_sync(1, 256);
      if (len > 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.o_free);
        ++no;
      }
    }
    FA_DTC_TEARDOWN();
  }
#undef FA_DTC_TEARDOWN
}

// Shapes and masks this path serves: bf16, page / block size 128, D 64 or 128, a step of at most
// 128 rows, and query heads of a group sharing their BlockMask row (h_dims == 1) when G > 1.
inline bool supported(const DecodeGeom& g) {
  const AttnGeom& a = g.a;
  return (a.D == 128 || a.D == 64) && a.bs_kv == kTile && a.Lq <= kTile && a.rows == 1 &&
         (a.bm_h == 1 || a.G == 1) && a.G * a.Lq >= FA_DEC_TC_MIN_ROWS;
}

template <int D, class MaskT, class ScoreT>
fa_status run(const DecodeGeom& dg, const void* q, const void* k, const void* v, void* o, float* lse,
              const BmView& bm, const PageView& pv, void* workspace, MaskT mask, ScoreT score, cudaStream_t st) {
  const AttnGeom& g = dg.a;
  CUtensorMap mk, mv;
  fa_status s;
  if ((s = make_map(&mk, k, g.Bkv * g.Hkv, g.Lkv, D)) != FA_OK) return s;
  if ((s = make_map(&mv, v, g.Bkv * g.Hkv, g.Lkv, D)) != FA_OK) return s;
  Params p{};
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.out = static_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.part = static_cast<float*>(workspace);
  p.B = g.B; p.Hq = g.Hq; p.Hkv = g.Hkv; p.Bkv = g.Bkv; p.G = g.G; p.n_new = g.Lq;
  const int rows_total = g.G * g.Lq;
  p.chunks = (rows_total + kTile - 1) / kTile;
  p.rows_per_item = std::min(kTile, rows_total);
  p.bm_b = g.bm_b; p.bm_h = g.bm_h; p.rows = g.rows; p.cols = g.cols; p.Lc = g.Lkv;
  p.kv_num = bm.kv_num; p.kv_idx = bm.kv_idx; p.full_num = bm.full_num; p.full_idx = bm.full_idx;
  p.p2l = pv.phys_to_logical; p.owner = pv.owner; p.seq_len = pv.seq_len; p.paged = pv.enabled;
  p.foreign = pv.foreign;
  p.logical_kv = dg.logical_kv;
  p.scale = g.scale;
  // split-KV: enough items for two waves, at most 64 splits and one page each
  const int base_items = g.B * g.Hkv * p.chunks;
  int splits = (2 * num_sms() + base_items - 1) / base_items;
  splits = std::max(1, std::min(splits, std::min(64, g.cols)));
  if (dg.num_splits > 0 && dg.num_splits < splits) splits = dg.num_splits;
  FA_REQUIRE(splits == 1 || workspace != nullptr, FA_SHAPE_MISMATCH, "decode: workspace required for split-KV");
  p.splits = splits;
  p.num_items = base_items * splits;
  p.work_counter = scheduler_counter(kSlotFwdSched, st);
  FA_REQUIRE(p.work_counter != nullptr, FA_CUDA_ERROR, "decode: cannot allocate the scheduler counter");
  FA_CHECK_CUDA(cudaMemsetAsync(p.work_counter, 0, sizeof(int), st));
  const size_t smem = sizeof(Smem<D>);
  auto kern = decode_tc_kernel<D, MaskT, ScoreT>;
  FA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = p.num_items < num_sms() ? p.num_items : num_sms();
  if (grid <= 0) return FA_OK;
  kern<<<grid, kThreads, smem, st>>>(mk, mv, p, mask, score);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  if (splits > 1) {
    const int rows = g.B * g.Hq * g.Lq;
    dec::decode_combine_kernel<D><<<(rows + 3) / 4, 128, 0, st>>>(p.part, rows, splits, p.out, p.lse);
    count_launch();
    FA_CHECK_CUDA(cudaGetLastError());
  }
  return FA_OK;
}

}  // namespace
}  // namespace dectc
}  // namespace fa
