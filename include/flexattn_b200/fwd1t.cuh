// fwd1t.cuh — block-sparse FlexAttention forward for sm_100a with ONE 128-row q tile per
// work item and the scores double-buffered in TMEM, the alternative organisation to
// fwd_sm100.cuh's two ping-ponging tiles. S(j+1) = Q K_{j+1}^T runs on the tensor core while
// the softmax works on S(j), so the per-block chain is softmax(j) -> PV(j) only.
//
// Persistent, warp-specialised CTA (384 threads, 1 CTA/SM; setmaxnreg 224 / 56):
//   warps 0-7  softmax: two warpgroups split every kv block's 128 columns (64 each); thread =
//              q row. The row max of a block is exchanged between the two halves through smem
//              (one named barrier per block); each half keeps its own part of the row sum and
//              rescales its half of O (lazily, when the max grows by more than 2^8).
//   warp 8     TMA producer: Q (double-buffered per item), K_j / V_j (2-stage rings).
//   warp 9     MMA issuer: S(j+1) | PV(j), P as bf16 over S(j)'s columns (TS MMA).
//   warps 10-11 idle.
// TMEM (512 columns): S0 [0,128), S1 [128,256), O [256, 256 + D).
// The visit order is the row's partial blocks then its full blocks (exact math in any order).
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
namespace fwd1t {
namespace {  // internal linkage: every including translation unit has its own copy

constexpr int kThreads = 384;
constexpr int kTile = 128;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
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
  float red[2][2][kTile];  // [block parity][half] partial row maxima
  float lred[2][kTile];    // [half] partial row sums (item end)
  uint64_t q_full[2], q_free[2];
  uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[2], p_full, pv_done, o_full, o_free;
  uint64_t item_full[2], item_empty[2];
  int32_t uitem[2];
  uint32_t tmem_base;
};

struct Params {
  __nv_bfloat16* out;
  float* lse;
  int B, Hq, Hkv, Bkv, Lq, Lkv, G;
  int bm_b, bm_h, rows, cols;
  const int32_t* kv_num;
  const int32_t* kv_idx;
  const int32_t* full_num;
  const int32_t* full_idx;
  float scale;
  int num_items;
  int* work_counter;
};

struct Item {
  int b, h, r;
};
__device__ __forceinline__ Item decode_item(const Params& p, int item) {
  const int bh_count = p.B * p.Hq;
  const int r = p.rows - 1 - item / bh_count;  // longest (causal) rows first: cheap LPT
  const int bh = item % bh_count;
  return Item{bh / p.Hq, bh % p.Hq, r};
}

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
    flex_fwd1t_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const Params p, MaskT mask, ScoreT score) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.q_full[s], 1);
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
    tma_prefetch_desc(&tmQ);
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

#define FA_F1T_TEARDOWN()      \
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
    FA_F1T_TEARDOWN();
  } else if (warp == 8) {
    if (lane == 0) {
      // ===================== TMA producer =====================
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
        RowList rl;
        rl.init(p, it);
        const int len = rl.len();
        const int kb = p.Bkv == 1 ? 0 : it.b, kh = it.h / p.G;
        mbar_wait(&sm.q_free[buf], ((n >> 1) & 1) ^ 1);
        mbar_expect_tx(&sm.q_full[buf], C::kTileBytes);
        for (int ch = 0; ch < C::kChunks; ++ch)
          tma_load_3d(sm.q[buf] + ch * C::kChunkBytes, &tmQ, &sm.q_full[buf], ch * 64, it.r * kTile,
                      it.b * p.Hq + it.h);
        int col = len > 0 ? rl.col(0) : 0;
        for (int j = 0; j < len; ++j, ++gb) {
          const int col_next = j + 1 < len ? rl.col(j + 1) : 0;
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
    FA_F1T_TEARDOWN();
  } else if (warp == 9) {
    // ===================== MMA issuer (whole warp, one elected lane issues) =====================
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
        umma_commit(&sm.k_empty[ks]);  // K_j's only reader
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
          // P of half w (kv 64w..64w+63) sits in columns [64w, 64w + 32) of S_g
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
      RowList rl;
      rl.init(p, it);
      const int len = rl.len();
      mbar_wait(&sm.q_full[buf], (n >> 1) & 1);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sm.q[buf]);
      if (len == 0) {
        commit(&sm.q_free[buf]);
        continue;
      }
      issue_qk(gb, q_addr);
      if (len == 1) commit(&sm.q_free[buf]);
      mbar_wait(&sm.o_free, (no & 1) ^ 1);  // the previous item's O was read out
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
    FA_F1T_TEARDOWN();
  } else {
    // ===================== softmax (thread = q row, half of every block's columns) =====================
    reg_alloc<224>();
    const int wg = warp >> 2;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
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
      RowList rl;
      rl.init(p, it);
      const int len = rl.len();
      const int qi = it.r * kTile + row;
      const bool q_ok = qi < p.Lq;
      const long long slot = (static_cast<long long>(it.b) * p.Hq + it.h) * p.Lq + qi;
      __nv_bfloat16* orow = p.out + slot * D + wg * (D / 2);
      if (len == 0) {  // no visited block: O = 0, lse = -inf
        if (q_ok) {
          for (int u = 0; u < D / 16; ++u) reinterpret_cast<uint4*>(orow)[u] = make_uint4(0, 0, 0, 0);
          if (wg == 0) p.lse[slot] = -INFINITY;
        }
        continue;
      }
      float m = -INFINITY, l = 0.f;
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
        constexpr bool kPlain = ScoreT::kIdentity;
        const auto rowc = score.row(it.b, it.h, qi, kv0, p.scale);
        mbar_wait(&sm.s_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        uint32_t r[64];
        tmem_ld32(tm + s_col, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
        tmem_ld32(tm + s_col + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
        tmem_wait_ld();
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        auto pass1 = [&](auto masked) {
#pragma unroll
          for (int i = 0; i < 64; i += 2) {
            float v0 = __uint_as_float(r[i]), v1 = __uint_as_float(r[i + 1]);
            if constexpr (!kPlain) {
              const auto rc = rowc.shifted(i & ~31);
              v0 = rc.log2(v0, i & 31);
              v1 = rc.log2(v1, (i + 1) & 31);
            }
            if constexpr (decltype(masked)::value) {
              const uint32_t bw = i < 32 ? bits0 : bits1;
              v0 = ((bw >> (i & 31)) & 1u) ? v0 : -INFINITY;
              v1 = ((bw >> ((i + 1) & 31)) & 1u) ? v1 : -INFINITY;
            }
            if constexpr (!kPlain || decltype(masked)::value) {
              r[i] = __float_as_uint(v0);
              r[i + 1] = __float_as_uint(v1);
            }
            mx4[(i >> 1) & 3] = fmax3(mx4[(i >> 1) & 3], v0, v1);
          }
        };
        if (full) pass1(std::false_type{});
        else pass1(std::true_type{});
        float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        if constexpr (kPlain) mx *= rowc.c;
        // the other half's maximum of this row (parity-double-buffered slots, one barrier)
        sm.red[g & 1][wg][row] = mx;
        named_bar_sync(1, 256);
        mx = fmaxf(mx, sm.red[g & 1][wg ^ 1][row]);
        const float m_new = fmaxf(m, mx);
        const bool need = (m != -INFINITY) && (m_new > m + kRescaleThreshold);
        if (__any_sync(0xffffffffu, need)) {
          // O holds PV up to block g-1: wait for it, then rescale this half of the row
          mbar_wait(&sm.pv_done, (g - 1) & 1);
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
        tmem_st32(tm + s_col, pk);  // P over this half's first 32 S columns
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
      // ---- epilogue: the row sum of both halves, O / l -> bf16, lse ----
      sm.lred[wg][row] = l;
      named_bar_sync(1, 256);
      l += sm.lred[wg ^ 1][row];
      mbar_wait(&sm.o_full, no & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
      for (int cc = 0; cc < D / 64; ++cc) {
        uint32_t a[32];
        tmem_ld32(tm + o_col + cc * 32, a);
        tmem_wait_ld();
        if (q_ok) {
          uint4* d4 = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            d4[u] = make_uint4(pack_bf16(__uint_as_float(a[8 * u]) * inv, __uint_as_float(a[8 * u + 1]) * inv),
                               pack_bf16(__uint_as_float(a[8 * u + 2]) * inv, __uint_as_float(a[8 * u + 3]) * inv),
                               pack_bf16(__uint_as_float(a[8 * u + 4]) * inv, __uint_as_float(a[8 * u + 5]) * inv),
                               pack_bf16(__uint_as_float(a[8 * u + 6]) * inv, __uint_as_float(a[8 * u + 7]) * inv));
        }
      }
      if (q_ok && wg == 0) p.lse[slot] = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
      tc_fence_before();
      named_bar_sync(1, 256);  // both halves read lred before the next item writes it
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.o_free);
      ++no;
    }
    FA_F1T_TEARDOWN();
  }
#undef FA_F1T_TEARDOWN
}

template <int D, class MaskT, class ScoreT>
fa_status run(const AttnGeom& g, const void* q, const void* k, const void* v, void* o, float* lse, const BmView& bm,
              MaskT mask, ScoreT score, cudaStream_t st) {
  CUtensorMap mq, mk, mv;
  fa_status s;
  if ((s = make_map(&mq, q, g.B * g.Hq, g.Lq, D)) != FA_OK) return s;
  if ((s = make_map(&mk, k, g.Bkv * g.Hkv, g.Lkv, D)) != FA_OK) return s;
  if ((s = make_map(&mv, v, g.Bkv * g.Hkv, g.Lkv, D)) != FA_OK) return s;
  Params p{};
  p.out = static_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.B = g.B; p.Hq = g.Hq; p.Hkv = g.Hkv; p.Bkv = g.Bkv; p.Lq = g.Lq; p.Lkv = g.Lkv; p.G = g.G;
  p.bm_b = g.bm_b; p.bm_h = g.bm_h; p.rows = g.rows; p.cols = g.cols;
  p.kv_num = bm.kv_num; p.kv_idx = bm.kv_idx; p.full_num = bm.full_num; p.full_idx = bm.full_idx;
  p.scale = g.scale;
  p.num_items = g.B * g.Hq * g.rows;
  p.work_counter = scheduler_counter(kSlotFwdSched, st);
  FA_REQUIRE(p.work_counter != nullptr, FA_CUDA_ERROR, "forward: cannot allocate the scheduler counter");
  FA_CHECK_CUDA(cudaMemsetAsync(p.work_counter, 0, sizeof(int), st));
  const size_t smem = sizeof(Smem<D>);
  auto kern = flex_fwd1t_kernel<D, MaskT, ScoreT>;
  FA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = p.num_items < num_sms() ? p.num_items : num_sms();
  if (grid <= 0) return FA_OK;
  kern<<<grid, kThreads, smem, st>>>(mq, mk, mv, p, mask, score);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

inline bool supported(const AttnGeom& g) { return (g.D == 128 || g.D == 64) && g.bs_q == kTile && g.bs_kv == kTile; }

}  // namespace
}  // namespace fwd1t
}  // namespace fa
