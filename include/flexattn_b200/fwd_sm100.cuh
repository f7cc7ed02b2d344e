// fwd_sm100.cuh — block-sparse FlexAttention forward for sm_100a (bf16 in,
// fp32 accumulate), the tensor-core replacement of forward_impl
// (engine.cpp:46-163).
//
// Persistent, warp-specialised CTA (384 threads, 1 CTA/SM; setmaxnreg 224 for
// the softmax warpgroups, 56 for the rest). A work item is a pair of 128-row
// query tiles (block rows 2p, 2p+1) of one (b, h):
//   warps 0-3  softmax/correction/epilogue for tile 0   (thread = query row)
//   warps 4-7  the same for tile 1
//   warp  8    TMA producer: claims items (dynamic scheduler), loads the item's Q
//              tiles, then streams K_j, V_j (per visited block) with
//              cp.async.bulk.tensor into a 2-stage (D=128) ring. Empty blocks
//              are never loaded.
//   warp  10   list builder: the union of the two rows' visit lists (partial +
//              full) in descending block order (any order is exact math;
//              descending keeps the running max stable), built from per-lane
//              column bitmaps while warp 8 loads Q
//   warp  11   idle (completes the third warpgroup for setmaxnreg)
//   warp  9    MMA issuer (warp-uniform control, one elected lane issues): S_t = Q_t K_j^T (SS, TMEM fp32) and
//              O_t += P_t V_j (TS: P from TMEM as bf16, V from smem, MN-major),
//              ordered  QK0 QK1 | PV0(j) QK0(j+1) PV1(j) QK1(j+1) | ...  so the
//              two tiles' softmax ping-pong against the tensor core; P is released
//              in two parts so each PV starts on the first half of the block.
// TMEM (512 columns): S0 [0,128) S1 [128,256) (P_t aliases S_t's first 64
// columns as packed bf16), O0 [256, 256+D), O1 [256+D, 256+2D).
// Epilogue: O_t is released right after tile t's last PV; each softmax warp
// converts its 32 rows to bf16 in 32-column chunks through a 64-byte-swizzled
// smem tile written to global by TMA stores (rows past Q_LEN clipped).
//
// The softmax applies score_mod to every live score and mask_mod (with the
// q<Q_LEN, kv<KV_LEN bounds of bound_mask, block_mask.cpp:14-19) only in
// partial blocks; full blocks skip it. Rescaling of O is lazy: only when the
// row max grows by more than 2^8 (exact math either way, since the final
// normalisation uses the same stale max for O and l).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <type_traits>

#include "host.cuh"
#include "mods.cuh"
#include "sm100_ptx.cuh"

namespace fa {
namespace fwd {
namespace {  // internal linkage: every including translation unit has its own copy

#ifndef FA_FWD_EMU
#define FA_FWD_EMU 1  // part of the exponentials on the FMA pipe
#endif
#ifndef FA_FWD_EMU_EVERY
#define FA_FWD_EMU_EVERY 4  // one exponential pair in this many is emulated (soft-capped scores)
#endif
#ifndef FA_FWD_EMU_EVERY_UNIT
#define FA_FWD_EMU_EVERY_UNIT 8  // the same for the other scores (one MUFU per score: less to offload)
#endif
template <class ScoreT>
constexpr int emu_every() { return ScoreT::kUnitGrad ? FA_FWD_EMU_EVERY_UNIT : FA_FWD_EMU_EVERY; }
#ifndef FA_FWD_ALIBI_REG
#define FA_FWD_ALIBI_REG 1  // ALiBi column term of a 32-column chunk in registers (float2 pairs): +5 % C2
#endif
#ifndef FA_FWD_EARLY_O
#define FA_FWD_EARLY_O 1  // O_t released to the epilogue right after tile t's last PV
#endif
#ifndef FA_FWD_PPARTS
#define FA_FWD_PPARTS 2  // parts of P released separately (2 or 4; 4 measured -3 %)
#endif
constexpr int kPParts = FA_FWD_PPARTS;
constexpr int kThreads = 384;  // 2 softmax warpgroups + (producer, MMA, list builder, idle) warpgroup
constexpr int kTile = 128;           // query rows per tile == kv rows per block
constexpr int kMaxCols = 1024;       // max kv blocks per row (KV_LEN <= 131072)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct FwdParams {
  __nv_bfloat16* out;
  float* lse;
  int B, Hq, Hkv, Bkv, Lq, Lkv, G;
  int bm_b, bm_h, rows, cols;
  const int32_t* kv_num;
  const int32_t* kv_idx;
  const int32_t* full_num;
  const int32_t* full_idx;
  float scale, scale_log2;
  int npairs, num_items;
  int* work_counter;  // zeroed before launch; dynamic item scheduler
  long long* trace;   // debug only (FA_FWD_TRACE with an instrumented build)
};

// Compiled in only with -DFA_FWD_TRACE_BUILD=1. Slots [tile-step][event] of CTA 0.
#ifndef FA_FWD_TRACE_BUILD
#define FA_FWD_TRACE_BUILD 0
#endif
constexpr int kFTraceSteps = 512, kFTraceEv = 32;
__device__ __forceinline__ void ftrace(const FwdParams& p, int step, int ev) {
  if constexpr (FA_FWD_TRACE_BUILD != 0) {
    if (p.trace != nullptr && blockIdx.x == 0 && step < kFTraceSteps && (threadIdx.x & 31) == 0) {
      long long t;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
      p.trace[step * kFTraceEv + ev] = t;
    }
  }
}

template <int D>
struct Cfg {
  static constexpr int kChunks = D / 64;                  // 128-byte swizzle atoms along D
  static constexpr int kStages = (D == 128) ? 2 : 4;      // K/V ring depth
  static constexpr int kTileBytes = kTile * D * 2;        // one 128 x D bf16 tile
  static constexpr int kChunkBytes = kTile * 128;         // 128 rows x 128 B
};

template <int D>
struct alignas(1024) Smem {
  uint8_t q[2][Cfg<D>::kTileBytes];
  uint8_t k[Cfg<D>::kStages][Cfg<D>::kTileBytes];
  uint8_t v[Cfg<D>::kStages][Cfg<D>::kTileBytes];
  int32_t ulist[2][kMaxCols];
  uint32_t ubits[4][kMaxCols / 32];  // the list builder's column bitmaps
  int32_t claim_item[2];             // item handed to the list builder
  uint64_t claim_full[2];
  alignas(512) uint8_t ostage[8][32 * 64];  // epilogue: per softmax warp, 32 rows x 32 bf16 (64-byte swizzle)
  int32_t ulen[2];
  int32_t uitem[2];   // work item of the buffer, -1 = no more work
  uint64_t q_full[2], q_free[2];
  uint64_t k_full[Cfg<D>::kStages], v_full[Cfg<D>::kStages];
  uint64_t k_empty[Cfg<D>::kStages], v_empty[Cfg<D>::kStages];  // released separately
  uint64_t s_full[2], p_full[2][kPParts], o_full[2];  // p_full[tile][part of the kv block]
  uint64_t item_full[2], item_empty[2];
  uint32_t tmem_base;
};

// union-list entry: block column | tile-membership and full-block flags
constexpr uint32_t kIn0 = 1u << 24, kFull0 = 1u << 25, kIn1 = 1u << 26, kFull1 = 1u << 27;
constexpr uint32_t kColMask = (1u << 24) - 1;

struct Item {
  int b, h, pair;
};
__device__ __forceinline__ Item decode_item(const FwdParams& p, int item) {
  // heaviest (highest) row pairs first across all heads: a cheap LPT order for causal-like masks
  const int bh_count = p.B * p.Hq;
  const int pr = p.npairs - 1 - item / bh_count;
  const int bh = item % bh_count;
  return Item{bh / p.Hq, bh % p.Hq, pr};
}

template <int D, class MaskT, class ScoreT>
__global__ void __launch_bounds__(kThreads, 1)
    flex_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmO, const FwdParams p, MaskT mask,
                          ScoreT score) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<D>& sm = *reinterpret_cast<Smem<D>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm.q_full[t], 1);
      mbar_init(&sm.q_free[t], 1);
      mbar_init(&sm.s_full[t], 1);
      // split P (soft-capped scores): one arrival per warp and half; else per thread, [1] only
      for (int pp = 0; pp < kPParts; ++pp)
        mbar_init(&sm.p_full[t][pp], 4);  // one arrival per softmax warp
      mbar_init(&sm.o_full[t], 1);
      mbar_init(&sm.item_full[t], 1);
      mbar_init(&sm.item_empty[t], 1 + 8);
      mbar_init(&sm.claim_full[t], 1);
    }
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
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

  // Each role ends in its own copy of the teardown so no code is shared between warpgroups
  // with different setmaxnreg budgets (ptxas allocates registers per region).
#define FA_FWD_TEARDOWN()  \
  do {                     \
    tc_fence_before();     \
    __syncthreads();       \
    if (warp == 9) {       \
      tc_fence_after();    \
      tmem_dealloc(tmem, 512); \
    }                      \
    return;                \
  } while (0)
  if (warp >= 8) {
    reg_dealloc<56>();
    if (warp == 8 && lane == 0) {
      // ===================== TMA producer (lists built by warp 10) =====================
      // claims an item, hands it to the list builder, loads its Q tiles while the list is
      // being built, then streams the K/V blocks of the list
      int kv_it = 0;
      int item = static_cast<int>(blockIdx.x);
      for (int n = 0;; ++n) {
        const int buf = n & 1;
        mbar_wait(&sm.item_empty[buf], ((n >> 1) & 1) ^ 1);
        sm.claim_item[buf] = item;
        mbar_arrive(&sm.claim_full[buf]);
        if (item >= p.num_items) break;
        const Item it = decode_item(p, item);
        const int r0 = 2 * it.pair;
        // ---- Q tiles ----
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&sm.q_free[t], (n & 1) ^ 1);
          mbar_expect_tx(&sm.q_full[t], C::kTileBytes);
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_3d(sm.q[t] + ch * C::kChunkBytes, &tmQ, &sm.q_full[t], ch * 64,
                        (r0 + t) * kTile, it.b * p.Hq + it.h);
        }
        ftrace(p, n, 20);
        mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
        const int len = sm.ulen[buf];
        // ---- K/V blocks ----
        const int kb = p.Bkv == 1 ? 0 : it.b, kh = it.h / p.G;
        for (int j = 0; j < len; ++j, ++kv_it) {
          const int st = kv_it % C::kStages;
          const int colb = static_cast<int>(static_cast<uint32_t>(sm.ulist[buf][j]) & kColMask);
          mbar_wait(&sm.k_empty[st], ((kv_it / C::kStages) & 1) ^ 1);
          ftrace(p, kv_it, 12);
          if (j == 0) ftrace(p, n, 26);
          mbar_expect_tx(&sm.k_full[st], C::kTileBytes);
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_3d(sm.k[st] + ch * C::kChunkBytes, &tmK, &sm.k_full[st], ch * 64,
                        colb * kTile, kb * p.Hkv + kh);
          mbar_wait(&sm.v_empty[st], ((kv_it / C::kStages) & 1) ^ 1);
          ftrace(p, kv_it, 13);
          mbar_expect_tx(&sm.v_full[st], C::kTileBytes);
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_3d(sm.v[st] + ch * C::kChunkBytes, &tmV, &sm.v_full[st], ch * 64,
                        colb * kTile, kb * p.Hkv + kh);
        }
        item = static_cast<int>(gridDim.x) + atomicAdd(p.work_counter, 1);
      }
    } else if (warp == 10) {
      // ===================== list builder =====================
      // the union of the item's two rows' visit lists in descending block order (blocks nearest
      // the diagonal first, so the running max is established early): one bitmap word of 32
      // block columns per lane, two global round trips
      for (int n = 0;; ++n) {
        const int buf = n & 1;
        mbar_wait(&sm.claim_full[buf], (n >> 1) & 1);
        const int item = *reinterpret_cast<volatile int32_t*>(&sm.claim_item[buf]);
        if (item >= p.num_items) {
          if (lane == 0) {
            sm.uitem[buf] = -1;
            mbar_arrive(&sm.item_full[buf]);
          }
          break;
        }
        const Item it = decode_item(p, item);
        const int mb = p.bm_b == 1 ? 0 : it.b, mh = p.bm_h == 1 ? 0 : it.h;
        const int r0 = 2 * it.pair, r1 = r0 + 1;
        const long long s0 = (static_cast<long long>(mb) * p.bm_h + mh) * p.rows + r0;
        const int np0 = __ldg(p.kv_num + s0), nf0 = __ldg(p.full_num + s0);
        const int np1 = r1 < p.rows ? __ldg(p.kv_num + s0 + 1) : 0;
        const int nf1 = r1 < p.rows ? __ldg(p.full_num + s0 + 1) : 0;
        const int32_t* pi0 = p.kv_idx + s0 * p.cols;
        const int32_t* fi0 = p.full_idx + s0 * p.cols;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) sm.ubits[q4][lane] = 0u;
        __syncwarp();
        auto scatter = [&](const int32_t* idx, int cnt, int which) {
          for (int i = lane; i < cnt; i += 32) {
            const int c = __ldg(idx + i);
            atomicOr(&sm.ubits[which][c >> 5], 1u << (c & 31));
          }
        };
        scatter(pi0, np0, 0);
        scatter(fi0, nf0, 1);
        scatter(pi0 + p.cols, np1, 2);
        scatter(fi0 + p.cols, nf1, 3);
        __syncwarp();
        const uint32_t bp0 = sm.ubits[0][lane], bf0 = sm.ubits[1][lane];
        const uint32_t bp1 = sm.ubits[2][lane], bf1 = sm.ubits[3][lane];
        const uint32_t in0 = bp0 | bf0, in1 = bp1 | bf1, any = in0 | in1;
        const int cnt = __popc(any);
        int incl = cnt;  // entries of this lane and the higher (larger column) lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_down_sync(0xffffffffu, incl, o);
          if (lane + o < 32) incl += v;
        }
        int pos = incl - cnt;
        for (uint32_t rem = any; rem != 0u;) {
          const int bit = 31 - __clz(rem);
          const uint32_t mbit = 1u << bit;
          rem &= ~mbit;
          uint32_t e = static_cast<uint32_t>(lane * 32 + bit);
          if (in0 & mbit) e |= kIn0;
          if (bf0 & mbit) e |= kFull0;
          if (in1 & mbit) e |= kIn1;
          if (bf1 & mbit) e |= kFull1;
          sm.ulist[buf][pos++] = static_cast<int32_t>(e);
        }
        if (lane == 0) {
          sm.ulen[buf] = incl;  // lane 0: all entries
          sm.uitem[buf] = item;
        }
        __threadfence_block();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&sm.item_full[buf]);
          ftrace(p, n, 19);
        }
      }
    } else if (warp == 9) {
      // ===================== MMA issuer =====================
      // The whole warp runs the (warp-uniform) control flow and one elected lane issues:
      // descriptors then live in uniform registers and each tcgen05.mma is one UTCHMMA
      // (a lane-0-only branch makes ptxas wrap every MMA in an ELECT/R2UR waterfall loop).
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, D, 0, 1);
      const uint32_t q_addr[2] = {smem_u32(sm.q[0]), smem_u32(sm.q[1])};
      uint32_t p_phase[2] = {0, 0};
      int mg[2] = {0, 0};  // per-tile step counters (trace only)
      int kv_it = 0;
      int n = 0;
      // descriptors rebuilt per GEMM from an opaque base (+ K-step offsets in the address
      // field): ptxas would otherwise hoist them all out of the loop and spill
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) umma_commit(bar);
        __syncwarp();
      };
      auto issue_qk = [&](int t, int st) {
        if (elect_one()) {
          const uint64_t a0 = make_sdesc_sw128(q_addr[t], 16, 1024);
          const uint64_t b0 = make_sdesc_sw128(smem_u32(sm.k[st]), 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * C::kChunkBytes + (kk & 3) * 32) >> 4;
            umma_ss(tm + t * 128, a0 + off, b0 + off, idesc_qk, kk > 0 ? 1u : 0u);
          }
          umma_commit(&sm.s_full[t]);
        }
        __syncwarp();
      };
      // O_t += P_t V: each part of the kv block (128 / kPParts kv, P columns of that part) as
      // soon as the softmax released it
      auto issue_pv = [&](int t, int st, bool acc, uint32_t ph) {
        const uint64_t b0 = make_sdesc_sw128(smem_u32(sm.v[st]), C::kChunkBytes, 1024);
        constexpr int kSteps = (kTile / 16) / kPParts;
#pragma unroll
        for (int hf = 0; hf < kPParts; ++hf) {
          mbar_wait(&sm.p_full[t][hf], ph);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = hf * kSteps; kk < hf * kSteps + kSteps; ++kk)
              umma_ts(tm + 256 + t * D, tm + t * 128 + kk * 8, b0 + kk * (2048 >> 4), idesc_pv,
                      (acc || kk > 0) ? 1u : 0u);
          }
          __syncwarp();
        }
      };
      for (;; ++n) {
        const int buf = n & 1;
        mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
        if (sm.uitem[buf] < 0) break;
        const int len = sm.ulen[buf];
        const uint32_t* U = reinterpret_cast<const uint32_t*>(sm.ulist[buf]);
        mbar_wait(&sm.q_full[0], n & 1);
        mbar_wait(&sm.q_full[1], n & 1);
        ftrace(p, n, 21);
        tc_fence_after();
        // last step that reads Q_t: Q_t's smem is released (q_free) as soon as that QK completes
        int last_qk[2] = {-1, -1};
        for (int j = 0; j < len; ++j) {
          if (U[j] & kIn0) last_qk[0] = j;
          if (U[j] & kIn1) last_qk[1] = j;
        }
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (last_qk[t] < 0) commit(&sm.q_free[t]);
        bool first_pv[2] = {true, true};
        if (len > 0) {
          const int st0 = kv_it % C::kStages;
          mbar_wait(&sm.k_full[st0], (kv_it / C::kStages) & 1);
          tc_fence_after();
          const uint32_t e0 = U[0];
          ftrace(p, n, 24);
          if (e0 & kIn0) { issue_qk(0, st0); if (last_qk[0] == 0) commit(&sm.q_free[0]); }
          if (e0 & kIn1) { issue_qk(1, st0); if (last_qk[1] == 0) commit(&sm.q_free[1]); }
          commit(&sm.k_empty[st0]);
        }
        for (int j = 0; j < len; ++j) {
          const int it_j = kv_it + j;
          const int st = it_j % C::kStages;
          const uint32_t e = U[j];
          const uint32_t en = (j + 1 < len) ? U[j + 1] : 0u;
          const int st1 = (it_j + 1) % C::kStages;
          bool k1_ready = false;
          ftrace(p, it_j, 15);
          mbar_wait(&sm.v_full[st], (it_j / C::kStages) & 1);
          ftrace(p, it_j, 14);
          tc_fence_after();
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const uint32_t in_bit = t == 0 ? kIn0 : kIn1;
            if (e & in_bit) {
              ftrace(p, mg[t], 4 + t);
              issue_pv(t, st, !first_pv[t], p_phase[t]);
              ftrace(p, mg[t], 8 + t);
              p_phase[t] ^= 1;
              first_pv[t] = false;
              ++mg[t];
              // O_t is final once tile t's last PV completes: its epilogue need not wait for
              // the other tile's last PV
              if (FA_FWD_EARLY_O != 0 && last_qk[t] == j) commit(&sm.o_full[t]);
            }
            if (en & in_bit) {
              if (!k1_ready) {
                mbar_wait(&sm.k_full[st1], ((it_j + 1) / C::kStages) & 1);
                tc_fence_after();
                k1_ready = true;
              }
              ftrace(p, mg[t], 10 + t);
              issue_qk(t, st1);
              ftrace(p, mg[t], 6 + t);
              if (last_qk[t] == j + 1) commit(&sm.q_free[t]);
            }
          }
          if (k1_ready) commit(&sm.k_empty[st1]);
          commit(&sm.v_empty[st]);
        }
        kv_it += len;
        for (int t = 0; t < 2; ++t)
          if (FA_FWD_EARLY_O == 0 || last_qk[t] < 0) commit(&sm.o_full[t]);
        ftrace(p, n, 22);
        if (lane == 0) mbar_arrive(&sm.item_empty[buf]);
      }
    }
    FA_FWD_TEARDOWN();
  } else {
    // ===================== softmax / correction / epilogue =====================
    reg_alloc<224>();
    const int t = warp >> 2;               // tile
    const int wq = warp & 3;               // TMEM lane quarter
    const int row = wq * 32 + lane;        // query row within the tile
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t s_tm = tmem + lane_base + t * 128;
    const uint32_t o_tm = tmem + lane_base + 256 + t * D;
    const uint32_t in_bit = t == 0 ? kIn0 : kIn1;
    const uint32_t full_bit = t == 0 ? kFull0 : kFull1;
    uint32_t s_phase = 0;
    int n = 0, gs = 0;
    for (;; ++n) {
      const int buf = n & 1;
      mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
      const int item = sm.uitem[buf];
      if (item < 0) break;
      const Item it = decode_item(p, item);
      const int len = sm.ulen[buf];
      const int qi = (2 * it.pair + t) * kTile + row;
      // ALiBi in registers: the column term step·i of a 32-column chunk as 16 float2 pairs (per
      // item: the slope is the head's); the chunk's offset (row term + step·32·chunk) joins the
      // max and the exponent per chunk, so a pair of scores costs one FFMA2
      constexpr bool kAlibiReg = FA_FWD_ALIBI_REG != 0 && ScoreT::kKind == 1;
      float2 abias[16];
      if constexpr (kAlibiReg) {
        const float st = -__ldg(score.p.slopes + it.h) * kLog2e;
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) abias[k2] = make_float2(st * (2 * k2), st * (2 * k2 + 1));
      }
      float m = -INFINITY, l = 0.f;
      bool any_blocks = false;
      for (int j = 0; j < len; ++j) {
        const uint32_t e = static_cast<uint32_t>(sm.ulist[buf][j]);
        if (!(e & in_bit)) continue;
        any_blocks = true;
        const bool full = (e & full_bit) != 0;
        const int kv0 = static_cast<int>(e & kColMask) * kTile;
        mbar_wait(&sm.s_full[t], s_phase);
        s_phase ^= 1;
        tc_fence_after();
        if (row == 0) ftrace(p, gs, t * 2 + 0);
        // One TMEM read of the whole 128-score row into registers: score_mod in the log2
        // domain (+ mask_mod and bounds in partial blocks) and the row max, then the
        // exponentials straight from registers. A plain (identity) score keeps raw scores
        // and scales the max once (c > 0 commutes with max).
        constexpr bool kPlain = ScoreT::kIdentity;
        const auto rowc = score.row(it.b, it.h, qi, kv0, p.scale);
        uint32_t r[128];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
          tmem_ld32(s_tm + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[cc * 32]));
        uint32_t bits[4] = {~0u, ~0u, ~0u, ~0u};
        if (!full) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            bits[cc] = qi < p.Lq ? mask.bits32(it.b, it.h, qi, kv0 + cc * 32, p.Lkv) : 0u;
        }
        tmem_wait_ld();
        if (row == 0) ftrace(p, gs, 16);
        // score_mod (log2 domain) and mask_mod of the score pair (i, i+1), from r
        auto score_pair = [&](int i, auto masked, float& v0, float& v1) {
          v0 = __uint_as_float(r[i]);
          v1 = __uint_as_float(r[i + 1]);
          if constexpr (kAlibiReg) {
            // chunk-relative: s·c + step·(i mod 32); max accumulator = the chunk
            const float2 vv = __ffma2_rn(make_float2(v0, v1), make_float2(rowc.c, rowc.c), abias[(i & 31) >> 1]);
            v0 = vv.x;
            v1 = vv.y;
          } else if constexpr (!kPlain) {
            const auto rc = rowc.shifted(i & ~31);
            v0 = rc.log2(v0, i & 31);
            v1 = rc.log2(v1, (i + 1) & 31);
          }
          if constexpr (decltype(masked)::value) {
            v0 = ((bits[i >> 5] >> (i & 31)) & 1u) ? v0 : -INFINITY;
            v1 = ((bits[i >> 5] >> ((i + 1) & 31)) & 1u) ? v1 : -INFINITY;
          }
        };
        auto max_acc = [&](float (&acc)[4], int i, float v0, float v1) {
          if constexpr (kAlibiReg) acc[i >> 5] = fmax3(acc[i >> 5], v0, v1);
          else acc[(i >> 1) & 3] = fmax3(acc[(i >> 1) & 3], v0, v1);
        };
        // the row max of the block from the accumulators (ALiBi chunk offsets added, a plain
        // score scaled once)
        float coff[4] = {0.f, 0.f, 0.f, 0.f};  // ALiBi chunk offsets (kAlibiReg)
        if constexpr (kAlibiReg) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) coff[cc] = rowc.shifted(32 * cc).base;
        }
        auto block_max = [&](float (&acc)[4]) {
          if constexpr (kAlibiReg) {
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) acc[cc] += coff[cc];  // -inf stays -inf
          }
          float mx = fmaxf(fmaxf(acc[0], acc[1]), fmaxf(acc[2], acc[3]));
          if constexpr (kPlain) mx *= rowc.c;
          return mx;
        };
        const float2 xs2 = make_float2(kPlain ? rowc.c : 1.f, kPlain ? rowc.c : 1.f);
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        auto pass1 = [&](auto masked) {
#pragma unroll
          for (int i = 0; i < 128; i += 2) {
            float v0, v1;
            score_pair(i, masked, v0, v1);
            if constexpr (!kPlain || decltype(masked)::value) {
              r[i] = __float_as_uint(v0);
              r[i + 1] = __float_as_uint(v1);
            }
            max_acc(mx4, i, v0, v1);
          }
        };
        if (full) pass1(std::false_type{});
        else pass1(std::true_type{});
        const float mx = block_max(mx4);
        // lazy rescale (warp-uniform decision; tcgen05.ld/st are warp-collective)
        const float m_new = fmaxf(m, mx);
        const bool need = (m != -INFINITY) && (m_new > m + kRescaleThreshold);
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = need ? ex2(m - m_new) : 1.f;
#pragma unroll 1
          for (int cc = 0; cc < D / 32; ++cc) {
            uint32_t o[32];
            tmem_ld32(o_tm + cc * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(o_tm + cc * 32, o);
          }
          l *= alpha;
        }
        if (need || m == -INFINITY) m = m_new;
        if (row == 0) ftrace(p, gs, 17);
        const float msub = (m == -INFINITY) ? 0.f : m;
        // P = exp2(x - m) as packed bf16 over S's first 64 columns (column c: kv 2c, 2c+1).
        // Each part of P releases its PV MMAs on its own (p_full[t][part]) so the tensor core
        // starts on the first kv of the block while the exponentials of the rest run. One
        // exponential pair in emu_every() runs on the FMA pipe (exp2_poly2, exactly 0 for a
        // masked score), chosen by column alone, so a block gives the same P whether it is
        // classified full or partial (demote_full_to_partial / promote stay bit-exact).
        float nmv = -msub;
        const float2 nm2 = make_float2(nmv, nmv);
        float2 ls[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
        {
          constexpr int kPairs = 64 / kPParts;  // packed P columns per part
          auto exp_part = [&](int hf) {
            uint32_t pk[kPairs];
#pragma unroll
            for (int k = 0; k < kPairs; ++k) {
              const int i = hf * kPairs + k;
              float2 nmc = nm2;
              if constexpr (kAlibiReg) nmc = make_float2(nm2.x + coff[i >> 4], nm2.y + coff[i >> 4]);
              const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])),
                                          xs2, nmc);
              float2 pv;
              if (FA_FWD_EMU != 0 && (k % emu_every<ScoreT>()) == emu_every<ScoreT>() - 1)
                pv = exp2_poly2(x);
              else pv = make_float2(ex2(x.x), ex2(x.y));
              ls[k & 3] = __fadd2_rn(ls[k & 3], pv);
              pk[k] = pack_bf16(pv.x, pv.y);
            }
            if constexpr (kPairs == 32) tmem_st32(s_tm + hf * kPairs, *reinterpret_cast<uint32_t(*)[32]>(pk));
            else tmem_st16(s_tm + hf * kPairs, *reinterpret_cast<uint32_t(*)[16]>(pk));
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.p_full[t][hf]);
          };
#pragma unroll
          for (int hf = 0; hf < kPParts; ++hf) exp_part(hf);
        }
        const float2 l01 = __fadd2_rn(ls[0], ls[1]), l23 = __fadd2_rn(ls[2], ls[3]);
        const float2 lt = __fadd2_rn(l01, l23);
        l += lt.x + lt.y;
        if (row == 0) ftrace(p, gs, 18);
        if (row == 0) ftrace(p, gs, t * 2 + 1);
        ++gs;
      }
      // ---- epilogue: O / l -> bf16, lse ----
      mbar_wait(&sm.o_full[t], n & 1);
      if (row == 0 && t == 0) ftrace(p, n, 23);
      tc_fence_after();
      const bool valid = qi < p.Lq;
      const long long slot = (static_cast<long long>(it.b) * p.Hq + it.h) * p.Lq + qi;
      __nv_bfloat16* orow = p.out + slot * D;
      if (any_blocks) {
        // 32 columns at a time through a per-warp 64-byte-swizzled smem tile and one TMA store of
        // 32 rows x 32 columns (row-per-thread global stores touch 32 lines per instruction and
        // kept the LSU busy ~5000 cycles at every item boundary)
        const float inv = l > 0.f ? 1.f / l : 0.f;
        uint8_t* stg = sm.ostage[warp];
        const int qrow0 = (2 * it.pair + t) * kTile + wq * 32;
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t r0[32];
          tmem_ld32(o_tm + cc * 32, r0);
          tmem_wait_ld();
          if (row == 0 && t == 0) ftrace(p, n, 27 + cc);
          if (lane == 0) bulk_wait_group_read<0>();  // the previous TMA store has read the tile
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(r0[8 * k + 0]) * inv, __uint_as_float(r0[8 * k + 1]) * inv);
            w.y = pack_bf16(__uint_as_float(r0[8 * k + 2]) * inv, __uint_as_float(r0[8 * k + 3]) * inv);
            w.z = pack_bf16(__uint_as_float(r0[8 * k + 4]) * inv, __uint_as_float(r0[8 * k + 5]) * inv);
            w.w = pack_bf16(__uint_as_float(r0[8 * k + 6]) * inv, __uint_as_float(r0[8 * k + 7]) * inv);
            *reinterpret_cast<uint4*>(stg + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4)) = w;
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmO, stg, cc * 32, qrow0, it.b * p.Hq + it.h);
            bulk_commit_group();
          }
        }
      } else if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(orow);
        for (int v4 = 0; v4 < D / 8; ++v4) dst[v4] = make_uint4(0, 0, 0, 0);
      }
      if (valid) p.lse[slot] = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
      if (row == 0 && t == 0) ftrace(p, n, 25);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.item_empty[buf]);
    }
    if (lane == 0) bulk_wait_group<0>();  // the epilogue's TMA stores have landed
    __syncwarp();
    FA_FWD_TEARDOWN();
  }
#undef FA_FWD_TEARDOWN
}

// ---------------------------------------------------------------- host side
template <int D, class MaskT, class ScoreT>
fa_status run(const AttnGeom& g, const void* q, const void* k, const void* v, void* o, float* lse,
              const BmView& bm, MaskT mask, ScoreT score, cudaStream_t st) {
  CUtensorMap mq, mk, mv, mo{};
  fa_status s;
  if ((s = make_map(&mq, q, g.B * g.Hq, g.Lq, D)) != FA_OK) return s;
  {
    const CUresult r = encode_o32_map(&mo, o, g.B * g.Hq, g.Lq, D);
    FA_REQUIRE(r == CUDA_SUCCESS, FA_CUDA_ERROR,
               "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  }
  if ((s = make_map(&mk, k, g.Bkv * g.Hkv, g.Lkv, D)) != FA_OK) return s;
  if ((s = make_map(&mv, v, g.Bkv * g.Hkv, g.Lkv, D)) != FA_OK) return s;
  FwdParams p{};
  p.out = static_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.B = g.B; p.Hq = g.Hq; p.Hkv = g.Hkv; p.Bkv = g.Bkv; p.Lq = g.Lq; p.Lkv = g.Lkv; p.G = g.G;
  p.bm_b = g.bm_b; p.bm_h = g.bm_h; p.rows = g.rows; p.cols = g.cols;
  p.kv_num = bm.kv_num; p.kv_idx = bm.kv_idx; p.full_num = bm.full_num; p.full_idx = bm.full_idx;
  p.scale = g.scale;
  p.scale_log2 = g.scale * kLog2e;
  p.npairs = (g.rows + 1) / 2;
  p.num_items = g.B * g.Hq * p.npairs;
  p.work_counter = scheduler_counter(kSlotFwdSched, st);
  long long* trace = nullptr;
  if (FA_FWD_TRACE_BUILD != 0 && getenv("FA_FWD_TRACE") != nullptr) {
    FA_CHECK_CUDA(cudaMalloc(&trace, sizeof(long long) * kFTraceSteps * kFTraceEv));
    FA_CHECK_CUDA(cudaMemsetAsync(trace, 0, sizeof(long long) * kFTraceSteps * kFTraceEv, st));
  }
  p.trace = trace;
  FA_REQUIRE(p.work_counter != nullptr, FA_CUDA_ERROR, "forward: cannot allocate the scheduler counter");
  FA_CHECK_CUDA(cudaMemsetAsync(p.work_counter, 0, sizeof(int), st));
  const size_t smem = sizeof(Smem<D>) + 1024;
  auto kern = flex_fwd_sm100_kernel<D, MaskT, ScoreT>;
  FA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = p.num_items < num_sms() ? p.num_items : num_sms();
  if (grid <= 0) return FA_OK;
  kern<<<grid, kThreads, smem, st>>>(mq, mk, mv, mo, p, mask, score);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  if (trace != nullptr) {  // debug: per-step events of CTA 0 (tile 0 and 1)
    static long long h[kFTraceSteps * kFTraceEv];
    FA_CHECK_CUDA(cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st));
    FA_CHECK_CUDA(cudaStreamSynchronize(st));
    cudaFree(trace);
    const int s_lo = getenv("FA_FWD_TRACE_FROM") ? atoi(getenv("FA_FWD_TRACE_FROM")) : 20;
    const int s_hi = s_lo + (getenv("FA_FWD_TRACE_FROM") ? 24 : 8);
    const long long t0 = h[20 * kFTraceEv];
    for (int s = s_lo; s < s_hi; ++s) {
      const long long* e = h + s * kFTraceEv;
      fprintf(stderr, "[fwd trace] step %d: S0seen %lld P0done %lld PV0 %lld..%lld QK0 %lld..%lld | S1seen %lld P1done %lld PV1 %lld..%lld QK1 %lld..%lld\n",
              s, e[0] - t0, e[1] - t0, e[4] - t0, e[8] - t0, e[10] - t0, e[6] - t0, e[2] - t0, e[3] - t0,
              e[5] - t0, e[9] - t0, e[11] - t0, e[7] - t0);
    }
    for (int s = s_lo; s < s_hi; ++s) {
      const long long* e = h + s * kFTraceEv;
      fprintf(stderr, "[fwd trace] softmax0 step %d: ld %lld  max %lld  exp+st %lld  end %lld\n", s, e[16] - e[0],
              e[17] - e[16], e[18] - e[17], e[1] - e[18]);
    }
    for (int s = s_lo; s < s_hi; ++s) {
      const long long* e = h + s * kFTraceEv;
      fprintf(stderr, "[fwd trace] block %d: K issued %lld  V issued %lld  MMA wants V %lld  V seen %lld\n", s,
              e[12] - t0, e[13] - t0, e[15] - t0, e[14] - t0);
    }
    for (int n = 0; n < 12; ++n) {
      const long long* e = h + n * kFTraceEv;
      fprintf(stderr, "[fwd trace] item %d: list %lld  Q issued %lld  K0 issued %lld  MMA has Q %lld  first QK %lld  MMA item end %lld  epi0 %lld..%lld (ld %lld %lld %lld %lld)\n", n,
              e[19] - t0, e[20] - t0, e[26] - t0, e[21] - t0, e[24] - t0, e[22] - t0, e[23] - t0, e[25] - t0,
              e[27] - e[23], e[28] - e[23], e[29] - e[23], e[30] - e[23]);
    }
    double sm0 = 0, per = 0;
    int cnt = 0;
    for (int s = 1; s + 1 < kFTraceSteps; ++s) {
      const long long* e = h + s * kFTraceEv;
      const long long* en = h + (s + 1) * kFTraceEv;
      if (e[0] == 0 || e[1] == 0 || en[0] == 0) break;
      sm0 += e[1] - e[0];
      per += en[0] - e[0];
      ++cnt;
    }
    if (cnt) fprintf(stderr, "[fwd trace] steps=%d softmax0 %.0f cycles, tile-0 period %.0f cycles\n", cnt, sm0 / cnt, per / cnt);
  }
  return FA_OK;
}

// Shapes the tensor-core forward is compiled for (else the CUDA-core forward runs).
inline bool supported(const AttnGeom& g) {
  return (g.D == 128 || g.D == 64) && g.bs_q == kTile && g.bs_kv == kTile && g.cols <= kMaxCols;
}

}  // namespace
}  // namespace fwd
}  // namespace fa
