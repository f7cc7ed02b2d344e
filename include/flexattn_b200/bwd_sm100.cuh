// bwd_sm100.cuh — block-sparse FlexAttention backward for sm_100a (bf16 in, fp32
// accumulate), the tensor-core replacement of backward (engine.cpp:174-401).
//
// Kernels (one stream, in order):
//   1. preprocess: Δ_i = Σ_d dO·O (engine.cpp:218-235) and the compute warps' log2-domain
//      column term log2(scale) - lse·log2e (-inf on fully masked rows so they contribute
//      exactly nothing, :257-260), both padded to 128-row q blocks; zeroes the fp32 dQ
//      accumulator (fused mode).
//   2. main: persistent, warp-specialised CTA (512 threads; setmaxnreg 144 compute / 160 dQ
//      reduction / 64 producer+MMA). A work item is one 128-row kv block of one (kv batch,
//      kv head) — the dK/dV pass of the reference (:307-395): it loops the kv-batch broadcast
//      and the G query heads of the group and walks the transposed (q-side) lists, so dK and
//      dV accumulate in TMEM for the whole item. Per visited q block t:
//        S^T  = K Q^T          (SS)             -> TMEM S    [0,128)
//        dP^T = V dO^T         (SS)             -> TMEM dP   [128,256)
//        compute warps, phase A (after S^T): (P·scale)^T = exp2(s·c + cterm), mask_mod only
//           in partial blocks, as bf16 into TMEM over S^T (dV is rescaled by 1/scale in the
//           epilogue); P·scale·mod' kept in registers (fp32)
//        compute warps, phase B (after dP^T): dS^T = P (dP^T - Δ) mod' scale (bf16) into the
//           smem dS^T buffer
//        dV  += P^T dO          (TS: P^T from TMEM)
//        dK  += dS^T Q          (SS: dS^T from the smem buffer)
//        dQ^T = K^T dS^T        (SS, both MN-major) -> TMEM over the dP columns
//      The MMA warp software-pipelines consecutive blocks so the tensor core runs the
//      GEMMs of one block while the compute warps work on the next:
//          S(t+1) | dQ(t) | dK(t) | dP(t+1) | dV(t+1) | S(t+2) | ...
//      dQ (the fused form of the reference's separate dQ pass, :237-305) is drained from
//      TMEM by the reduction warpgroup into per-warp 32x32 fp32 smem tiles and added into
//      the fp32 accumulator in L2 with TMA cp.reduce.async.bulk.tensor (add). The order of
//      those adds across kv blocks is not fixed, so the fused dQ is not bitwise reproducible
//      run to run; FA_FLAG_DETERMINISTIC runs the split backward instead (kModeNoDQ here,
//      dK/dV only, plus the dQ pass of bwd_dq.cuh).
//      Warps 0-7 compute (two warpgroups, 64 q columns each; thread = kv row),
//      warps 8-11 dQ reduction + dK/dV epilogue, warp 12 TMA producer, warp 13 MMA.
//   3. convert: dQ fp32 -> bf16 (fused mode).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <type_traits>

#include "bwd_dq.cuh"
#include "host.cuh"
#include "mods.cuh"
#include "sm100_ptx.cuh"

namespace fa {
namespace bwd {
namespace {  // internal linkage: every including translation unit has its own copy

constexpr int kThreads = 512;  // 2 compute WGs + dQ/epilogue WG + producer/MMA WG
constexpr int kTile = 128;
constexpr float kLog2e = 1.4426950408889634f;

struct BwdParams {
  int B, Hq, Hkv, Bkv, Lq, Lkv, G, Lq_pad;
  int bm_b, bm_h, rows, cols;
  const int32_t* q_num;
  const int32_t* q_idx;
  const int32_t* fq_num;
  const int32_t* fq_idx;
  const int32_t* kv_num;   // kv side (deterministic mode: rank of a kv block in a q row's list)
  const int32_t* kv_idx;
  const int32_t* fkv_num;
  const int32_t* fkv_idx;
  const float* lse2;   // (B*Hq, Lq_pad): cterm, see bwd_preprocess_kernel
  const float* delta;  // (B*Hq, Lq_pad)
  float* dq_acc;       // (B*Hq, Lq, D) fp32
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  float scale;
  int num_items;
  int* work_counter;
  long long* trace;  // debug only (FA_BWD_TRACE): per-block phase timestamps of CTA 0
};

// trace slots [block][event] of CTA 0 (FA_BWD_TRACE); see the host-side summary in run().
// Compiled in only with -DFA_BWD_TRACE_BUILD=1 (make EXTRA=-DFA_BWD_TRACE_BUILD=1).
#ifndef FA_BWD_TRACE_BUILD
#define FA_BWD_TRACE_BUILD 0
#endif
constexpr int kTraceTasks = 256, kTraceEv = 24;
__device__ __forceinline__ void trace_ev(const BwdParams& p, int task, int ev) {
  if constexpr (FA_BWD_TRACE_BUILD != 0) {
    if (p.trace != nullptr && blockIdx.x == 0 && task < kTraceTasks && (threadIdx.x & 31) == 0) {
      long long t;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
      p.trace[task * kTraceEv + ev] = t;
    }
  }
}

#ifndef FA_BWD_DKSS
#define FA_BWD_DKSS 1  // dK as an SS MMA from the dS^T smem buffer, issued after dQ
#endif
constexpr bool kDkSS = FA_BWD_DKSS != 0;

#ifndef FA_BWD_REG_REDUCE
#define FA_BWD_REG_REDUCE 160  // setmaxnreg of the dQ reduction / epilogue warpgroup (128-column drain)
#endif
#ifndef FA_BWD_REG_OTHER
#define FA_BWD_REG_OTHER 64  // setmaxnreg of the producer / MMA warpgroup (160/64: +1..2 %, fewer spills)
#endif
#ifndef FA_BWD_PAIRED
#define FA_BWD_PAIRED 0  // 1: phase A's exponents of plain / ALiBi scores as FFMA2 pairs
#endif
#ifndef FA_BWD_NODQ_DO2
#define FA_BWD_NODQ_DO2 1  // split mode (no dQ staging): two dO stages
#endif
#ifndef FA_BWD_L2PF
#define FA_BWD_L2PF 0  // 1: L2 prefetch of the next task's Q / dO tiles (one task ahead)
#endif
#ifndef FA_BWD_DK_FIRST
#define FA_BWD_DK_FIRST 0  // 1: issue dK(b) before dQ(b) (frees Q(b) earlier, delays the dQ chain)
#endif
#ifndef FA_BWD_DQ_TMA
#define FA_BWD_DQ_TMA 1
#endif
template <int D>
struct BCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = kTile * D * 2;
  static constexpr int kChunkBytes = kTile * 128;
  // dQ goes to L2 by TMA reduce-add from per-warp smem staging tiles (kTmaReduce) or by
  // red.global.add from registers; at D = 128 the staging costs one dO stage (227 KB budget)
  static constexpr bool kTmaReduce = FA_BWD_DQ_TMA != 0;
  static constexpr int kDoStages = (kTmaReduce && D == 128) ? 1 : 2;
  static constexpr int kBoxD = D == 128 ? 32 : 64;                     // staging tile: 32 q x kBoxD
  static constexpr int kStageFloats = kTmaReduce ? 32 * kBoxD : 4;
};

// kDoSt: dO stages (the split mode's dK/dV kernel has no dQ staging and spends it on a second
// dO stage)
template <int D, int kDoSt = BCfg<D>::kDoStages, int kStageFl = BCfg<D>::kStageFloats>
struct alignas(1024) BSmem {
  uint8_t k[BCfg<D>::kTileBytes];
  uint8_t v[BCfg<D>::kTileBytes];
  uint8_t q[2][BCfg<D>::kTileBytes];
  uint8_t dO[kDoSt][BCfg<D>::kTileBytes];
  uint8_t ds[kTile * kTile * 2];  // dS^T [kv][q], SW128, two 64-wide q chunks
  float lse2[2][kTile];
  float delta[2][kTile];  // Δ rides with the q stage (q_full), so dO frees after dV alone
  float dq_stage[4][2][kStageFl];  // per reduction warp, double-buffered
  uint64_t k_full, v_full, k_free, v_free;
  uint64_t q_full[2], q_free[2];
  uint64_t do_full[kDoSt], do_free[kDoSt];
  uint64_t s_full, p_full, dp_full, ds_full, ds_free, dq_full, dq_empty, dkdv_full, dkdv_free;
  uint64_t item_full[2], item_empty[2];
  int32_t uitem[2];
  uint32_t tmem_base;
};

struct KvItem {
  int kb, kh, c;
};
__device__ __forceinline__ KvItem decode_kv_item(const BwdParams& p, int item) {
  // kv blocks of one (kv batch, kv head) are consecutive items: the CTAs working at the same
  // time share their q-side Q/dO tiles through L2 instead of each missing to HBM
  const int c = item % p.cols, rem = item / p.cols;
  return KvItem{rem / p.Hkv, rem % p.Hkv, c};
}

// The q blocks an item visits: for each query batch of the kv batch (kv-batch broadcast,
// engine.cpp:326-328) and each q head of the group (:330-331), the partial then the full
// q-side list of kv block c. Every role walks this sequence identically.
struct TaskIter {
  const BwdParams* p;
  int c, b, b_end, g, kh, phase, i, n;
  long long slot;
  __device__ void init(const BwdParams& pp, const KvItem& it) {
    p = &pp;
    c = it.c;
    kh = it.kh;
    b = pp.Bkv == 1 ? 0 : it.kb;
    b_end = pp.Bkv == 1 ? pp.B : it.kb + 1;
    g = 0;
    phase = 0;
    i = 0;
    load();
  }
  __device__ void load() {
    const int h = kh * p->G + g;
    const int mb = p->bm_b == 1 ? 0 : b, mh = p->bm_h == 1 ? 0 : h;
    slot = (static_cast<long long>(mb) * p->bm_h + mh) * p->cols + c;
    n = phase == 0 ? __ldg(p->q_num + slot) : __ldg(p->fq_num + slot);
  }
  // advance to the next task; false when exhausted
  __device__ bool next(int& ob, int& oh, int& orow, bool& ofull) {
    while (i >= n) {
      i = 0;
      if (phase == 0) {
        phase = 1;
      } else {
        phase = 0;
        if (++g == p->G) {
          g = 0;
          if (++b >= b_end) return false;
        }
      }
      load();
    }
    ob = b;
    oh = kh * p->G + g;
    ofull = phase == 1;
    orow = phase == 0 ? __ldg(p->q_idx + slot * p->rows + i) : __ldg(p->fq_idx + slot * p->rows + i);
    ++i;
    return true;
  }
};

__device__ __forceinline__ int count_tasks(const BwdParams& p, const KvItem& it) {
  int total = 0;
  const int b0 = p.Bkv == 1 ? 0 : it.kb, b1 = p.Bkv == 1 ? p.B : it.kb + 1;
  for (int b = b0; b < b1; ++b)
    for (int g = 0; g < p.G; ++g) {
      const int h = it.kh * p.G + g;
      const int mb = p.bm_b == 1 ? 0 : b, mh = p.bm_h == 1 ? 0 : h;
      const long long slot = (static_cast<long long>(mb) * p.bm_h + mh) * p.cols + it.c;
      total += __ldg(p.q_num + slot) + __ldg(p.fq_num + slot);
    }
  return total;
}

// kMode: kModeFused (dQ reduce-added by the reduction warps), kModeNoDQ (dK/dV only; dQ by the
// separate pass in bwd_dq.cuh)
enum { kModeFused = 0, kModeNoDQ = 2 };
#ifndef FA_BWD_SPLIT
#define FA_BWD_SPLIT 0  // 1: the split (dK/dV kernel + dQ pass) backward by default
#endif
constexpr int kDefaultMode = FA_BWD_SPLIT ? kModeNoDQ : kModeFused;
// FA_FLAG_DETERMINISTIC: the split backward, reproducible by construction (dQ accumulates in
// TMEM in one fixed kv order; dK/dV per kv block in one fixed q order)
constexpr int kDeterministicMode = kModeNoDQ;

template <int D, class MaskT, class ScoreT, int kMode>
__global__ void __launch_bounds__(kThreads, 1)
    flex_bwd_sm100_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmDO,
                          const __grid_constant__ CUtensorMap tmDQ, const BwdParams p, MaskT mask,
                          ScoreT score) {
  using C = BCfg<D>;
  constexpr bool kNoDQ = kMode == kModeNoDQ;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // the split mode keeps no dQ staging and gives its 32 KB to a second dO stage
  constexpr int kDoSt = (kNoDQ && FA_BWD_NODQ_DO2 != 0) ? 2 : C::kDoStages;
  using Sm = BSmem<D, kDoSt, (kNoDQ && FA_BWD_NODQ_DO2 != 0) ? 4 : C::kStageFloats>;
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();  // SWIZZLE_128B operands need 1 KiB alignment

  if (threadIdx.x == 0) {
    mbar_init(&sm.k_full, 1);
    mbar_init(&sm.v_full, 1);
    mbar_init(&sm.k_free, 1);
    mbar_init(&sm.v_free, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.q_full[s], 1);
      mbar_init(&sm.q_free[s], 1);
      mbar_init(&sm.item_full[s], 1);
      mbar_init(&sm.item_empty[s], 1 + 8 + 4);
    }
    for (int s = 0; s < kDoSt; ++s) {
      mbar_init(&sm.do_full[s], 1);
      mbar_init(&sm.do_free[s], 1);  // the dV MMA commit
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.p_full, 8);
    mbar_init(&sm.dp_full, 1);
    mbar_init(&sm.ds_full, 8);
    mbar_init(&sm.ds_free, 1);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_empty, 4);
    mbar_init(&sm.dkdv_full, 1);
    mbar_init(&sm.dkdv_free, 4);
    fence_barrier_init();
  }
  if (warp == 12 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
    if constexpr (C::kTmaReduce && !kNoDQ) tma_prefetch_desc(&tmDQ);
  }
  if (warp == 13) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  constexpr uint32_t kS = 0, kDP = 128, kDV = 256, kDK = 256 + D;

  // Every role ends in its own copy of the teardown so no code is shared between
  // warpgroups with different setmaxnreg budgets (ptxas allocates per region).
#define FA_BWD_TEARDOWN()                     \
  do {                                        \
    tc_fence_before();                        \
    __syncthreads();                          \
    if (warp == 13) {                         \
      tc_fence_after();                       \
      tmem_dealloc(tmem, 512);                \
    }                                         \
    return;                                   \
  } while (0)
  if (warp >= 12) {
    reg_dealloc<FA_BWD_REG_OTHER>();
  }
  if (warp == 12) {
    if (lane == 0) {
      // ===================== TMA producer =====================
      int blk = 0;
      for (int n = 0;; ++n) {
        const int item = n == 0 ? static_cast<int>(blockIdx.x)
                                : static_cast<int>(gridDim.x) + atomicAdd(p.work_counter, 1);
        const int buf = n & 1;
        mbar_wait(&sm.item_empty[buf], ((n >> 1) & 1) ^ 1);
        sm.uitem[buf] = item < p.num_items ? item : -1;
        mbar_arrive(&sm.item_full[buf]);
        if (item >= p.num_items) break;
        const KvItem it = decode_kv_item(p, item);
        // K first (the item's first GEMM needs it), then V
        mbar_wait(&sm.k_free, (n & 1) ^ 1);
        mbar_expect_tx(&sm.k_full, C::kTileBytes);
        for (int ch = 0; ch < C::kChunks; ++ch)
          tma_load_3d(sm.k + ch * C::kChunkBytes, &tmK, &sm.k_full, ch * 64, it.c * kTile,
                      it.kb * p.Hkv + it.kh);
        TaskIter ti;
        ti.init(p, it);
        int b, h, r;
        bool full;
        bool v_loaded = false;
        // one task of lookahead: the next q block's Q / dO tiles are prefetched into L2 while
        // this one's buffers are still busy (FA_BWD_L2PF)
        int nb_ = 0, nh_ = 0, nr_ = 0;
        bool nfull_ = false;
        bool have = ti.next(nb_, nh_, nr_, nfull_);
        while (have) {
          b = nb_;
          h = nh_;
          r = nr_;
          full = nfull_;
          have = ti.next(nb_, nh_, nr_, nfull_);
          if (FA_BWD_L2PF != 0 && have) {
            for (int ch = 0; ch < C::kChunks; ++ch) {
              tma_prefetch_l2_3d(&tmQ, ch * 64, nr_ * kTile, nb_ * p.Hq + nh_);
              tma_prefetch_l2_3d(&tmDO, ch * 64, nr_ * kTile, nb_ * p.Hq + nh_);
            }
          }
          const int st = blk & 1;
          const long long row0 = static_cast<long long>(b * p.Hq + h) * p.Lq_pad + r * kTile;
          mbar_wait(&sm.q_free[st], ((blk >> 1) & 1) ^ 1);
          trace_ev(p, blk, 10);
          mbar_expect_tx(&sm.q_full[st], C::kTileBytes + 2 * kTile * 4);
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_3d(sm.q[st] + ch * C::kChunkBytes, &tmQ, &sm.q_full[st], ch * 64, r * kTile,
                        b * p.Hq + h);
          bulk_load(sm.lse2[st], p.lse2 + row0, kTile * 4, &sm.q_full[st]);
          bulk_load(sm.delta[st], p.delta + row0, kTile * 4, &sm.q_full[st]);
          if (!v_loaded) {
            mbar_wait(&sm.v_free, (n & 1) ^ 1);
            mbar_expect_tx(&sm.v_full, C::kTileBytes);
            for (int ch = 0; ch < C::kChunks; ++ch)
              tma_load_3d(sm.v + ch * C::kChunkBytes, &tmV, &sm.v_full, ch * 64, it.c * kTile,
                          it.kb * p.Hkv + it.kh);
            v_loaded = true;
          }
          const int ds_ = blk % kDoSt;
          mbar_wait(&sm.do_free[ds_], ((blk / kDoSt) & 1) ^ 1);
          trace_ev(p, blk, 11);
          mbar_expect_tx(&sm.do_full[ds_], C::kTileBytes);
          for (int ch = 0; ch < C::kChunks; ++ch)
            tma_load_3d(sm.dO[ds_] + ch * C::kChunkBytes, &tmDO, &sm.do_full[ds_], ch * 64, r * kTile,
                        b * p.Hq + h);
          ++blk;
        }
        if (!v_loaded) {  // an item with no q blocks still owns one V phase
          mbar_wait(&sm.v_free, (n & 1) ^ 1);
          mbar_arrive(&sm.v_full);
        }
      }
    }
    FA_BWD_TEARDOWN();
  } else if (warp == 13) {
    {
      // ===================== MMA issuer =====================
      // The whole warp runs the warp-uniform control flow and one elected lane issues, so
      // descriptors sit in uniform registers (a lane-0-only branch costs an ELECT/R2UR
      // waterfall loop around every tcgen05.mma).
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) umma_commit(bar);
        __syncwarp();
      };
      constexpr uint32_t idesc_ss = make_idesc_bf16(128, 128, 0, 0);   // S^T, dP^T
      constexpr uint32_t idesc_kn = make_idesc_bf16(128, D, 0, 1);     // dV (TS), dK (SS)
      constexpr uint32_t idesc_mm = make_idesc_bf16(128, D, 1, 1);     // dQ = dS K (D = 64)
      constexpr uint32_t idesc_mmT = make_idesc_bf16(D, 128, 1, 1);    // dQ^T = K^T dS^T (D = 128)
      const uint32_t k_addr = smem_u32(sm.k), v_addr = smem_u32(sm.v), ds_addr = smem_u32(sm.ds);
      // issue + commit in one elected region
      auto mma_kmajor = [&](uint32_t d_col, uint32_t a_addr, uint32_t b_addr, uint64_t* bar) {
        if (elect_one()) {
          const uint64_t a0 = make_sdesc_sw128(a_addr, 16, 1024);
          const uint64_t b0 = make_sdesc_sw128(b_addr, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * C::kChunkBytes + (kk & 3) * 32) >> 4;
            umma_ss(tm + d_col, a0 + off, b0 + off, idesc_ss, kk > 0 ? 1u : 0u);
          }
          umma_commit(bar);
        }
        __syncwarp();
      };
      auto issue_s = [&](int b) {  // S^T(b) = K Q(b)^T
        const int st = b & 1;
        trace_ev(p, b, 12);
        mbar_wait(&sm.q_full[st], (b >> 1) & 1);
        trace_ev(p, b, 13);
        tc_fence_after();
        mma_kmajor(kS, k_addr, smem_u32(sm.q[st]), &sm.s_full);
        trace_ev(p, b, 4);
      };
      auto issue_dp = [&](int b) {  // dP^T(b) = V dO(b)^T, after dQ(b-1) left TMEM
        const int ds_ = b % kDoSt;
        trace_ev(p, b, 14);
        mbar_wait(&sm.do_full[ds_], (b / kDoSt) & 1);
        trace_ev(p, b, 15);
        if constexpr (!kNoDQ) mbar_wait(&sm.dq_empty, (b & 1) ^ 1);  // dQ^T(b-1) left TMEM
        trace_ev(p, b, 16);
        tc_fence_after();
        mma_kmajor(kDP, v_addr, smem_u32(sm.dO[ds_]), &sm.dp_full);
        trace_ev(p, b, 6);
      };
      auto issue_dv = [&](int b, bool acc) {  // dV += P^T(b) dO(b)   (TS)
        const int ds_ = b % kDoSt;
        trace_ev(p, b, 17);
        mbar_wait(&sm.p_full, b & 1);
        trace_ev(p, b, 18);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t b0 = make_sdesc_sw128(smem_u32(sm.dO[ds_]), C::kChunkBytes, 1024);
#pragma unroll
          for (int kk = 0; kk < kTile / 16; ++kk) {
            const uint32_t a_col = kS + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8);
            umma_ts(tm + kDV, tm + a_col, b0 + kk * (2048 >> 4), idesc_kn, (acc || kk > 0) ? 1u : 0u);
          }
          umma_commit(&sm.do_free[ds_]);
        }
        __syncwarp();
      };
      auto issue_dq_impl = [&](int b, bool wait) {  // dQ(b) over the dP columns (dS^T(b) read from smem)
        if constexpr (kNoDQ) {  // no dQ here: dK(b) only needs dS^T(b) in smem
          if (wait) {
            mbar_wait(&sm.ds_full, b & 1);
            tc_fence_after();
          }
          return;
        }
        if constexpr (kDkSS) {
          if (wait) {
            mbar_wait(&sm.ds_full, b & 1);
            tc_fence_after();
          }
          trace_ev(p, b, 5);
        }
        trace_ev(p, b, 19);
        if (elect_one()) {
          const uint64_t k0 = make_sdesc_sw128(k_addr, C::kChunkBytes, 1024);
          const uint64_t s0 = make_sdesc_sw128(ds_addr, kTile * 128, 1024);
          if constexpr (D == 128) {
            // dQ^T = K^T dS^T (M = head dim, N = q): the reduction warps own one head-dim
            // index per lane and add whole 128-byte lines
#pragma unroll
            for (int kk = 0; kk < kTile / 16; ++kk)
              umma_ss(tm + kDP, k0 + kk * (2048 >> 4), s0 + kk * (2048 >> 4), idesc_mmT, kk > 0 ? 1u : 0u);
          } else {
#pragma unroll
            for (int kk = 0; kk < kTile / 16; ++kk)
              umma_ss(tm + kDP, s0 + kk * (2048 >> 4), k0 + kk * (2048 >> 4), idesc_mm, kk > 0 ? 1u : 0u);
          }
          umma_commit(&sm.dq_full);
          if constexpr (!kDkSS) umma_commit(&sm.ds_free);
        }
        __syncwarp();
      };
      auto issue_dq = [&](int b) { issue_dq_impl(b, true); };
      auto issue_dq_nowait = [&](int b) { issue_dq_impl(b, false); };
      auto issue_dk = [&](int b, bool acc) {  // dK += dS^T(b) Q(b)
        if constexpr (kDkSS) {
          // SS, dS^T from the smem buffer (K-major, the layout of a TMA tile): dK is off the
          // B -> dQ -> drain -> dP chain and B stores dS^T to smem only
          if (elect_one()) {
            const uint64_t a0 = make_sdesc_sw128(ds_addr, 16, 1024);
            const uint64_t b0 = make_sdesc_sw128(smem_u32(sm.q[b & 1]), C::kChunkBytes, 1024);
#pragma unroll
            for (int kk = 0; kk < kTile / 16; ++kk) {
              const uint32_t aoff = ((kk >> 2) * (kTile * 128) + (kk & 3) * 32) >> 4;
              umma_ss(tm + kDK, a0 + aoff, b0 + kk * (2048 >> 4), idesc_kn, (acc || kk > 0) ? 1u : 0u);
            }
            umma_commit(&sm.q_free[b & 1]);
            umma_commit(&sm.ds_free);
          }
          __syncwarp();
          trace_ev(p, b, 20);
          return;
        }
        mbar_wait(&sm.ds_full, b & 1);
        tc_fence_after();
        trace_ev(p, b, 5);
        if (elect_one()) {
          const uint64_t b0 = make_sdesc_sw128(smem_u32(sm.q[b & 1]), C::kChunkBytes, 1024);
#pragma unroll
          for (int kk = 0; kk < kTile / 16; ++kk) {
            const uint32_t a_col = kDP + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8);
            umma_ts(tm + kDK, tm + a_col, b0 + kk * (2048 >> 4), idesc_kn, (acc || kk > 0) ? 1u : 0u);
          }
          umma_commit(&sm.q_free[b & 1]);
        }
        __syncwarp();
        trace_ev(p, b, 20);
      };
      int blk = 0;
      for (int n = 0;; ++n) {
        const int buf = n & 1;
        mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
        const int item = sm.uitem[buf];
        if (lane == 0) mbar_arrive(&sm.item_empty[buf]);
        if (item < 0) break;
        const KvItem it = decode_kv_item(p, item);
        const int T = count_tasks(p, it);
        mbar_wait(&sm.k_full, n & 1);
        if (T == 0) {
          mbar_wait(&sm.dkdv_free, (n & 1) ^ 1);
          mbar_wait(&sm.v_full, n & 1);
          commit(&sm.dkdv_full);
          commit(&sm.k_free);
          commit(&sm.v_free);
          continue;
        }
        issue_s(blk);
        mbar_wait(&sm.v_full, n & 1);
        issue_dp(blk);
        mbar_wait(&sm.dkdv_free, (n & 1) ^ 1);  // the previous item's dK/dV were read out
        issue_dv(blk, false);
        for (int t = 0; t < T; ++t) {
          const int b = blk + t;
          if (t + 1 < T) issue_s(b + 1);
          if constexpr (kDkSS && FA_BWD_DK_FIRST != 0) {
            // dK(b) first: Q(b)'s buffer frees a GEMM earlier for the load of Q(b+2)
            mbar_wait(&sm.ds_full, b & 1);
            tc_fence_after();
            issue_dk(b, t > 0);
            issue_dq_nowait(b);
          } else if constexpr (kDkSS) {
            issue_dq(b);
            issue_dk(b, t > 0);
          } else {
            issue_dk(b, t > 0);
            issue_dq(b);
          }
          if (t + 1 == T) commit(&sm.k_free);  // K's last reader was dQ(T-1)
          if (t + 1 < T) {
            issue_dp(b + 1);
            if (t + 2 == T) commit(&sm.v_free);  // V's last reader was dP(T-1)
            issue_dv(b + 1, true);
          } else if (T == 1) {
            commit(&sm.v_free);
          }
        }
        commit(&sm.dkdv_full);
        blk += T;
      }
    }
    FA_BWD_TEARDOWN();
  } else if (warp < 8) {
    // ===================== compute warpgroups: P^T, dS^T =====================
    reg_alloc<144>();
    const int wg = warp >> 2;          // which 64 q columns
    const int wq = warp & 3;           // TMEM lane quarter
    const int j = wq * 32 + lane;      // kv row within the block
    const uint32_t tm = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    int blk = 0;
    for (int n = 0;; ++n) {
      const int buf = n & 1;
      mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
      const int item = sm.uitem[buf];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.item_empty[buf]);
      if (item < 0) break;
      const KvItem it = decode_kv_item(p, item);
      const int kv = it.c * kTile + j;
      const bool kv_in = kv < p.Lkv;
      TaskIter ti;
      ti.init(p, it);
      int b, h, r;
      bool full;
      while (ti.next(b, h, r, full)) {
        const int qst = blk & 1;
        const int q0 = r * kTile + wg * 64;
        // ---------------- phase A: P^T ----------------
        // The preprocess stored per q column  cterm = log2(scale) - lse·log2e  (+ the q part of
        // ALiBi), so P·scale = exp2(s·c + cterm [+ kv part of ALiBi]) is one FFMA + one MUFU.
        // P·scale (bf16) feeds dV (rescaled by 1/scale in the epilogue) and, times mod'(s), dS.
        mbar_wait(&sm.s_full, blk & 1);
        mbar_wait(&sm.q_full[qst], (blk >> 1) & 1);  // cterm of this q block
        tc_fence_after();
        if (threadIdx.x == 0) trace_ev(p, blk, 0);
        float pg[64];  // P·scale·mod'(s), kept in fp32 for phase B
        {
          uint32_t sr[64];
          tmem_ld32(tm + kS + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
          // mask bits for this kv row over the 64 q columns (bounds folded in)
          uint32_t bits0 = 0u, bits1 = 0u;
          if (!full && kv_in) {
            bits0 = mask.bits32_q(b, h, q0, kv, p.Lq);
            bits1 = mask.bits32_q(b, h, q0 + 32, kv, p.Lq);
          }
          const float4* ct4 = reinterpret_cast<const float4*>(sm.lse2[qst] + wg * 64);
          const auto colc = score.col(b, h, q0, kv, p.scale);
          float rowc = 0.f;  // ALiBi: slope·log2e·(block q start + q_offset - kv)
          if constexpr (ScoreT::kKind == 1)
            rowc = colc.step * static_cast<float>(r * kTile + score.p.q_offset - kv);
          tmem_wait_ld();
          // the second half of S^T loads while the first half is exponentiated
          tmem_ld32(tm + kS + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
          uint32_t pp[32];
          // full blocks skip mask_mod entirely (no per-score select)
          auto body = [&](auto masked) {
#pragma unroll
            for (int i4 = 0; i4 < 16; ++i4) {
              if (i4 == 8) tmem_wait_ld();
              const float4 c4 = ct4[i4];
              const float cv[4] = {c4.x, c4.y, c4.z, c4.w};
              float pv[4], gv[4];
              float xp[4];  // plain / ALiBi: the exponents of the 4 scores as two FFMA2 pairs
              if constexpr (FA_BWD_PAIRED != 0 && (ScoreT::kKind == 0 || ScoreT::kKind == 1)) {
#pragma unroll
                for (int e = 0; e < 4; e += 2) {
                  float2 add = make_float2(cv[e], cv[e + 1]);
                  if constexpr (ScoreT::kKind == 1) add = __fadd2_rn(add, make_float2(rowc, rowc));
                  const float2 xx = __ffma2_rn(make_float2(__uint_as_float(sr[i4 * 4 + e]), __uint_as_float(sr[i4 * 4 + e + 1])),
                                               make_float2(colc.c, colc.c), add);
                  xp[e] = xx.x;
                  xp[e + 1] = xx.y;
                }
              }
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int ii = i4 * 4 + e;
                const float sv = __uint_as_float(sr[ii]);
                float x;
                if constexpr (FA_BWD_PAIRED != 0 && (ScoreT::kKind == 0 || ScoreT::kKind == 1)) {
                  x = xp[e];
                } else if constexpr (ScoreT::kKind == 0) {
                  x = fmaf(sv, colc.c, cv[e]);
                } else if constexpr (ScoreT::kKind == 1) {
                  x = fmaf(sv, colc.c, cv[e] + rowc);
                } else {
                  const auto cc = colc.shifted(ii & ~31);
                  float g;
                  const float t = cc.log2_grad(sv, ii & 31, g);  // outer·tanh(u), g = 1 - tanh²
                  x = t + cv[e];
                  gv[e] = g;
                }
                if constexpr (decltype(masked)::value) {
                  const uint32_t bits = ii < 32 ? bits0 : bits1;
                  pv[e] = ((bits >> (ii & 31)) & 1u) ? ex2(x) : 0.f;
                } else {
                  pv[e] = ex2(x);
                }
              }
              pp[2 * i4] = pack_bf16(pv[0], pv[1]);
              pp[2 * i4 + 1] = pack_bf16(pv[2], pv[3]);
#pragma unroll
              for (int e = 0; e < 4; ++e) pg[i4 * 4 + e] = ScoreT::kUnitGrad ? pv[e] : pv[e] * gv[e];
            }
          };
          if (full) body(std::false_type{});
          else body(std::true_type{});
          tmem_st32(tm + kS + wg * 64, pp);  // P^T over S^T columns already read
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.p_full);
        if (threadIdx.x == 0) trace_ev(p, blk, 1);
        // ---------------- phase B: dS^T ----------------
        mbar_wait(&sm.dp_full, blk & 1);
        tc_fence_after();
        if (threadIdx.x == 0) trace_ev(p, blk, 2);
        {
          const float4* dlt4 = reinterpret_cast<const float4*>(sm.delta[qst] + wg * 64);
          // the previous block's dQ must have read the dS^T smem buffer
          mbar_wait(&sm.ds_free, (blk & 1) ^ 1);
          uint8_t* ds_row = sm.ds + wg * (kTile * 128) + j * 128;
          uint32_t dpr[2][32];
          tmem_ld32(tm + kDP + wg * 64, dpr[0]);
          tmem_wait_ld();
          tmem_ld32(tm + kDP + wg * 64 + 32, dpr[1]);  // overlaps the first half's math
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            if (hh == 1) tmem_wait_ld();
            uint32_t dsp[16];
#pragma unroll
            for (int i4 = 0; i4 < 8; ++i4) {
              const float4 d4 = dlt4[hh * 8 + i4];
              const float dv4[4] = {d4.x, d4.y, d4.z, d4.w};
              float a[4];
#pragma unroll
              for (int e = 0; e < 4; ++e)
                a[e] = pg[hh * 32 + i4 * 4 + e] * (__uint_as_float(dpr[hh][i4 * 4 + e]) - dv4[e]);
              dsp[2 * i4] = pack_bf16(a[0], a[1]);
              dsp[2 * i4 + 1] = pack_bf16(a[2], a[3]);
            }
            // dS^T (bf16) over dP^T columns already read: the A operand of dK (TS)
            if constexpr (!kDkSS) tmem_st16(tm + kDP + wg * 64 + hh * 16, dsp);
            // dS^T row j (the MN-major operand of dQ): 16-byte units 4hh..4hh+3 of this
            // warpgroup's 64-wide q chunk, 128-byte swizzle
#pragma unroll
            for (int u = 0; u < 4; ++u)
              *reinterpret_cast<uint4*>(ds_row + (((hh * 4 + u) ^ (j & 7)) << 4)) =
                  make_uint4(dsp[4 * u], dsp[4 * u + 1], dsp[4 * u + 2], dsp[4 * u + 3]);
          }
        }
        fence_proxy_async();
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.ds_full);
        if (threadIdx.x == 0) trace_ev(p, blk, 3);
        ++blk;
      }
    }
    FA_BWD_TEARDOWN();
  } else if (warp < 12) {
    // ===================== dQ reduction + dK/dV epilogue warpgroup =====================
    reg_alloc<FA_BWD_REG_REDUCE>();
    const int wq = warp & 3;
    const uint32_t tm = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    int blk = 0, stage_it = 0;
    for (int n = 0;; ++n) {
      const int buf = n & 1;
      mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
      const int item = sm.uitem[buf];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.item_empty[buf]);
      if (item < 0) break;
      const KvItem it = decode_kv_item(p, item);
      TaskIter ti;
      ti.init(p, it);
      int T = 0, b, h, r;
      bool full;
      while (ti.next(b, h, r, full)) {
        if constexpr (kNoDQ) {  // the epilogue only needs the task count
          ++blk;
          ++T;
          continue;
        }
        mbar_wait(&sm.dq_full, blk & 1);
        tc_fence_after();
        if (threadIdx.x == 256) trace_ev(p, blk, 7);
        if constexpr (D == 128) {
          // dQ^T: lane = head-dim index d = 32 wq + lane, columns = the block's 128 q rows
          uint32_t a[128];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            tmem_ld32(tm + kDP + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&a[cc * 32]));
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.dq_empty);
          if (threadIdx.x == 256) trace_ev(p, blk, 8);
          if constexpr (C::kTmaReduce) {
            // four 32 (q) x 32 (d) fp32 tiles per warp: st.shared rows of 128 B (lane = d),
            // then one TMA reduce-add each (rows past Q_LEN are clipped by the tensor map)
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4, ++stage_it) {
              float* stg = sm.dq_stage[wq][stage_it & 1];
              if (lane == 0) bulk_wait_group_read<1>();  // the reduce that last read this buffer
              __syncwarp();
#pragma unroll
              for (int qq = 0; qq < 32; ++qq) stg[qq * 32 + lane] = __uint_as_float(a[c4 * 32 + qq]);
              fence_proxy_async();
              __syncwarp();
              if (lane == 0) {
                tma_reduce_add_3d(&tmDQ, stg, wq * 32, r * kTile + c4 * 32, b * p.Hq + h);
                bulk_commit_group();
              }
            }
          } else {
          // per q row the warp's 32 lanes add 32 consecutive floats: one 128-byte line per red
          const int d = wq * 32 + lane;
          const int nq = min(kTile, p.Lq - r * kTile);
          float* base = p.dq_acc + (static_cast<long long>(b * p.Hq + h) * p.Lq + r * kTile) * D + d;
          if (nq == kTile) {
#pragma unroll
            for (int qq = 0; qq < kTile; ++qq) red_add_f32(base + qq * D, __uint_as_float(a[qq]));
          } else {
#pragma unroll
            for (int qq = 0; qq < kTile; ++qq)
              if (qq < nq) red_add_f32(base + qq * D, __uint_as_float(a[qq]));
          }
          }
        } else {
          // dQ: lane = q row 32 wq + lane, columns = the D head-dim values
          uint32_t a[D];
#pragma unroll
          for (int cc = 0; cc < D / 32; ++cc)
            tmem_ld32(tm + kDP + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&a[cc * 32]));
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.dq_empty);
          if constexpr (C::kTmaReduce) {
            // one 32 (q) x D fp32 tile per warp (row per lane; bank conflicts accepted at D=64)
            float* stg = sm.dq_stage[wq][stage_it & 1];
            if (lane == 0) bulk_wait_group_read<1>();
            __syncwarp();
#pragma unroll
            for (int u = 0; u < D / 4; ++u) {
              float4 w4;
              w4.x = __uint_as_float(a[4 * u]);
              w4.y = __uint_as_float(a[4 * u + 1]);
              w4.z = __uint_as_float(a[4 * u + 2]);
              w4.w = __uint_as_float(a[4 * u + 3]);
              *reinterpret_cast<float4*>(stg + lane * D + 4 * u) = w4;
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              tma_reduce_add_3d(&tmDQ, stg, 0, r * kTile + wq * 32, b * p.Hq + h);
              bulk_commit_group();
            }
            ++stage_it;
          } else {
            const int qrow = r * kTile + wq * 32 + lane;
            if (qrow < p.Lq) {
              float* dst = p.dq_acc + (static_cast<long long>(b * p.Hq + h) * p.Lq + qrow) * D;
#pragma unroll
              for (int v4 = 0; v4 < D / 4; ++v4)
                red_add_v4(dst + v4 * 4, __uint_as_float(a[4 * v4]), __uint_as_float(a[4 * v4 + 1]),
                           __uint_as_float(a[4 * v4 + 2]), __uint_as_float(a[4 * v4 + 3]));
            }
          }
        }
        if (threadIdx.x == 256) trace_ev(p, blk, 9);
        ++blk;
        ++T;
      }
      // ---- epilogue: dK, dV rows (lanes = kv rows) ----
      mbar_wait(&sm.dkdv_full, n & 1);
      tc_fence_after();
      const int kv = it.c * kTile + wq * 32 + lane;
      const bool kv_ok = kv < p.Lkv;
      const long long orow = (static_cast<long long>(it.kb) * p.Hkv + it.kh) * p.Lkv + kv;
#pragma unroll 1
      for (int which = 0; which < 2; ++which) {
        __nv_bfloat16* dst = (which == 0 ? p.dk : p.dv) + orow * D;
        const uint32_t col = which == 0 ? kDK : kDV;
        const float mul = which == 0 ? 1.f : 1.f / p.scale;  // dV accumulated (P·scale)^T dO
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t v[32];
          if (T > 0) {  // warp-collective loads: every lane loads, rows >= KV_LEN do not store
            tmem_ld32(tm + col + cc * 32, v);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0u;
          }
          if (kv_ok) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              d4[q4] = make_uint4(pack_bf16(__uint_as_float(v[8 * q4]) * mul, __uint_as_float(v[8 * q4 + 1]) * mul),
                                  pack_bf16(__uint_as_float(v[8 * q4 + 2]) * mul, __uint_as_float(v[8 * q4 + 3]) * mul),
                                  pack_bf16(__uint_as_float(v[8 * q4 + 4]) * mul, __uint_as_float(v[8 * q4 + 5]) * mul),
                                  pack_bf16(__uint_as_float(v[8 * q4 + 6]) * mul, __uint_as_float(v[8 * q4 + 7]) * mul));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.dkdv_free);
    }
    if constexpr (C::kTmaReduce && !kNoDQ) {
      if (lane == 0) bulk_wait_group<0>();  // every dQ reduce-add has landed before exit
      __syncwarp();
    }
    FA_BWD_TEARDOWN();
  } else {
    FA_BWD_TEARDOWN();  // warps 14-15: idle
  }
#undef FA_BWD_TEARDOWN
}

// Per q row: Δ = Σ dO·O, and the column term of the compute warps' exponent,
//   cterm = log2(scale) - lse·log2e  (+ slope·log2e·(q mod 128) for ALiBi, whose kv and
//   block parts the compute warps add), so that exp2(s·c + cterm) = P·scale.
// Fully masked rows (lse = -inf) and the padding to whole q blocks get cterm = -inf (P = 0).
template <class ScoreT>
__global__ void __launch_bounds__(256) bwd_preprocess_kernel(
    const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, int BH, int Hq, int Lq, int Lq_pad, int D, float scale, ScoreT score,
    float* __restrict__ cterm, float* __restrict__ delta, float* __restrict__ dq_acc,
    int* __restrict__ dout_bad) {
  // 8 lanes per row: each lane reads D/8 contiguous bf16 of O and dO with 16-byte loads and
  // zeroes its D/8 floats of the dQ accumulator (the memset of the fp32 workspace, fused)
  const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 3;
  const int sub = threadIdx.x & 7;
  if (row >= (long long)BH * Lq_pad) return;
  const int q = (int)(row % Lq_pad);
  const long long bh = row / Lq_pad;
  if (q >= Lq) {
    if (sub == 0) {
      cterm[row] = -INFINITY;
      delta[row] = 0.f;
    }
    return;
  }
  const long long src = (bh * Lq + q) * D + sub * (D / 8);
  const uint4* o4 = reinterpret_cast<const uint4*>(o + src);
  const uint4* d4 = reinterpret_cast<const uint4*>(dout + src);
  float4* z4 = reinterpret_cast<float4*>(dq_acc + src);
  float a = 0.f;
  bool bad = false;
  for (int v = 0; v < D / 64; ++v) {
    const uint4 x = __ldg(o4 + v), y = __ldg(d4 + v);
    if (dout_bad != nullptr) {  // d_out finiteness (engine.cpp:196), folded into this read
      const uint32_t w[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t t = w[e] & 0x7f807f80u;
        bad |= (t & 0xffffu) == 0x7f80u || (t >> 16) == 0x7f80u;
      }
    }
    const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* yp = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      a = fmaf(__low2float(xp[e]), __low2float(yp[e]), a);
      a = fmaf(__high2float(xp[e]), __high2float(yp[e]), a);
    }
    if (dq_acc != nullptr) {  // the fused dQ reduce-adds into it
      z4[2 * v] = make_float4(0.f, 0.f, 0.f, 0.f);
      z4[2 * v + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (bad) atomicOr(dout_bad, 1);
  a += __shfl_xor_sync(0xffffffffu, a, 4);
  a += __shfl_xor_sync(0xffffffffu, a, 2);
  a += __shfl_xor_sync(0xffffffffu, a, 1);
  if (sub == 0) {
    const float l = lse[bh * Lq + q];
    float ct = l == -INFINITY ? -INFINITY : __log2f(scale) - l * kLog2e;
    if constexpr (ScoreT::kKind == 1)
      ct += __ldg(score.p.slopes + (int)(bh % Hq)) * kLog2e * static_cast<float>(q & (kTile - 1));
    cterm[row] = ct;
    delta[row] = a;
  }
}

__global__ void dq_convert_kernel(const float4* __restrict__ acc, uint4* __restrict__ dq, long long n8) {
  // 8 floats -> 8 bf16 per step: two 16-byte loads, one 16-byte store
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const float4 a = acc[2 * i], b = acc[2 * i + 1];
    dq[i] = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
  }
}

template <int D, class MaskT, class ScoreT, int kMode>
fa_status run(const AttnGeom& g, const void* q, const void* k, const void* v, const void* o,
              const float* lse, const void* dout, void* dq, void* dk, void* dv, const BmView& bm,
              const BmView& bmt, MaskT mask, ScoreT score, void* workspace, const BwdOptions& opt,
              cudaStream_t st) {
  const int Lq_pad = (g.Lq + kTile - 1) / kTile * kTile;
  const long long rows = (long long)g.B * g.Hq * g.Lq;
  const long long prow = (long long)g.B * g.Hq * Lq_pad;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* ws = static_cast<char*>(workspace);
  float* dq_acc = reinterpret_cast<float*>(ws);
  float* lse2 = reinterpret_cast<float*>(ws + al(rows * D * 4));
  float* delta = reinterpret_cast<float*>(ws + al(rows * D * 4) + al(prow * 4));
  constexpr bool kNoDQ = kMode == kModeNoDQ;
  if (kNoDQ) dq_acc = nullptr;  // dQ comes from its own pass: nothing to zero or convert
  if (opt.events[0]) FA_CHECK_CUDA(cudaEventRecord(opt.events[0], st));
  // preprocess: Δ, cterm, and the zeroing of the fp32 dQ accumulator (8 threads per row)
  bwd_preprocess_kernel<ScoreT><<<(unsigned)((prow + 31) / 32), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), lse,
      g.B * g.Hq, g.Hq, g.Lq, Lq_pad, D, g.scale, score, lse2, delta, dq_acc, opt.dout_nonfinite);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());

  CUtensorMap mq, mk, mv, mdo, mdq{};
  CUresult cr;
  if ((cr = encode_tile_map(&mq, q, g.B * g.Hq, g.Lq, D)) != CUDA_SUCCESS ||
      (cr = encode_tile_map(&mk, k, g.Bkv * g.Hkv, g.Lkv, D)) != CUDA_SUCCESS ||
      (cr = encode_tile_map(&mv, v, g.Bkv * g.Hkv, g.Lkv, D)) != CUDA_SUCCESS ||
      (cr = encode_tile_map(&mdo, dout, g.B * g.Hq, g.Lq, D)) != CUDA_SUCCESS ||
      (!kNoDQ && (cr = encode_f32_map(&mdq, dq_acc, g.B * g.Hq, g.Lq, D, BCfg<D>::kBoxD, 32)) != CUDA_SUCCESS))
    return set_error(FA_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string((int)cr) + ")");
  BwdParams p{};
  p.B = g.B; p.Hq = g.Hq; p.Hkv = g.Hkv; p.Bkv = g.Bkv; p.Lq = g.Lq; p.Lkv = g.Lkv; p.G = g.G;
  p.Lq_pad = Lq_pad;
  p.bm_b = g.bm_b; p.bm_h = g.bm_h; p.rows = g.rows; p.cols = g.cols;
  p.q_num = bmt.kv_num; p.q_idx = bmt.kv_idx; p.fq_num = bmt.full_num; p.fq_idx = bmt.full_idx;
  p.kv_num = bm.kv_num; p.kv_idx = bm.kv_idx; p.fkv_num = bm.full_num; p.fkv_idx = bm.full_idx;
  p.lse2 = lse2; p.delta = delta; p.dq_acc = dq_acc;
  p.dk = static_cast<__nv_bfloat16*>(dk);
  p.dv = static_cast<__nv_bfloat16*>(dv);
  p.scale = g.scale;
  p.num_items = g.Bkv * g.Hkv * g.cols;
  p.work_counter = scheduler_counter(kSlotBwdSched, st);
  FA_REQUIRE(p.work_counter != nullptr, FA_CUDA_ERROR, "backward: cannot allocate the scheduler counter");
  FA_CHECK_CUDA(cudaMemsetAsync(p.work_counter, 0, sizeof(int), st));
  long long* trace = nullptr;
  if (FA_BWD_TRACE_BUILD != 0 && getenv("FA_BWD_TRACE") != nullptr) {
    FA_CHECK_CUDA(cudaMalloc(&trace, sizeof(long long) * kTraceTasks * kTraceEv));
    FA_CHECK_CUDA(cudaMemsetAsync(trace, 0, sizeof(long long) * kTraceTasks * kTraceEv, st));
  }
  p.trace = trace;
  constexpr bool kNoDQ2 = kMode == kModeNoDQ && FA_BWD_NODQ_DO2 != 0;
  const size_t smem = sizeof(BSmem<D, kNoDQ2 ? 2 : BCfg<D>::kDoStages, kNoDQ2 ? 4 : BCfg<D>::kStageFloats>);
  auto kern = flex_bwd_sm100_kernel<D, MaskT, ScoreT, kMode>;
  FA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = p.num_items < num_sms() ? p.num_items : num_sms();
  if (opt.events[1]) FA_CHECK_CUDA(cudaEventRecord(opt.events[1], st));
  if (grid > 0) {
    kern<<<grid, kThreads, smem, st>>>(mq, mk, mv, mdo, mdq, p, mask, score);
    count_launch();
    FA_CHECK_CUDA(cudaGetLastError());
  }
  if (trace != nullptr) {  // debug: per-phase cycle deltas of CTA 0, averaged over its blocks
    static long long h[kTraceTasks * kTraceEv];
    FA_CHECK_CUDA(cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st));
    FA_CHECK_CUDA(cudaStreamSynchronize(st));
    cudaFree(trace);
    // events: 0 A start, 1 A end, 2 B start, 3 B end (compute) | 4 S issued, 5 ds_full seen
    // (dQ issue), 6 dP issued (MMA) | 7 dq_full seen, 8 dq_empty arrived, 9 reduces issued
    double acc[12] = {0};
    int cnt = 0;
    for (int t = 1; t + 1 < kTraceTasks; ++t) {
      const long long* e = h + t * kTraceEv;
      const long long* en = h + (t + 1) * kTraceEv;
      if (e[0] == 0 || en[0] == 0 || e[9] == 0 || en[6] == 0) break;
      acc[0] += e[1] - e[0];    // phase A
      acc[1] += e[2] - e[1];    // wait for dP
      acc[2] += e[3] - e[2];    // phase B
      acc[3] += en[0] - e[3];   // B end -> next A start
      acc[4] += e[5] - e[3];    // ds_full -> MMA sees it
      acc[5] += e[7] - e[5];    // dQ issue -> reduce sees dq_full
      acc[6] += e[8] - e[7];    // dQ TMEM drain
      acc[7] += en[6] - e[8];   // dq_empty -> next dP issued
      acc[8] += en[2] - en[6];  // dP issued -> next B start
      acc[9] += en[0] - e[0];   // period
      acc[10] += en[4] - en[10];  // Q load issued -> S issued (includes the q_full wait)
      acc[11] += en[6] - en[11];  // dO load issued -> dP issued
      ++cnt;
    }
    if (getenv("FA_BWD_TRACE")[0] == '2') {
      static const char* names[24] = {"A0", "A1", "B0", "B1", "Sdone", "dQiss", "dPiss", "rdq", "rempty", "rred",
                                      "ldQ", "ldO", "S_in", "S_q", "dP_in", "dP_do", "dP_em", "dV_in", "dV_p",
                                      "dQ_in", "dKiss", "", "", ""};
      const long long t0 = h[10 * kTraceEv + 0];
      for (int t = 10; t < 14; ++t) {
        fprintf(stderr, "[bwd trace] block %d:", t);
        for (int e = 0; e < 21; ++e)
          if (h[t * kTraceEv + e] != 0) fprintf(stderr, " %s=%lld", names[e], h[t * kTraceEv + e] - t0);
        fprintf(stderr, "\n");
      }
    }
    if (cnt > 0)
      fprintf(stderr,
              "[bwd trace] blocks=%d cycles: A %.0f | wait dP %.0f | B %.0f | B->nextA %.0f | ds->mma %.0f | "
              "dQ mma %.0f | dQ drain %.0f | empty->dP %.0f | dP->B %.0f | period %.0f | Qld->S %.0f | dOld->dP %.0f\n",
              cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt,
              acc[6] / cnt, acc[7] / cnt, acc[8] / cnt, acc[9] / cnt, acc[10] / cnt, acc[11] / cnt);
  }
  if (opt.events[2]) FA_CHECK_CUDA(cudaEventRecord(opt.events[2], st));
  if constexpr (kNoDQ) {
    // the dQ pass: dQ accumulated in TMEM per q tile, written as bf16
    const fa_status s = bdq::run<D>(g, q, k, v, dout, lse, delta, dq, bm, mask, score, st);
    if (s != FA_OK) return s;
    if (opt.events[3]) FA_CHECK_CUDA(cudaEventRecord(opt.events[3], st));
    return FA_OK;
  }
  const long long n8 = rows * D / 8;
  dq_convert_kernel<<<(unsigned)std::min<long long>((n8 + 255) / 256, 148LL * 16), 256, 0, st>>>(
      reinterpret_cast<const float4*>(dq_acc), static_cast<uint4*>(dq), n8);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  if (opt.events[3]) FA_CHECK_CUDA(cudaEventRecord(opt.events[3], st));
  return FA_OK;
}

// Shapes the tensor-core backward is compiled for (else the CUDA-core passes run).
inline bool supported(const AttnGeom& g) {
  return (g.D == 128 || g.D == 64) && g.bs_q == kTile && g.bs_kv == kTile;
}

}  // namespace
}  // namespace bwd
}  // namespace fa
