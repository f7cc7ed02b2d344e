// bwd_sm100.cu — block-sparse FlexAttention backward for sm_100a (bf16 in, fp32
// accumulate), the tensor-core replacement of backward (engine.cpp:174-401).
//
// Kernels (one stream, in order):
//   1. preprocess: Δ_i = Σ_d dO·O (engine.cpp:218-235), lse in log2 units (+inf on
//      fully masked rows so they contribute exactly nothing, :257-260), padded to
//      128-row q blocks; dQ accumulator zeroed.
//   2. main: persistent, warp-specialised CTA (512 threads). A work item is one
//      128-row kv block of one (kv batch, kv head) — the dK/dV pass of the
//      reference (:307-395): it loops the kv-batch broadcast and the G query
//      heads of the group and walks the transposed (q-side) lists, so dK and dV
//      accumulate in TMEM for the whole item. Per visited q block:
//        MMA1 S^T  = K Q^T            (SS, TMEM fp32, 128 x 128)
//        MMA2 dP^T = V dO^T           (SS)
//        compute warps (thread = kv row, two warpgroups split the 128 q columns):
//           P^T  = exp2(score_mod(S^T) - lse)      mask_mod only in partial blocks
//           dS^T = P^T (dP^T - Δ) score_mod'(s) scale
//           -> P^T, dS^T as bf16 into TMEM (aliasing S^T / dP^T) and dS^T into smem
//        MMA3 dV += P^T dO            (TS, dO MN-major)
//        MMA4 dK += dS^T Q            (TS, Q MN-major)
//        MMA5 dQ_blk = dS K           (SS, both MN-major) into the dP^T columns
//        reduce warps: dQ_blk -> red.global.add.v4.f32 into the fp32 dQ accumulator
//      (the fused form of the reference's separate dQ pass, :237-305).
//      Warps 0-7 = compute (two warpgroups, 64 q columns each); warps 8-11 = dQ
//      reduction (pull the dQ tile out of TMEM, release it, red.add while the next
//      block runs) and the dK/dV epilogue; warp 12 = TMA producer (K/V once per
//      item; Q, dO, lse, Δ per q block, 2-stage ring); warp 13 = MMA issuer.
//      Register budgets per warpgroup via setmaxnreg (136 / 152 / 80).
//      TMEM: S^T [0,128)  dP^T/dQ [128,256)  dV [256,256+D)  dK [256+D,256+2D).
//   3. convert: dQ fp32 -> bf16.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>

#include "internal.h"
#include "mods.cuh"
#include "sm100_ptx.cuh"

namespace fa {

CUresult encode_tile_map(CUtensorMap* map, const void* base, int bh, int len, int d);
int* scheduler_counter(int slot);

namespace {

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
  const float* lse2;   // (B*Hq, Lq_pad)
  const float* delta;  // (B*Hq, Lq_pad)
  float* dq_acc;       // (B*Hq, Lq, D) fp32
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  float scale;
  int num_items;
  int* work_counter;
  long long* trace;  // debug only (FA_BWD_TRACE): per-block phase timestamps of CTA 0
  int exp_flags;     // debug only (FA_BWD_EXP): 1 = skip dQ reductions
};

// trace slots: [task][event], events: 0 compute-start 1 compute-done 2 mma-ds_full 3 mma5-issued
// 4 dq_free-wait-done 5 reduce-dq_full 6 reduce-released 7 reduce-red-issued
constexpr int kTraceTasks = 256, kTraceEv = 12;
__device__ __forceinline__ void trace_ev(const BwdParams& p, int task, int ev) {
  if (p.trace != nullptr && blockIdx.x == 0 && task < kTraceTasks) {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    p.trace[task * kTraceEv + ev] = t;
  }
}

template <int D>
struct BCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = kTile * D * 2;
  static constexpr int kChunkBytes = kTile * 128;
};

template <int D>
struct alignas(1024) BSmem {
  uint8_t k[BCfg<D>::kTileBytes];
  uint8_t v[BCfg<D>::kTileBytes];
  uint8_t q[2][BCfg<D>::kTileBytes];
  uint8_t dO[2][BCfg<D>::kTileBytes];
  uint8_t ds[kTile * kTile * 2];  // dS^T as the MN-major A operand of MMA5
  float lse2[2][kTile];
  float delta[2][kTile];
  uint64_t kv_full, kv_free;
  uint64_t q_full[2], q_free[2];
  uint64_t s_full, dp_full, ds_full, dq_full, dq_free, dkdv_full, dkdv_free;
  uint64_t item_full[2], item_empty[2];
  int32_t uitem[2];
  uint32_t tmem_base;
};

struct KvItem {
  int kb, kh, c;
};
__device__ __forceinline__ KvItem decode_kv_item(const BwdParams& p, int item) {
  const int per = p.Bkv * p.Hkv;
  const int c = item / per, rem = item % per;  // low kv blocks first: the heaviest for causal masks
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

template <int D, class MaskT, class ScoreT>
__global__ void __launch_bounds__(kThreads, 1)
    flex_bwd_sm100_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmDO, const BwdParams p, MaskT mask,
                          ScoreT score) {
  using C = BCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  BSmem<D>& sm = *reinterpret_cast<BSmem<D>*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();  // SWIZZLE_128B operands need 1 KiB alignment

  if (threadIdx.x == 0) {
    mbar_init(&sm.kv_full, 1);
    mbar_init(&sm.kv_free, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.q_full[s], 1);
      mbar_init(&sm.q_free[s], 1);
      mbar_init(&sm.item_full[s], 1);
      mbar_init(&sm.item_empty[s], 1 + 8 + 4);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.dp_full, 1);
    mbar_init(&sm.ds_full, 256);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_free, 128);
    mbar_init(&sm.dkdv_full, 1);
    mbar_init(&sm.dkdv_free, 128);
    fence_barrier_init();
  }
  if (warp == 12 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
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
    reg_dealloc<80>();
  }
  if (warp == 12) {
    if (lane == 0) {
      // ===================== TMA producer =====================
      int qs_it = 0;
      for (int n = 0;; ++n) {
        const int item = n == 0 ? static_cast<int>(blockIdx.x)
                                : static_cast<int>(gridDim.x) + atomicAdd(p.work_counter, 1);
        const int buf = n & 1;
        mbar_wait(&sm.item_empty[buf], ((n >> 1) & 1) ^ 1);
        sm.uitem[buf] = item < p.num_items ? item : -1;
        mbar_arrive(&sm.item_full[buf]);
        if (item >= p.num_items) break;
        const KvItem it = decode_kv_item(p, item);
        mbar_wait(&sm.kv_free, (n & 1) ^ 1);
        mbar_expect_tx(&sm.kv_full, 2 * C::kTileBytes);
        for (int ch = 0; ch < C::kChunks; ++ch) {
          tma_load_3d(sm.k + ch * C::kChunkBytes, &tmK, &sm.kv_full, ch * 64, it.c * kTile,
                      it.kb * p.Hkv + it.kh);
          tma_load_3d(sm.v + ch * C::kChunkBytes, &tmV, &sm.kv_full, ch * 64, it.c * kTile,
                      it.kb * p.Hkv + it.kh);
        }
        TaskIter ti;
        ti.init(p, it);
        int b, h, r;
        bool full;
        while (ti.next(b, h, r, full)) {
          const int st = qs_it & 1;
          mbar_wait(&sm.q_free[st], ((qs_it >> 1) & 1) ^ 1);
          mbar_expect_tx(&sm.q_full[st], 2 * C::kTileBytes + 2 * kTile * 4);
          for (int ch = 0; ch < C::kChunks; ++ch) {
            tma_load_3d(sm.q[st] + ch * C::kChunkBytes, &tmQ, &sm.q_full[st], ch * 64, r * kTile,
                        b * p.Hq + h);
            tma_load_3d(sm.dO[st] + ch * C::kChunkBytes, &tmDO, &sm.q_full[st], ch * 64, r * kTile,
                        b * p.Hq + h);
          }
          const long long row0 = static_cast<long long>(b * p.Hq + h) * p.Lq_pad + r * kTile;
          bulk_load(sm.lse2[st], p.lse2 + row0, kTile * 4, &sm.q_full[st]);
          bulk_load(sm.delta[st], p.delta + row0, kTile * 4, &sm.q_full[st]);
          ++qs_it;
        }
      }
    }
    FA_BWD_TEARDOWN();
  } else if (warp == 13) {
    if (lane == 0) {
      // ===================== MMA issuer =====================
      constexpr uint32_t idesc_ss = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_ts = make_idesc_bf16(128, D, 0, 1);
      constexpr uint32_t idesc_mm = make_idesc_bf16(128, D, 1, 1);
      constexpr uint32_t idesc_mmT = make_idesc_bf16(D, 128, 1, 1);
      const uint32_t k_addr = smem_u32(sm.k), v_addr = smem_u32(sm.v), ds_addr = smem_u32(sm.ds);
      int qs_it = 0;
      uint32_t ds_ph = 0, mma2_count = 0;
      auto mma_kmajor = [&](uint32_t d_col, uint32_t a_addr, uint32_t b_addr, uint64_t* bar) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::kChunkBytes + (kk & 3) * 32;
          umma_ss(tmem + d_col, make_sdesc_sw128(a_addr + off, 16, 1024),
                  make_sdesc_sw128(b_addr + off, 16, 1024), idesc_ss, kk > 0 ? 1u : 0u);
        }
        umma_commit(bar);
      };
      for (int n = 0;; ++n) {
        const int buf = n & 1;
        mbar_wait(&sm.item_full[buf], (n >> 1) & 1);
        const int item = sm.uitem[buf];
        mbar_arrive(&sm.item_empty[buf]);
        if (item < 0) break;
        const KvItem it = decode_kv_item(p, item);
        const int T = count_tasks(p, it);
        mbar_wait(&sm.kv_full, n & 1);
        tc_fence_after();
        if (T > 0) {
          const int st0 = qs_it & 1;
          mbar_wait(&sm.q_full[st0], (qs_it >> 1) & 1);
          tc_fence_after();
          mma_kmajor(kS, k_addr, smem_u32(sm.q[st0]), &sm.s_full);
          mbar_wait(&sm.dq_free, (mma2_count & 1) ^ 1);
          tc_fence_after();
          mma_kmajor(kDP, v_addr, smem_u32(sm.dO[st0]), &sm.dp_full);
          ++mma2_count;
        }
        for (int t = 0; t < T; ++t) {
          const int st = (qs_it + t) & 1;
          if (t == 0) mbar_wait(&sm.dkdv_free, (n & 1) ^ 1);  // previous item's dK/dV read out
          mbar_wait(&sm.ds_full, ds_ph);
          ds_ph ^= 1;
          tc_fence_after();
          trace_ev(p, qs_it + t, 2);
          const uint32_t q_addr = smem_u32(sm.q[st]), do_addr = smem_u32(sm.dO[st]);
#pragma unroll
          for (int kk = 0; kk < kTile / 16; ++kk) {  // MMA3: dV += P^T dO
            const uint32_t a_col = kS + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8);
            umma_ts(tmem + kDV, tmem + a_col, make_sdesc_sw128(do_addr + kk * 2048, C::kChunkBytes, 1024),
                    idesc_ts, (t > 0 || kk > 0) ? 1u : 0u);
          }
#pragma unroll
          for (int kk = 0; kk < kTile / 16; ++kk) {  // MMA4: dK += dS^T Q
            const uint32_t a_col = kDP + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8);
            umma_ts(tmem + kDK, tmem + a_col, make_sdesc_sw128(q_addr + kk * 2048, C::kChunkBytes, 1024),
                    idesc_ts, (t > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&sm.q_free[st]);
          if constexpr (D == 128) {
            // MMA5: dQ_blk^T = K^T dS^T (M = head dim, N = q) over the dP^T columns, so the
            // reduction warps own one head-dim index each and write coalesced 128-byte lines
#pragma unroll
            for (int kk = 0; kk < kTile / 16; ++kk)
              umma_ss(tmem + kDP, make_sdesc_sw128(k_addr + kk * 2048, C::kChunkBytes, 1024),
                      make_sdesc_sw128(ds_addr + kk * 2048, kTile * 128, 1024), idesc_mmT,
                      kk > 0 ? 1u : 0u);
          } else {
#pragma unroll
            for (int kk = 0; kk < kTile / 16; ++kk)  // MMA5: dQ_blk = dS K (over the dP^T columns)
              umma_ss(tmem + kDP, make_sdesc_sw128(ds_addr + kk * 2048, kTile * 128, 1024),
                      make_sdesc_sw128(k_addr + kk * 2048, C::kChunkBytes, 1024), idesc_mm,
                      kk > 0 ? 1u : 0u);
          }
          umma_commit(&sm.dq_full);
          trace_ev(p, qs_it + t, 3);
          if (t + 1 < T) {
            const int st1 = (qs_it + t + 1) & 1;
            mbar_wait(&sm.q_full[st1], ((qs_it + t + 1) >> 1) & 1);
            tc_fence_after();
            mma_kmajor(kS, k_addr, smem_u32(sm.q[st1]), &sm.s_full);
            mbar_wait(&sm.dq_free, (mma2_count & 1) ^ 1);
            tc_fence_after();
            trace_ev(p, qs_it + t, 4);
            mma_kmajor(kDP, v_addr, smem_u32(sm.dO[st1]), &sm.dp_full);
            trace_ev(p, qs_it + t, 11);
            ++mma2_count;
          }
        }
        qs_it += T;
        umma_commit(&sm.dkdv_full);
        umma_commit(&sm.kv_free);
      }
    }
    FA_BWD_TEARDOWN();
  } else if (warp < 8) {
    // ===================== compute warpgroups: P^T, dS^T =====================
    reg_alloc<136>();
    const int wg = warp >> 2;          // which 64 q columns
    const int wq = warp & 3;           // TMEM lane quarter
    const int j = wq * 32 + lane;      // kv row within the block
    const uint32_t tm = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    uint32_t s_ph = 0;
    int qs_it = 0;
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
        const int st = qs_it & 1;
        const int q0 = r * kTile + wg * 64;
        const auto colc = score.col(b, h, q0, kv, p.scale);
        if (threadIdx.x == 0) trace_ev(p, qs_it, 8);
        mbar_wait(&sm.s_full, s_ph);
        if (threadIdx.x == 0) trace_ev(p, qs_it, 9);
        mbar_wait(&sm.dp_full, s_ph);
        s_ph ^= 1;
        if (threadIdx.x == 0) trace_ev(p, qs_it, 10);
        mbar_wait(&sm.q_full[st], (qs_it >> 1) & 1);  // lse2 / delta of this q block
        tc_fence_after();
        if (threadIdx.x == 0) trace_ev(p, qs_it, 0);
        uint8_t* ds_row = sm.ds + wg * (kTile * 128) + j * 128;
        // two halves of 32 q columns keep ~100 registers live
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          const int qc = q0 + hh * 32;
          const auto cc = colc.shifted(hh * 32);
          uint32_t sr[32], dpr[32];
          tmem_ld32(tm + kS + wg * 64 + hh * 32, sr);
          tmem_ld32(tm + kDP + wg * 64 + hh * 32, dpr);
          // mask bits for this kv row over the 32 q columns (bounds folded in)
          const uint32_t bits = full ? 0xffffffffu : (kv_in ? mask.bits32_q(b, h, qc, kv, p.Lq) : 0u);
          const float4* lse4 = reinterpret_cast<const float4*>(sm.lse2[st] + wg * 64 + hh * 32);
          const float4* dlt4 = reinterpret_cast<const float4*>(sm.delta[st] + wg * 64 + hh * 32);
          tmem_wait_ld();
          uint32_t pp[16], dsp[16];
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4) {
            const float4 l4 = lse4[i4], d4 = dlt4[i4];
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dv4[4] = {d4.x, d4.y, d4.z, d4.w};
            float pv[4], dsv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int ii = i4 * 4 + e;
              float g;
              const float x = cc.log2_grad(__uint_as_float(sr[ii]), ii, g);
              const float pr = ((bits >> ii) & 1u) ? ex2(x - lv[e]) : 0.f;
              pv[e] = pr;
              dsv[e] = pr * (__uint_as_float(dpr[ii]) - dv4[e]) * (g * p.scale);
            }
            pp[2 * i4] = pack_bf16(pv[0], pv[1]);
            pp[2 * i4 + 1] = pack_bf16(pv[2], pv[3]);
            dsp[2 * i4] = pack_bf16(dsv[0], dsv[1]);
            dsp[2 * i4 + 1] = pack_bf16(dsv[2], dsv[3]);
          }
          tmem_st16(tm + kS + wg * 64 + hh * 16, pp);    // P^T  over S^T columns already read
          tmem_st16(tm + kDP + wg * 64 + hh * 16, dsp);  // dS^T over dP^T columns already read
          // dS^T row j (MN-major SW128 A operand of MMA5): 16-byte units 4hh..4hh+3
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int uu = hh * 4 + u;
            *reinterpret_cast<uint4*>(ds_row + ((uu ^ (j & 7)) << 4)) =
                make_uint4(dsp[4 * u], dsp[4 * u + 1], dsp[4 * u + 2], dsp[4 * u + 3]);
          }
        }
        tmem_wait_st();
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(&sm.ds_full);
        if (threadIdx.x == 0) trace_ev(p, qs_it, 1);
        ++qs_it;
      }
    }
    FA_BWD_TEARDOWN();
  } else if (warp < 12) {
    // ===================== dQ reduction + dK/dV epilogue warpgroup =====================
    reg_alloc<152>();
    const int wq = warp & 3;
    const uint32_t tm = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    uint32_t dq_ph = 0;
    int red_it = 0;
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
        // dQ_blk (lanes = q rows): pull all D columns out of TMEM, release it, then reduce
        mbar_wait(&sm.dq_full, dq_ph);
        dq_ph ^= 1;
        tc_fence_after();
        if (threadIdx.x == 256) trace_ev(p, red_it, 5);
        uint32_t a[128];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
          tmem_ld32(tm + kDP + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&a[cc * 32]));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&sm.dq_free);
        if (threadIdx.x == 256) trace_ev(p, red_it, 6);
        if (!(p.exp_flags & 1)) {
          if constexpr (D == 128) {
            // lanes = head-dim index d, columns = q rows of the block: per q row the warp's 32
            // lanes add 32 consecutive floats (one 128-byte line)
            const int d = wq * 32 + lane;
            const int q0r = r * kTile;
            const int nq = min(kTile, p.Lq - q0r);
            float* base = p.dq_acc + (static_cast<long long>(b * p.Hq + h) * p.Lq + q0r) * D + d;
            if (nq == kTile) {
#pragma unroll
              for (int qq = 0; qq < kTile; ++qq) red_add_f32(base + qq * D, __uint_as_float(a[qq]));
            } else {
#pragma unroll
              for (int qq = 0; qq < kTile; ++qq)
                if (qq < nq) red_add_f32(base + qq * D, __uint_as_float(a[qq]));
            }
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
        if (threadIdx.x == 256) trace_ev(p, red_it, 7);
        ++red_it;
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
              d4[q4] = make_uint4(pack_bf16(__uint_as_float(v[8 * q4]), __uint_as_float(v[8 * q4 + 1])),
                                  pack_bf16(__uint_as_float(v[8 * q4 + 2]), __uint_as_float(v[8 * q4 + 3])),
                                  pack_bf16(__uint_as_float(v[8 * q4 + 4]), __uint_as_float(v[8 * q4 + 5])),
                                  pack_bf16(__uint_as_float(v[8 * q4 + 6]), __uint_as_float(v[8 * q4 + 7])));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.dkdv_free);
    }
    FA_BWD_TEARDOWN();
  } else {
    FA_BWD_TEARDOWN();  // warps 14-15: idle
  }
#undef FA_BWD_TEARDOWN
}

// Δ and log2-domain lse, padded to whole q blocks (+inf lse / 0 Δ in the padding).
__global__ void bwd_preprocess_kernel(const __nv_bfloat16* __restrict__ o,
                                      const __nv_bfloat16* __restrict__ dout,
                                      const float* __restrict__ lse, int BH, int Lq, int Lq_pad, int D,
                                      float* __restrict__ lse2, float* __restrict__ delta) {
  const long long row = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (long long)BH * Lq_pad) return;
  const int q = (int)(row % Lq_pad);
  const long long bh = row / Lq_pad;
  if (q >= Lq) {
    if (lane == 0) {
      lse2[row] = INFINITY;
      delta[row] = 0.f;
    }
    return;
  }
  const long long src = (bh * Lq + q) * D;
  float a = 0.f;
  for (int d = lane * 2; d < D; d += 64) {
    const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(o + src + d);
    const __nv_bfloat162 y = *reinterpret_cast<const __nv_bfloat162*>(dout + src + d);
    a = fmaf(__low2float(x), __low2float(y), a);
    a = fmaf(__high2float(x), __high2float(y), a);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
  if (lane == 0) {
    const float l = lse[bh * Lq + q];
    lse2[row] = l == -INFINITY ? INFINITY : l * kLog2e;
    delta[row] = a;
  }
}

__global__ void dq_convert_kernel(const float4* __restrict__ acc, __nv_bfloat162* __restrict__ dq, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = acc[i];
    dq[2 * i] = __floats2bfloat162_rn(v.x, v.y);
    dq[2 * i + 1] = __floats2bfloat162_rn(v.z, v.w);
  }
}

template <int D, class MaskT, class ScoreT>
fa_status run(const AttnGeom& g, const void* q, const void* k, const void* v, const void* o,
              const float* lse, const void* dout, void* dq, void* dk, void* dv, const BmView& bmt,
              MaskT mask, ScoreT score, void* workspace, cudaStream_t st) {
  const int Lq_pad = (g.Lq + kTile - 1) / kTile * kTile;
  const long long rows = (long long)g.B * g.Hq * g.Lq;
  const long long prow = (long long)g.B * g.Hq * Lq_pad;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* ws = static_cast<char*>(workspace);
  float* dq_acc = reinterpret_cast<float*>(ws);
  float* lse2 = reinterpret_cast<float*>(ws + al(rows * D * 4));
  float* delta = reinterpret_cast<float*>(ws + al(rows * D * 4) + al(prow * 4));
  FA_CHECK_CUDA(cudaMemsetAsync(dq_acc, 0, rows * D * 4, st));
  bwd_preprocess_kernel<<<(unsigned)((prow + 7) / 8), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), lse,
      g.B * g.Hq, g.Lq, Lq_pad, D, lse2, delta);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());

  CUtensorMap mq, mk, mv, mdo;
  CUresult cr;
  if ((cr = encode_tile_map(&mq, q, g.B * g.Hq, g.Lq, D)) != CUDA_SUCCESS ||
      (cr = encode_tile_map(&mk, k, g.Bkv * g.Hkv, g.Lkv, D)) != CUDA_SUCCESS ||
      (cr = encode_tile_map(&mv, v, g.Bkv * g.Hkv, g.Lkv, D)) != CUDA_SUCCESS ||
      (cr = encode_tile_map(&mdo, dout, g.B * g.Hq, g.Lq, D)) != CUDA_SUCCESS)
    return set_error(FA_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string((int)cr) + ")");
  BwdParams p{};
  p.B = g.B; p.Hq = g.Hq; p.Hkv = g.Hkv; p.Bkv = g.Bkv; p.Lq = g.Lq; p.Lkv = g.Lkv; p.G = g.G;
  p.Lq_pad = Lq_pad;
  p.bm_b = g.bm_b; p.bm_h = g.bm_h; p.rows = g.rows; p.cols = g.cols;
  p.q_num = bmt.kv_num; p.q_idx = bmt.kv_idx; p.fq_num = bmt.full_num; p.fq_idx = bmt.full_idx;
  p.lse2 = lse2; p.delta = delta; p.dq_acc = dq_acc;
  p.dk = static_cast<__nv_bfloat16*>(dk);
  p.dv = static_cast<__nv_bfloat16*>(dv);
  p.scale = g.scale;
  p.num_items = g.Bkv * g.Hkv * g.cols;
  p.work_counter = scheduler_counter(1);
  FA_REQUIRE(p.work_counter != nullptr, FA_CUDA_ERROR, "backward: cannot allocate the scheduler counter");
  FA_CHECK_CUDA(cudaMemsetAsync(p.work_counter, 0, sizeof(int), st));
  long long* trace = nullptr;
  if (getenv("FA_BWD_TRACE") != nullptr) {
    FA_CHECK_CUDA(cudaMalloc(&trace, sizeof(long long) * kTraceTasks * kTraceEv));
    FA_CHECK_CUDA(cudaMemsetAsync(trace, 0, sizeof(long long) * kTraceTasks * kTraceEv, st));
  }
  p.trace = trace;
  p.exp_flags = getenv("FA_BWD_EXP") ? atoi(getenv("FA_BWD_EXP")) : 0;
  const size_t smem = sizeof(BSmem<D>);
  auto kern = flex_bwd_sm100_kernel<D, MaskT, ScoreT>;
  FA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = p.num_items < num_sms() ? p.num_items : num_sms();
  if (grid > 0) {
    kern<<<grid, kThreads, smem, st>>>(mq, mk, mv, mdo, p, mask, score);
    count_launch();
    FA_CHECK_CUDA(cudaGetLastError());
  }
  if (trace != nullptr) {  // debug: per-phase cycle deltas of CTA 0, averaged over its blocks
    long long h[kTraceTasks * kTraceEv];
    FA_CHECK_CUDA(cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st));
    FA_CHECK_CUDA(cudaStreamSynchronize(st));
    cudaFree(trace);
    double acc[12] = {0};
    int cnt = 0;
    for (int t = 1; t + 1 < kTraceTasks; ++t) {
      const long long* e = h + t * kTraceEv;
      const long long* en = h + (t + 1) * kTraceEv;
      if (e[0] == 0 || en[0] == 0 || e[7] == 0) break;
      acc[0] += e[1] - e[0];    // compute
      acc[1] += e[2] - e[1];    // ds_full -> MMA sees it
      acc[2] += e[5] - e[3];    // MMA5 issue -> dQ ready (MMA3..5 execution)
      acc[3] += e[6] - e[5];    // dQ TMEM load
      acc[4] += e[4] - e[6];    // dq_free -> MMA2 issue
      acc[5] += en[0] - e[4];   // MMA2 issue -> next compute start
      acc[6] += en[0] - e[0];   // period
      acc[7] += e[7] - e[6];    // red issue
      acc[8] += e[3] - e[2];    // MMA3..5 issue duration
      acc[9] += e[11] - e[4];   // MMA2 issue duration
      acc[10] += en[9] - e[11]; // MMA2 issued -> next s_full seen
      acc[11] += en[10] - en[9];// s_full -> dp_full
      ++cnt;
    }
    if (cnt > 0)
      fprintf(stderr,
              "[bwd trace] blocks=%d cycles: compute %.0f | ds->mma %.0f | mma3-5 %.0f | dq ld %.0f | "
              "free->mma2 %.0f | mma2->compute %.0f | period %.0f | red issue %.0f | mma3-5 issue %.0f | "
              "mma2 issue %.0f | mma2 issued->s_full %.0f | s_full->dp_full %.0f\n",
              cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt,
              acc[6] / cnt, acc[7] / cnt, acc[8] / cnt, acc[9] / cnt, acc[10] / cnt, acc[11] / cnt);
  }
  const long long n4 = rows * D / 4;
  dq_convert_kernel<<<(unsigned)std::min<long long>((n4 + 255) / 256, 148LL * 16), 256, 0, st>>>(
      reinterpret_cast<const float4*>(dq_acc), static_cast<__nv_bfloat162*>(dq), n4);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

template <int D, class ScoreT>
fa_status by_mask(const AttnGeom& g, const void* q, const void* k, const void* v, const void* o,
                  const float* lse, const void* dout, void* dq, void* dk, void* dv, const BmView& bmt,
                  const MaskParams& mp, int mk, ScoreT s, void* ws, cudaStream_t st) {
  switch (mk) {
    case kMaskNoop: return run<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, MaskFn<kMaskNoop>{mp}, s, ws, st);
    case kMaskCausalOnly: return run<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, MaskFn<kMaskCausalOnly>{mp}, s, ws, st);
    case kMaskSlidingOnly: return run<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, MaskFn<kMaskSlidingOnly>{mp}, s, ws, st);
    case kMaskDocCausal: return run<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, MaskFn<kMaskDocCausal>{mp}, s, ws, st);
    default: return run<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, MaskFn<kMaskDynamic>{mp}, s, ws, st);
  }
}

template <int D>
fa_status by_score(const AttnGeom& g, const void* q, const void* k, const void* v, const void* o,
                   const float* lse, const void* dout, void* dq, void* dk, void* dv, const BmView& bmt,
                   const MaskParams& mp, int mk, const ScoreParams& sp, int sk, void* ws, cudaStream_t st) {
  switch (sk) {
    case 0: return by_mask<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, mp, mk, ScoreFn<0>{sp}, ws, st);
    case 1: return by_mask<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, mp, mk, ScoreFn<1>{sp}, ws, st);
    case 2: return by_mask<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, mp, mk, ScoreFn<2>{sp}, ws, st);
    default: return by_mask<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, mp, mk, ScoreFn<3>{sp}, ws, st);
  }
}

}  // namespace

bool bwd_sm100_supported(const AttnGeom& g) {
  return (g.D == 128 || g.D == 64) && g.bs_q == kTile && g.bs_kv == kTile;
}

fa_status launch_bwd_sm100(const AttnGeom& g, const void* q, const void* k, const void* v,
                           const void* o, const float* lse, const void* dout, void* dq, void* dk,
                           void* dv, const BmView& bm, const BmView& bmt, const MaskParams& mp,
                           int mkind, const ScoreParams& sp, int skind, void* workspace,
                           cudaStream_t st) {
  (void)bm;
  if (g.D == 128)
    return by_score<128>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, mp, mkind, sp, skind, workspace, st);
  return by_score<64>(g, q, k, v, o, lse, dout, dq, dk, dv, bmt, mp, mkind, sp, skind, workspace, st);
}

}  // namespace fa
