// entry.cuh — the call-level logic of forward / backward / decode shared by the C ABI (built-in
// descriptor functors, paper_2412_05496_b200/csrc/capi.cu) and the templated entry points for
// user functors (flexattn_b200_device.cuh): argument validation with the reference's error
// taxonomy (validate.cpp:16-34, engine.cpp:21-42, :174-201, :403-427), problem geometry, the
// data-dependent checks (FA_FLAG_VALIDATE), the choice between the tensor-core and the CUDA-core
// kernels, and the work counters.
#pragma once

#include <algorithm>
#include <string>

#include "block_mask.cuh"
#include "bwd_simt.cuh"
#include "bwd_sm100.cuh"
#include "dec_tc.cuh"
#include "decode.cuh"
#include "fwd1t.cuh"
#include "fwd_simt.cuh"
#include "fwd_sm100.cuh"
#include "host.cuh"
#include "validate.cuh"

namespace fa {

// ---- forward (engine.cpp:46-172) ----------------------------------------------------------------
inline fa_status prepare_fwd(const fa_fwd_args* a, AttnGeom* g) {
  FA_REQUIRE(a != nullptr, FA_SHAPE_MISMATCH, "forward: NULL args");
  fa_status s;
  if ((s = check_qkv(a->q, a->k, a->v, a->gqa_group))) return s;
  if ((s = check_tensor(a->out, "out"))) return s;
  FA_REQUIRE(same_shape(a->out, a->q) && a->out.dtype == a->q.dtype, FA_SHAPE_MISMATCH, "out must match q");
  FA_REQUIRE(a->lse != nullptr, FA_SHAPE_MISMATCH, "forward: NULL lse");
  if ((s = check_bm(a->bm, a->q.b, a->q.h, a->q.l, a->k.l))) return s;
  *g = geom_of(a->q, a->k, a->bm, a->scale, a->gqa_group);
  return FA_OK;
}

// validate_inputs' finiteness (validate.hpp:36-38) of q/k/v when FA_FLAG_VALIDATE
inline fa_status validate_qkv(const fa_tensor& q, const fa_tensor& k, const fa_tensor& v, uint32_t flags,
                              cudaStream_t st) {
  if (!(flags & FA_FLAG_VALIDATE)) return FA_OK;
  const fa_tensor ts[3] = {q, k, v};
  const char* names[3] = {"q", "k", "v"};
  return check_finite_list(ts, names, 3, st);
}

// After the checks of the mods: the flags and the finiteness scan.
inline fa_status begin_fwd(const fa_fwd_args* a, cudaStream_t st) {
  FA_REQUIRE(!(a->flags & ~uint32_t(FA_FLAG_VALIDATE)), FA_SHAPE_MISMATCH, "forward: unknown flags");
  return validate_qkv(a->q, a->k, a->v, a->flags, st);
}

// Forward for one mask and one score functor: the tensor-core kernel for bf16 at the compiled
// shapes, else the CUDA-core kernel; then the counters.
template <class MaskT, class ScoreT>
fa_status flex_fwd_t(const fa_fwd_args* a, MaskT mask, ScoreT score, cudaStream_t st) {
  AttnGeom g;
  fa_status s;
  if ((s = prepare_fwd(a, &g)) != FA_OK) return s;
  if ((s = begin_fwd(a, st)) != FA_OK) return s;
  const BmView bm = kv_view(a->bm);
  if (a->q.dtype == FA_BF16 && fwd::supported(g)) {
    s = g.D == 128 ? fwd::run<128>(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, bm, mask, score, st)
                   : fwd::run<64>(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, bm, mask, score, st);
  } else if (a->q.dtype == FA_BF16 && fwd1t::supported(g)) {  // rows past the two-tile kernel's list
    s = g.D == 128 ? fwd1t::run<128>(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, bm, mask, score, st)
                   : fwd1t::run<64>(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, bm, mask, score, st);
  } else if (a->q.dtype == FA_F32) {
    s = fsimt::run_any_dim<float>(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, bm, mask, score, st);
  } else {
    s = fsimt::run_any_dim<__nv_bfloat16>(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, bm, mask,
                                          score, st);
  }
  if (s != FA_OK || a->counters == nullptr) return s;
  return compute_counters(g, bm, mask, nullptr, g.Lkv, kPassForward, a->counters, st);
}

// ---- backward (engine.cpp:174-401) ----------------------------------------------------------------
inline fa_status prepare_bwd(const fa_bwd_args* a, AttnGeom* g) {
  FA_REQUIRE(a != nullptr, FA_SHAPE_MISMATCH, "backward: NULL args");
  fa_status s;
  if ((s = check_qkv(a->q, a->k, a->v, a->gqa_group))) return s;
  if ((s = check_tensor(a->out, "out")) || (s = check_tensor(a->d_out, "d_out")) || (s = check_tensor(a->dq, "dq")) ||
      (s = check_tensor(a->dk, "dk")) || (s = check_tensor(a->dv, "dv")))
    return s;
  FA_REQUIRE(same_shape(a->d_out, a->q) && a->d_out.dtype == a->q.dtype, FA_SHAPE_MISMATCH,
             "backward: d_out " + shp(a->d_out) + " must match q " + shp(a->q));
  FA_REQUIRE(same_shape(a->dq, a->q) && a->dq.dtype == a->q.dtype, FA_SHAPE_MISMATCH,
             "backward: dq " + shp(a->dq) + " must match q " + shp(a->q));
  FA_REQUIRE(same_shape(a->dk, a->k) && same_shape(a->dv, a->k) && a->dk.dtype == a->q.dtype &&
                 a->dv.dtype == a->q.dtype,
             FA_SHAPE_MISMATCH, "backward: dk/dv must match k " + shp(a->k));
  FA_REQUIRE(a->out.dtype == a->q.dtype, FA_STALE_STATISTICS, "backward: saved forward output has another dtype than q");
  FA_REQUIRE(same_shape(a->out, a->q), FA_STALE_STATISTICS,
             "backward: saved forward statistics do not match these tensors");
  FA_REQUIRE(a->lse != nullptr, FA_STALE_STATISTICS, "backward: NULL lse");
  if ((s = check_bm(a->bm, a->q.b, a->q.h, a->q.l, a->k.l))) return s;
  FA_REQUIRE(a->bm->q_num_blocks && a->bm->q_indices && a->bm->full_q_num_blocks && a->bm->full_q_indices,
             FA_BLOCK_MASK_MISMATCH, "backward: q-side (transposed) arrays required");
  FA_REQUIRE(a->workspace != nullptr &&
                 a->workspace_bytes >= bwd_workspace_bytes(a->q.b, a->q.h, a->q.l, a->q.d),
             FA_SHAPE_MISMATCH, "backward: workspace too small");
  *g = geom_of(a->q, a->k, a->bm, a->scale, a->gqa_group);
  return FA_OK;
}

// After the checks of the mods: the flags, the data-dependent checks before the launch (q/k/v as validate_inputs; d_out, engine.cpp:196, is
// checked inside the tensor-core path's preprocess read of d_out, else scanned here) and the
// phase events.
inline fa_status begin_bwd(const fa_bwd_args* a, bool tc_path, BwdOptions* opt, cudaStream_t st) {
  FA_REQUIRE(!(a->flags & ~uint32_t(FA_FLAG_VALIDATE | FA_FLAG_DETERMINISTIC)), FA_SHAPE_MISMATCH,
             "backward: unknown flags");
  opt->flags = a->flags;
  for (int i = 0; i < 4; ++i) opt->events[i] = static_cast<cudaEvent_t>(a->phase_events[i]);
  if (!(a->flags & FA_FLAG_VALIDATE)) return FA_OK;
  const fa_tensor ts[4] = {a->q, a->k, a->v, a->d_out};
  const char* names[4] = {"q", "k", "v", "d_out"};
  fa_status s;
  if ((s = check_finite_list(ts, names, tc_path ? 3 : 4, st)) != FA_OK) return s;
  if (tc_path) {
    opt->dout_nonfinite = scheduler_counter(kSlotFiniteErr, st);
    FA_REQUIRE(opt->dout_nonfinite != nullptr, FA_CUDA_ERROR, "backward: status word");
    FA_CHECK_CUDA(cudaMemsetAsync(opt->dout_nonfinite, 0, sizeof(int), st));
  }
  return FA_OK;
}
inline fa_status end_bwd(const BwdOptions& opt, cudaStream_t st) {
  if (opt.dout_nonfinite == nullptr) return FA_OK;
  int bad = 0;
  FA_CHECK_CUDA(cudaMemcpyAsync(&bad, opt.dout_nonfinite, sizeof(int), cudaMemcpyDeviceToHost, st));
  FA_CHECK_CUDA(cudaStreamSynchronize(st));
  FA_REQUIRE(bad == 0, FA_NON_FINITE_INPUT, "backward: d_out contains NaN or inf");
  return FA_OK;
}

template <class MaskT, class ScoreT>
fa_status flex_bwd_t(const fa_bwd_args* a, MaskT mask, ScoreT score, cudaStream_t st) {
  AttnGeom g;
  fa_status s;
  if ((s = prepare_bwd(a, &g)) != FA_OK) return s;
  const bool tc_path = a->q.dtype == FA_BF16 && bwd::supported(g);
  BwdOptions opt;
  if ((s = begin_bwd(a, tc_path, &opt, st)) != FA_OK) return s;
  const BmView bm = kv_view(a->bm), bmt = q_view(a->bm);
  const bool det = (a->flags & FA_FLAG_DETERMINISTIC) != 0;
  if (tc_path) {
#define FA_BWD_RUN(D, DET)                                                                                       \
  bwd::run<D, MaskT, ScoreT, DET>(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, a->d_out.data, a->dq.data, \
                                  a->dk.data, a->dv.data, bm, bmt, mask, score, a->workspace, opt, st)
    if (g.D == 128) s = det ? FA_BWD_RUN(128, bwd::kDeterministicMode) : FA_BWD_RUN(128, bwd::kDefaultMode);
    else s = det ? FA_BWD_RUN(64, bwd::kDeterministicMode) : FA_BWD_RUN(64, bwd::kDefaultMode);
#undef FA_BWD_RUN
  } else {
    s = bsimt::run_any(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, a->d_out.data, a->dq.data, a->dk.data,
                       a->dv.data, a->q.dtype, bm, bmt, mask, score, a->workspace, st);
  }
  if (s != FA_OK) return s;
  if ((s = end_bwd(opt, st)) != FA_OK) return s;
  if (a->counters == nullptr) return FA_OK;
  return compute_counters(g, bm, mask, nullptr, g.Lkv, kPassBackward, a->counters, st);
}

// ---- decode (engine.cpp:403-427, paged: paged_kv.cpp:154-310) -----------------------------------
struct DecodePlan {
  DecodeGeom g;
  PageView pv;
  int64_t mask_kv;  // kv positions the mask can be evaluated at (the paged kernel also stops at seq_len)
};

inline fa_status prepare_decode(const fa_decode_args* a, DecodePlan* plan, cudaStream_t st) {
  FA_REQUIRE(a != nullptr, FA_SHAPE_MISMATCH, "decode: NULL args");
  FA_REQUIRE(a->bm != nullptr, FA_BLOCK_MASK_MISMATCH, "decode: NULL block mask");
  fa_status s;
  if ((s = check_qkv(a->q, a->k_cache, a->v_cache, a->gqa_group))) return s;
  if ((s = check_tensor(a->out, "out"))) return s;
  FA_REQUIRE(same_shape(a->out, a->q) && a->out.dtype == a->q.dtype, FA_SHAPE_MISMATCH,
             "decode: out " + shp(a->out) + " must match q " + shp(a->q));
  FA_REQUIRE(a->lse != nullptr, FA_SHAPE_MISMATCH, "decode: NULL lse");
  FA_REQUIRE(a->q.dtype == FA_BF16 || a->pt == nullptr, FA_UNSUPPORTED,
             "decode: a paged cache needs bf16 (float32 decode is unpaged)");
  const int64_t n_new = a->q.l;
  int64_t logical_kv = a->k_cache.l;
  if (a->pt != nullptr) {
    const fa_page_table* pt = a->pt;
    FA_REQUIRE(pt->table && pt->phys_to_logical && pt->owner && pt->seq_len, FA_SHAPE_MISMATCH,
               "decode: page table arrays missing");
    FA_REQUIRE(a->k_cache.b == 1, FA_SHAPE_MISMATCH, "decode: paged cache must have batch 1");
    FA_REQUIRE(pt->batches == a->q.b, FA_SHAPE_MISMATCH, "decode: page table batches must equal q batch");
    FA_REQUIRE(pt->page_size == a->bm->bs_kv, FA_BLOCK_MASK_MISMATCH, "decode: page size must equal bs_kv");
    FA_REQUIRE(a->k_cache.l == pt->num_physical_pages * pt->page_size, FA_SHAPE_MISMATCH,
               "decode: physical cache length must be pages * page_size");
    // a converted mask (convert_block_mask): batch materialised, one column per physical page
    FA_REQUIRE(a->bm->b_dims == a->q.b, FA_BLOCK_MASK_MISMATCH, "decode: converted block mask must materialise the batch");
    FA_REQUIRE(a->bm->h_dims == 1 || a->bm->h_dims == a->q.h, FA_BLOCK_MASK_MISMATCH,
               "decode: block mask head dim must be 1 or " + std::to_string(a->q.h));
    FA_REQUIRE(a->bm->q_len == n_new && a->bm->kv_len == a->k_cache.l && a->bm->bs_q >= 1 &&
                   a->bm->rows == (n_new + a->bm->bs_q - 1) / a->bm->bs_q && a->bm->cols == pt->num_physical_pages,
               FA_BLOCK_MASK_MISMATCH, "decode: converted block mask geometry does not match the physical cache");
    FA_REQUIRE(a->bm->kv_num_blocks && a->bm->kv_indices && a->bm->full_kv_num_blocks && a->bm->full_kv_indices,
               FA_BLOCK_MASK_MISMATCH, "decode: block mask kv-side arrays missing");
    logical_kv = pt->max_logical_pages * pt->page_size;
    FA_REQUIRE(pt->max_seq_len >= 0 && pt->max_seq_len <= logical_kv, FA_SHAPE_MISMATCH,
               "decode: page table max_seq_len outside [0, max_logical_pages * page_size]");
  }
  plan->mask_kv = (a->pt && a->pt->max_seq_len > 0) ? a->pt->max_seq_len : logical_kv;
  // engine.cpp:410-414
  FA_REQUIRE(a->offset >= 0 && a->offset + n_new <= logical_kv, FA_OFFSET_OUT_OF_RANGE,
             "decode: rows [" + std::to_string(a->offset) + ", " + std::to_string(a->offset + n_new) +
                 ") fall outside cache");
  if (a->pt == nullptr) {
    if ((s = check_bm(a->bm, a->q.b, a->q.h, n_new, a->k_cache.l))) return s;
  }
  DecodeGeom& g = plan->g;
  g = DecodeGeom{};
  g.a = geom_of(a->q, a->k_cache, a->bm, a->scale, a->gqa_group);
  g.logical_kv = (int)plan->mask_kv;
  int splits = a->num_splits;
  if (splits <= 0) {
    // the row-per-CTA kernel holds one CTA per SM (192 KB smem): aim for ~28 waves of CTAs
    // (measured on C5: 2 splits 83.5 % of HBM vs 81.2 % with 1)
    const int64_t rows_total = a->q.b * a->q.h * n_new;
    const int64_t want = (28LL * num_sms() + rows_total - 1) / rows_total;
    splits = (int)std::max<int64_t>(1, std::min<int64_t>(want, std::min<int64_t>(64, a->bm->cols)));
  }
  g.num_splits = splits;
  if (splits > 1 && a->q.dtype == FA_BF16)
    FA_REQUIRE(a->workspace != nullptr &&
                   a->workspace_bytes >= decode_workspace_bytes(a->q.b, a->q.h, n_new, a->q.d, splits),
               FA_SHAPE_MISMATCH, "decode: workspace too small");
  plan->pv = PageView{};
  if (a->pt) {
    plan->pv.phys_to_logical = a->pt->phys_to_logical;
    plan->pv.owner = a->pt->owner;
    plan->pv.seq_len = a->pt->seq_len;
    plan->pv.page_size = (int)a->pt->page_size;
    plan->pv.enabled = 1;
  }
  (void)st;
  return FA_OK;
}

// After the checks of the mods: the finiteness scan and the foreign-page status word.
inline fa_status begin_decode(const fa_decode_args* a, DecodePlan* plan, cudaStream_t st) {
  FA_REQUIRE(!(a->flags & ~uint32_t(FA_FLAG_VALIDATE)), FA_SHAPE_MISMATCH, "decode: unknown flags");
  fa_status s;
  if ((s = validate_qkv(a->q, a->k_cache, a->v_cache, a->flags, st)) != FA_OK) return s;
  if (a->pt && (a->flags & FA_FLAG_VALIDATE) && a->q.dtype == FA_BF16) {
    // foreign pages -> UnmappedPhysicalIndex (paged_kv.cpp:265-269)
    plan->pv.foreign = scheduler_counter(kSlotConvertErr, st);
    FA_REQUIRE(plan->pv.foreign != nullptr, FA_CUDA_ERROR, "decode: status word");
    FA_CHECK_CUDA(cudaMemsetAsync(plan->pv.foreign, 0, sizeof(int), st));
  }
  return FA_OK;
}
inline fa_status end_decode(const DecodePlan& plan, cudaStream_t st) {
  if (plan.pv.foreign == nullptr) return FA_OK;
  int bad = 0;
  FA_CHECK_CUDA(cudaMemcpyAsync(&bad, plan.pv.foreign, sizeof(int), cudaMemcpyDeviceToHost, st));
  FA_CHECK_CUDA(cudaStreamSynchronize(st));
  FA_REQUIRE(bad == 0, FA_UNMAPPED_PHYSICAL_INDEX,
             "converted modifier: a visited physical page is not mapped for its batch element");
  return FA_OK;
}

// Decode with mask/score functors that already see absolute query positions (the offset shift
// of offset_mask / offset_score applied by the caller).
template <class MaskT, class ScoreT>
fa_status flex_decode_t(const fa_decode_args* a, const DecodePlan& plan_in, MaskT mask, ScoreT score,
                        cudaStream_t st) {
  DecodePlan plan = plan_in;
  fa_status s;
  if ((s = begin_decode(a, &plan, st)) != FA_OK) return s;
  const BmView bm = kv_view(a->bm);
  if (a->q.dtype == FA_F32) {
    // decode<float> is forward_impl over the shifted mask (engine.cpp:403-427)
    s = fsimt::run_any_dim<float>(plan.g.a, a->q.data, a->k_cache.data, a->v_cache.data, a->out.data, a->lse, bm,
                                  mask, score, st);
    if (s != FA_OK || a->counters == nullptr) return s;
    return compute_counters(plan.g.a, bm, mask, nullptr, plan.g.a.Lkv, kPassForward, a->counters, st);
  }
  dec::DecParams p{};
  if ((s = dec::make_params(plan.g, a->q.data, a->k_cache.data, a->v_cache.data, a->out.data, a->lse, bm, plan.pv,
                            a->workspace, &p)) != FA_OK)
    return s;
  if (dectc::supported(plan.g)) {  // several rows per kv head: one tensor-core tile per (b, kv head)
    s = plan.g.a.D == 128 ? dectc::run<128>(plan.g, a->q.data, a->k_cache.data, a->v_cache.data, a->out.data, a->lse,
                                            bm, plan.pv, a->workspace, mask, score, st)
                          : dectc::run<64>(plan.g, a->q.data, a->k_cache.data, a->v_cache.data, a->out.data, a->lse,
                                           bm, plan.pv, a->workspace, mask, score, st);
  } else {
    s = dec::run_any_dim(p, mask, score, st);
  }
  if (s != FA_OK) return s;
  if ((s = end_decode(plan, st)) != FA_OK) return s;
  if (a->counters == nullptr) return FA_OK;
  return compute_counters(plan.g.a, bm, mask, &plan.pv, plan.g.logical_kv, kPassForward, a->counters, st);
}

}  // namespace fa
