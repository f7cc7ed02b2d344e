// bwd_sm100.cu — the library's instantiations of the tensor-core backward
// (include/flexattn_b200/bwd_sm100.cuh) for the built-in mask/score functors, and the choice
// between it and the CUDA-core passes (include/flexattn_b200/bwd_simt.cuh).
#include "internal.h"
#include "flexattn_b200/bwd_simt.cuh"
#include "flexattn_b200/bwd_sm100.cuh"

namespace fa {
namespace {

template <int D, class ScoreT>
fa_status by_mask(const AttnGeom& g, const void* q, const void* k, const void* v, const void* o,
                  const float* lse, const void* dout, void* dq, void* dk, void* dv, const BmView& bm,
                  const BmView& bmt, const MaskParams& mp, int mk, ScoreT s, void* ws,
                  const BwdOptions& opt, cudaStream_t st) {
  // deterministic mode: one instantiation per score kind, the dynamic (any-combination) mask
  if (opt.flags & FA_FLAG_DETERMINISTIC && bwd::kDeterministicMode != bwd::kDefaultMode)
    return bwd::run<D, MaskFn<kMaskDynamic>, ScoreT, bwd::kDeterministicMode>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt,
                                                            MaskFn<kMaskDynamic>{mp}, s, ws, opt, st);
  switch (mk) {
    case kMaskNoop:
      return bwd::run<D, MaskFn<kMaskNoop>, ScoreT, bwd::kDefaultMode>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt,
                                                            MaskFn<kMaskNoop>{mp}, s, ws, opt, st);
    case kMaskCausalOnly:
      return bwd::run<D, MaskFn<kMaskCausalOnly>, ScoreT, bwd::kDefaultMode>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt,
                                                                  MaskFn<kMaskCausalOnly>{mp}, s, ws, opt, st);
    case kMaskSlidingOnly:
      return bwd::run<D, MaskFn<kMaskSlidingOnly>, ScoreT, bwd::kDefaultMode>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt,
                                                                   MaskFn<kMaskSlidingOnly>{mp}, s, ws, opt, st);
    case kMaskDocCausal:
      return bwd::run<D, MaskFn<kMaskDocCausal>, ScoreT, bwd::kDefaultMode>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt,
                                                                 MaskFn<kMaskDocCausal>{mp}, s, ws, opt, st);
    default:
      return bwd::run<D, MaskFn<kMaskDynamic>, ScoreT, bwd::kDefaultMode>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt,
                                                               MaskFn<kMaskDynamic>{mp}, s, ws, opt, st);
  }
}

template <int D>
fa_status by_score(const AttnGeom& g, const void* q, const void* k, const void* v, const void* o,
                   const float* lse, const void* dout, void* dq, void* dk, void* dv, const BmView& bm,
                   const BmView& bmt, const MaskParams& mp, int mk, const ScoreParams& sp, int sk,
                   void* ws, const BwdOptions& opt, cudaStream_t st) {
  switch (sk) {
    case 0: return by_mask<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mp, mk, ScoreFn<0>{sp}, ws, opt, st);
    case 1: return by_mask<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mp, mk, ScoreFn<1>{sp}, ws, opt, st);
    case 2: return by_mask<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mp, mk, ScoreFn<2>{sp}, ws, opt, st);
    default: return by_mask<D>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mp, mk, ScoreFn<3>{sp}, ws, opt, st);
  }
}

template <class ScoreT>
fa_status simt(const AttnGeom& g, const void* q, const void* k, const void* v, const void* o,
               const float* lse, const void* dout, void* dq, void* dk, void* dv, int dtype, const BmView& bm,
               const BmView& bmt, const MaskParams& mp, ScoreT s, void* ws, cudaStream_t st) {
  return bsimt::run_any(g, q, k, v, o, lse, dout, dq, dk, dv, dtype, bm, bmt, MaskFn<kMaskDynamic>{mp}, s, ws, st);
}

}  // namespace

bool bwd_sm100_supported(const AttnGeom& g) { return bwd::supported(g); }

fa_status launch_bwd_sm100(const AttnGeom& g, const void* q, const void* k, const void* v,
                           const void* o, const float* lse, const void* dout, void* dq, void* dk,
                           void* dv, const BmView& bm, const BmView& bmt, const MaskParams& mp,
                           int mkind, const ScoreParams& sp, int skind, void* workspace,
                           const BwdOptions& opt, cudaStream_t st) {
  if (g.D == 128)
    return by_score<128>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mp, mkind, sp, skind, workspace, opt, st);
  return by_score<64>(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mp, mkind, sp, skind, workspace, opt, st);
}

fa_status launch_bwd(const AttnGeom& g, const void* q, const void* k, const void* v,
                     const void* o, const float* lse, const void* dout, void* dq, void* dk,
                     void* dv, int dtype, const BmView& bm, const BmView& bmt,
                     const MaskParams& mp, int mkind, const ScoreParams& sp, int skind,
                     void* workspace, const BwdOptions& opt, cudaStream_t st) {
  if (dtype == FA_BF16 && bwd::supported(g))
    return launch_bwd_sm100(g, q, k, v, o, lse, dout, dq, dk, dv, bm, bmt, mp, mkind, sp, skind,
                            workspace, opt, st);
  // the CUDA-core passes are deterministic by construction (separate dq pass, no atomics)
  switch (skind) {
    case 0: return simt(g, q, k, v, o, lse, dout, dq, dk, dv, dtype, bm, bmt, mp, ScoreFn<0, true>{sp}, workspace, st);
    case 1: return simt(g, q, k, v, o, lse, dout, dq, dk, dv, dtype, bm, bmt, mp, ScoreFn<1, true>{sp}, workspace, st);
    case 2: return simt(g, q, k, v, o, lse, dout, dq, dk, dv, dtype, bm, bmt, mp, ScoreFn<2, true>{sp}, workspace, st);
    default: return simt(g, q, k, v, o, lse, dout, dq, dk, dv, dtype, bm, bmt, mp, ScoreFn<3, true>{sp}, workspace, st);
  }
}

}  // namespace fa
