// fwd_sm100.cu — the library's instantiations of the tensor-core forward
// (include/flexattn_b200/fwd_sm100.cuh) for the built-in mask/score functors.
#include "internal.h"
#include "flexattn_b200/fwd1t.cuh"
#include "flexattn_b200/fwd_sm100.cuh"

#ifndef FA_FWD_1T
#define FA_FWD_1T 0  // 1: the one-tile forward (fwd1t.cuh) instead of the two-tile ping-pong
#endif

namespace fa {
namespace {

template <int D, class MaskT, class ScoreT>
fa_status run_fwd(const AttnGeom& g, const void* q, const void* k, const void* v, void* o, float* lse,
                  const BmView& bm, MaskT mask, ScoreT score, cudaStream_t st) {
  // rows longer than the two-tile kernel's smem visit list (KV_LEN > 131072) take the one-tile
  // kernel, which streams the lists from global memory
  if (FA_FWD_1T != 0 || !fwd::supported(g)) return fwd1t::run<D>(g, q, k, v, o, lse, bm, mask, score, st);
  return fwd::run<D>(g, q, k, v, o, lse, bm, mask, score, st);
}

template <int D, class ScoreT>
fa_status by_mask(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                  float* lse, const BmView& bm, const MaskParams& mp, int mk, ScoreT s,
                  cudaStream_t st) {
  switch (mk) {
    case kMaskNoop: return run_fwd<D>(g, q, k, v, o, lse, bm, MaskFn<kMaskNoop>{mp}, s, st);
    case kMaskCausalOnly: return run_fwd<D>(g, q, k, v, o, lse, bm, MaskFn<kMaskCausalOnly>{mp}, s, st);
    case kMaskSlidingOnly: return run_fwd<D>(g, q, k, v, o, lse, bm, MaskFn<kMaskSlidingOnly>{mp}, s, st);
    case kMaskDocCausal: return run_fwd<D>(g, q, k, v, o, lse, bm, MaskFn<kMaskDocCausal>{mp}, s, st);
    default: return run_fwd<D>(g, q, k, v, o, lse, bm, MaskFn<kMaskDynamic>{mp}, s, st);
  }
}

template <int D>
fa_status by_score(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                   float* lse, const BmView& bm, const MaskParams& mp, int mk,
                   const ScoreParams& sp, int sk, cudaStream_t st) {
  switch (sk) {
    case 0: return by_mask<D>(g, q, k, v, o, lse, bm, mp, mk, ScoreFn<0>{sp}, st);
    case 1: return by_mask<D>(g, q, k, v, o, lse, bm, mp, mk, ScoreFn<1>{sp}, st);
    case 2: return by_mask<D>(g, q, k, v, o, lse, bm, mp, mk, ScoreFn<2>{sp}, st);
    default: return by_mask<D>(g, q, k, v, o, lse, bm, mp, mk, ScoreFn<3>{sp}, st);
  }
}

}  // namespace

bool fwd_sm100_supported(const AttnGeom& g) { return fwd::supported(g) || fwd1t::supported(g); }

fa_status launch_fwd_sm100(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                           float* lse, const BmView& bm, const MaskParams& mp, int mkind,
                           const ScoreParams& sp, int skind, cudaStream_t st) {
  if (g.D == 128) return by_score<128>(g, q, k, v, o, lse, bm, mp, mkind, sp, skind, st);
  return by_score<64>(g, q, k, v, o, lse, bm, mp, mkind, sp, skind, st);
}

}  // namespace fa
