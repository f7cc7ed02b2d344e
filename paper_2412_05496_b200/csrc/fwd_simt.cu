// fwd_simt.cu — the library's instantiations of the CUDA-core forward
// (include/flexattn_b200/fwd_simt.cuh) for the built-in mask/score functors.
#include "internal.h"
#include "flexattn_b200/fwd_simt.cuh"

namespace fa {
namespace {

template <typename T, class ScoreT>
fa_status by_mask(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                  float* lse, const BmView& bm, const MaskParams& mp, int mk, ScoreT s,
                  cudaStream_t st) {
  switch (mk) {
    case kMaskCausalOnly: return fsimt::run_any_dim<T>(g, q, k, v, o, lse, bm, MaskFn<kMaskCausalOnly>{mp}, s, st);
    default: return fsimt::run_any_dim<T>(g, q, k, v, o, lse, bm, MaskFn<kMaskDynamic>{mp}, s, st);
  }
}

template <typename T>
fa_status by_score(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                   float* lse, const BmView& bm, const MaskParams& mp, int mk,
                   const ScoreParams& sp, int sk, cudaStream_t st) {
  switch (sk) {
    case 0: return by_mask<T>(g, q, k, v, o, lse, bm, mp, mk, ScoreFn<0, true>{sp}, st);
    case 1: return by_mask<T>(g, q, k, v, o, lse, bm, mp, mk, ScoreFn<1, true>{sp}, st);
    case 2: return by_mask<T>(g, q, k, v, o, lse, bm, mp, mk, ScoreFn<2, true>{sp}, st);
    default: return by_mask<T>(g, q, k, v, o, lse, bm, mp, mk, ScoreFn<3, true>{sp}, st);
  }
}

}  // namespace

fa_status launch_fwd_simt(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                          float* lse, int dtype, const BmView& bm, const MaskParams& mp,
                          int mkind, const ScoreParams& sp, int skind, cudaStream_t st) {
  if (dtype == FA_F32) return by_score<float>(g, q, k, v, o, lse, bm, mp, mkind, sp, skind, st);
  return by_score<__nv_bfloat16>(g, q, k, v, o, lse, bm, mp, mkind, sp, skind, st);
}

}  // namespace fa
