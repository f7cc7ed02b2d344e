// decode.cu — the library's instantiations of the split-KV (paged) decode
// (include/flexattn_b200/decode.cuh) for the built-in mask/score functors.
#include "internal.h"
#include "flexattn_b200/decode.cuh"

namespace fa {
namespace {

template <class ScoreT>
fa_status by_mask(const dec::DecParams& p, const MaskParams& mp, int mk, ScoreT s, cudaStream_t st) {
  switch (mk) {
    case kMaskCausalOnly: return dec::run_any_dim(p, MaskFn<kMaskCausalOnly>{mp}, s, st);
    case kMaskSlidingOnly: return dec::run_any_dim(p, MaskFn<kMaskSlidingOnly>{mp}, s, st);
    default: return dec::run_any_dim(p, MaskFn<kMaskDynamic>{mp}, s, st);
  }
}

}  // namespace

fa_status launch_decode(const DecodeGeom& g, const void* q, const void* k, const void* v, void* o,
                        float* lse, const BmView& bm, const PageView& pv, const MaskParams& mp,
                        int mkind, const ScoreParams& sp, int skind, void* workspace,
                        cudaStream_t st) {
  dec::DecParams p{};
  fa_status s = dec::make_params(g, q, k, v, o, lse, bm, pv, workspace, &p);
  if (s != FA_OK) return s;
  switch (skind) {
    case 0: return by_mask(p, mp, mkind, ScoreFn<0>{sp}, st);
    case 1: return by_mask(p, mp, mkind, ScoreFn<1>{sp}, st);
    case 2: return by_mask(p, mp, mkind, ScoreFn<2>{sp}, st);
    default: return by_mask(p, mp, mkind, ScoreFn<3>{sp}, st);
  }
}

}  // namespace fa
