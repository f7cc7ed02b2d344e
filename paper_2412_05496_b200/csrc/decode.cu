// decode.cu — the library's instantiations of the split-KV (paged) decode
// (include/flexattn_b200/decode.cuh) for the built-in mask/score functors.
#include "internal.h"
#include "flexattn_b200/dec_tc.cuh"
#include "flexattn_b200/decode.cuh"

namespace fa {
namespace {

struct TcCall {  // the tensor-core path's arguments (several rows per kv head)
  const DecodeGeom* g;
  const void *q, *k, *v;
  void* o;
  float* lse;
  const BmView* bm;
  const PageView* pv;
  void* ws;
};

template <class MaskT, class ScoreT>
fa_status run_one(const dec::DecParams& p, const TcCall* tc, MaskT m, ScoreT s, cudaStream_t st) {
  if (tc != nullptr) {
    if (tc->g->a.D == 128) return dectc::run<128>(*tc->g, tc->q, tc->k, tc->v, tc->o, tc->lse, *tc->bm, *tc->pv, tc->ws, m, s, st);
    return dectc::run<64>(*tc->g, tc->q, tc->k, tc->v, tc->o, tc->lse, *tc->bm, *tc->pv, tc->ws, m, s, st);
  }
  return dec::run_any_dim(p, m, s, st);
}

template <class ScoreT>
fa_status by_mask(const dec::DecParams& p, const TcCall* tc, const MaskParams& mp, int mk, ScoreT s, cudaStream_t st) {
  switch (mk) {
    case kMaskCausalOnly: return run_one(p, tc, MaskFn<kMaskCausalOnly>{mp}, s, st);
    case kMaskSlidingOnly: return run_one(p, tc, MaskFn<kMaskSlidingOnly>{mp}, s, st);
    default: return run_one(p, tc, MaskFn<kMaskDynamic>{mp}, s, st);
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
  // several query rows per kv head (GQA group and/or a multi-token step): packed into one
  // tensor-core tile so each page streams once per (batch element, kv head)
  const TcCall call{&g, q, k, v, o, lse, &bm, &pv, workspace};
  const TcCall* tc = dectc::supported(g) ? &call : nullptr;
  switch (skind) {
    case 0: return by_mask(p, tc, mp, mkind, ScoreFn<0>{sp}, st);
    case 1: return by_mask(p, tc, mp, mkind, ScoreFn<1>{sp}, st);
    case 2: return by_mask(p, tc, mp, mkind, ScoreFn<2>{sp}, st);
    default: return by_mask(p, tc, mp, mkind, ScoreFn<3>{sp}, st);
  }
}

}  // namespace fa
