// validate.cu — the library's instantiations of the work counters and the finiteness scan
// (include/flexattn_b200/validate.cuh) for the built-in mask functors, and fa_check_finite.
#include "internal.h"
#include "flexattn_b200/validate.cuh"

namespace fa {

fa_status counters_by_desc(const AttnGeom& a, const BmView& bm, const MaskParams& mp, int mkind,
                           const PageView* pv, int logical_kv, int pass, fa_op_counters* out,
                           cudaStream_t st) {
  switch (mkind) {
    case kMaskNoop: return compute_counters(a, bm, MaskFn<kMaskNoop>{mp}, pv, logical_kv, pass, out, st);
    case kMaskCausalOnly: return compute_counters(a, bm, MaskFn<kMaskCausalOnly>{mp}, pv, logical_kv, pass, out, st);
    case kMaskSlidingOnly: return compute_counters(a, bm, MaskFn<kMaskSlidingOnly>{mp}, pv, logical_kv, pass, out, st);
    case kMaskDocCausal: return compute_counters(a, bm, MaskFn<kMaskDocCausal>{mp}, pv, logical_kv, pass, out, st);
    default: return compute_counters(a, bm, MaskFn<kMaskDynamic>{mp}, pv, logical_kv, pass, out, st);
  }
}

fa_status check_finite(const fa_tensor* ts, const char* const* names, int n, cudaStream_t st) {
  return check_finite_list(ts, names, n, st);
}

}  // namespace fa

extern "C" fa_status fa_check_finite(const fa_tensor* tensors, const char* const* names, int32_t n,
                                     void* stream) {
  fa::clear_error();
  FA_REQUIRE(tensors != nullptr || n == 0, FA_SHAPE_MISMATCH, "check_finite: NULL tensors");
  return fa::check_finite_list(tensors, names, n, static_cast<cudaStream_t>(stream));
}
