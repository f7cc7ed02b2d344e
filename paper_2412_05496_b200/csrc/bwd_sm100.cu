// bwd_sm100.cu — tensor-core backward (placeholder until the tcgen05 kernel lands).
#include "internal.h"

namespace fa {

bool bwd_sm100_supported(const AttnGeom& g) {
  (void)g;
  return false;
}

fa_status launch_bwd_sm100(const AttnGeom&, const void*, const void*, const void*, const void*,
                           const float*, const void*, void*, void*, void*, const BmView&,
                           const BmView&, const MaskParams&, int, const ScoreParams&, int, void*,
                           cudaStream_t) {
  return set_error(FA_UNSUPPORTED, "tcgen05 backward not built");
}

}  // namespace fa
