// internal.h — declarations shared by the C-ABI translation units of the library: the
// descriptor (fa_mask_desc / fa_score_desc) plumbing and the descriptor-dispatched launchers,
// i.e. the library's own instantiations of the kernel templates in include/flexattn_b200/
// for the built-in mask/score functors (templates cannot cross the C ABI). A user functor
// reaches the same kernel templates through include/flexattn_b200_device.cuh instead.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "flexattn_b200/host.cuh"
#include "flexattn_b200/mods.cuh"

namespace fa {

// Host mirror of the descriptors (validated, device pointers).
MaskParams to_mask_params(const fa_mask_desc& d);
ScoreParams to_score_params(const fa_score_desc& d);
// Pick the specialised kernel kind for a mask (kMaskDynamic if none matches).
int mask_kind_of(const fa_mask_desc& d);
// Reference-equivalent checks of a mask descriptor for q in [0, q_len), kv in [0, kv_len).
fa_status check_mask_desc(const fa_mask_desc& m, int64_t q_len, int64_t kv_len);

fa_status launch_fwd_simt(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                          float* lse, int dtype, const BmView& bm, const MaskParams& mp,
                          int mkind, const ScoreParams& sp, int skind, cudaStream_t st);
bool fwd_sm100_supported(const AttnGeom& g);
fa_status launch_fwd_sm100(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                           float* lse, const BmView& bm, const MaskParams& mp, int mkind,
                           const ScoreParams& sp, int skind, cudaStream_t st);
fa_status launch_decode(const DecodeGeom& g, const void* q, const void* k, const void* v, void* o,
                        float* lse, const BmView& bm, const PageView& pv, const MaskParams& mp,
                        int mkind, const ScoreParams& sp, int skind, void* workspace,
                        cudaStream_t st);
bool bwd_sm100_supported(const AttnGeom& g);
fa_status launch_bwd_sm100(const AttnGeom& g, const void* q, const void* k, const void* v,
                           const void* o, const float* lse, const void* dout, void* dq, void* dk,
                           void* dv, const BmView& bm, const BmView& bmt, const MaskParams& mp,
                           int mkind, const ScoreParams& sp, int skind, void* workspace,
                           const BwdOptions& opt, cudaStream_t st);
fa_status launch_bwd(const AttnGeom& g, const void* q, const void* k, const void* v,
                     const void* o, const float* lse, const void* dout, void* dq, void* dk,
                     void* dv, int dtype, const BmView& bm, const BmView& bmt,
                     const MaskParams& mp, int mkind, const ScoreParams& sp, int skind,
                     void* workspace, const BwdOptions& opt, cudaStream_t st);

// OpCounters of one call (engine.hpp:21-32) for a descriptor mask; synchronises `st`.
// pass: 0 forward / decode, 1 backward.
fa_status counters_by_desc(const AttnGeom& a, const BmView& bm, const MaskParams& mp, int mkind,
                           const PageView* pv, int logical_kv, int pass, fa_op_counters* out,
                           cudaStream_t st);
// NaN/inf scan of n tensors (validate.hpp:36-38); synchronises `st`.
fa_status check_finite(const fa_tensor* ts, const char* const* names, int n, cudaStream_t st);

}  // namespace fa
