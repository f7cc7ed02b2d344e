// internal.h — host-side plumbing shared by the C-ABI translation units:
// thread-local error state, status helpers, launch accounting and the
// internal launcher signatures (templates cannot cross the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/flexattn_b200.h"
#include "mods.cuh"

namespace fa {

fa_status set_error(fa_status s, const std::string& msg);
void clear_error();
fa_status cuda_status(cudaError_t e, const char* what);
void count_launch(uint64_t n = 1);
int num_sms();
// 64 bytes of device scratch per (device, stream, slot): work counters of the persistent
// kernels and device status flags. Slots:
enum { kSlotFwdSched = 0, kSlotBwdSched = 1, kSlotConvertErr = 2, kSlotFiniteErr = 3, kSlotCounters = 4 };
int* scheduler_counter(int slot, cudaStream_t st);

#define FA_CHECK_CUDA(expr)                                          \
  do {                                                               \
    cudaError_t e__ = (expr);                                        \
    if (e__ != cudaSuccess) return ::fa::cuda_status(e__, #expr);    \
  } while (0)

#define FA_REQUIRE(cond, status, msg)                                \
  do {                                                               \
    if (!(cond)) return ::fa::set_error((status), (msg));            \
  } while (0)

// Host mirror of the descriptors (validated, device pointers).
MaskParams to_mask_params(const fa_mask_desc& d);
ScoreParams to_score_params(const fa_score_desc& d);
// Pick the specialised kernel kind for a mask (kMaskDynamic if none matches).
int mask_kind_of(const fa_mask_desc& d);
// Reference-equivalent checks of a mask descriptor for q in [0, q_len), kv in [0, kv_len).
fa_status check_mask_desc(const fa_mask_desc& m, int64_t q_len, int64_t kv_len);

// Geometry of the forward problem, shared by the launchers.
struct AttnGeom {
  int B, Hq, Hkv, Bkv, Lq, Lkv, D, G;
  int bm_b, bm_h, rows, cols, bs_q, bs_kv;
  float scale;
};

struct BmView {
  const int32_t* kv_num;
  const int32_t* kv_idx;
  const int32_t* full_num;
  const int32_t* full_idx;
};

fa_status launch_fwd_simt(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                          float* lse, int dtype, const BmView& bm, const MaskParams& mp,
                          int mkind, const ScoreParams& sp, int skind, cudaStream_t st);

bool fwd_sm100_supported(const AttnGeom& g);
fa_status launch_fwd_sm100(const AttnGeom& g, const void* q, const void* k, const void* v, void* o,
                           float* lse, const BmView& bm, const MaskParams& mp, int mkind,
                           const ScoreParams& sp, int skind, cudaStream_t st);

struct DecodeGeom {
  AttnGeom a;        // Lq = n_new, Lkv = cache length (physical when paged)
  int num_splits;
  int logical_kv;    // kv bound in logical coordinates (cache length / seq_len source)
};
struct PageView {
  const int32_t* phys_to_logical;
  const int32_t* owner;
  const int32_t* seq_len;
  int page_size;
  int enabled;
  int* foreign = nullptr;  // device word set when a visited page is not the row's batch element's
};

fa_status launch_decode(const DecodeGeom& g, const void* q, const void* k, const void* v, void* o,
                        float* lse, const BmView& bm, const PageView& pv, const MaskParams& mp,
                        int mkind, const ScoreParams& sp, int skind, void* workspace,
                        cudaStream_t st);

// OpCounters of one call (engine.hpp:21-32) from the BlockMask and the mask; synchronises `st`.
enum { kPassForward = 0, kPassBackward = 1 };
fa_status compute_counters(const AttnGeom& a, const BmView& bm, const MaskParams& mp, int mkind,
                           const PageView* pv, int logical_kv, int pass, fa_op_counters* out,
                           cudaStream_t st);
// NaN/inf scan of n tensors (validate.hpp:36-38); synchronises `st`.
fa_status check_finite_list(const fa_tensor* ts, const char* const* names, int n, cudaStream_t st);

// Backward options beyond the tensors (ABI v3 fields of fa_bwd_args).
struct BwdOptions {
  uint32_t flags = 0;               // FA_FLAG_*
  cudaEvent_t events[4] = {nullptr, nullptr, nullptr, nullptr};  // phase timing, may be null
  int* dout_nonfinite = nullptr;    // device word set by the preprocess when d_out has NaN/inf
};

bool bwd_sm100_supported(const AttnGeom& g);
fa_status launch_bwd(const AttnGeom& g, const void* q, const void* k, const void* v,
                     const void* o, const float* lse, const void* dout, void* dq, void* dk,
                     void* dv, int dtype, const BmView& bm, const BmView& bmt,
                     const MaskParams& mp, int mkind, const ScoreParams& sp, int skind,
                     void* workspace, const BwdOptions& opt, cudaStream_t st);

}  // namespace fa
