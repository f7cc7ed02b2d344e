// custom_mods.cu — a USER translation unit instantiating the sm100a kernels with its own
// __device__ mask_mod / score_mod functors through include/flexattn_b200_device.cuh (the
// reference's any-callable modifiers, modifiers.hpp:17-40). Built by __graft_entry__.build()
// into tests/cpp/libcustom_mods.so and driven from tests/test_gpu_custom_mods.py, which checks
// it against a dense fp32 restatement of the same functors.
//
//   mask  "window + global columns": q >= kv && (q - kv < window || kv % stride == 0)
//   score per-head soft cap over a relative-position bias (T5-style clipped distance table):
//         apply(s) = cap[h] * tanh((s + bias[clip(q - kv, 0, R)]) / cap[h])
//         grad(s)  = 1 - tanh^2((s + bias[...]) / cap[h])
#include <cuda_runtime.h>

#include "flexattn_b200_device.cuh"

namespace user {

struct WindowGlobal {
  int window, stride;
  __device__ bool operator()(int, int, int q, int kv) const {
    return q >= kv && (q - kv < window || kv % stride == 0);
  }
};

struct CappedRelBias {
  const float* bias;  // [R + 1]
  const float* cap;   // [heads]
  int R;
  __device__ float apply(float s, int, int h, int q, int kv) const {
    const int d = min(max(q - kv, 0), R);
    const float c = __ldg(cap + h);
    return c * tanhf((s + __ldg(bias + d)) / c);
  }
  __device__ float grad(float s, int, int h, int q, int kv) const {
    const int d = min(max(q - kv, 0), R);
    const float c = __ldg(cap + h);
    const float t = tanhf((s + __ldg(bias + d)) / c);
    return 1.f - t * t;
  }
};

// A unit-gradient score: the relative-position bias alone (kUnitGrad skips grad in the backward).
struct RelBias {
  const float* bias;
  int R;
  static constexpr bool kUnitGrad = true;
  __device__ float apply(float s, int, int, int q, int kv) const { return s + __ldg(bias + min(max(q - kv, 0), R)); }
  __device__ float grad(float, int, int, int, int) const { return 1.f; }
};

}  // namespace user

namespace dev = flexattn::device;

extern "C" {

const char* cm_last_error(void) { return dev::last_error(); }

int cm_create_block_mask(int window, int stride, int64_t q_len, int64_t kv_len, int64_t bs, fa_block_mask* bm,
                         void* ws, size_t ws_bytes, void* stream) {
  return dev::create_block_mask(user::WindowGlobal{window, stride}, 1, 1, q_len, kv_len, bs, bs, bm, ws, ws_bytes,
                                static_cast<cudaStream_t>(stream));
}

int cm_forward(const fa_fwd_args* a, int window, int stride, const float* bias, const float* cap, int R, int unit,
               void* stream) {
  const user::WindowGlobal m{window, stride};
  if (unit) return dev::flex_attention(*a, user::RelBias{bias, R}, m, static_cast<cudaStream_t>(stream));
  return dev::flex_attention(*a, user::CappedRelBias{bias, cap, R}, m, static_cast<cudaStream_t>(stream));
}

int cm_backward(const fa_bwd_args* a, int window, int stride, const float* bias, const float* cap, int R, int unit,
                void* stream) {
  const user::WindowGlobal m{window, stride};
  if (unit) return dev::flex_attention_backward(*a, user::RelBias{bias, R}, m, static_cast<cudaStream_t>(stream));
  return dev::flex_attention_backward(*a, user::CappedRelBias{bias, cap, R}, m, static_cast<cudaStream_t>(stream));
}

int cm_decode(const fa_decode_args* a, int window, int stride, const float* bias, const float* cap, int R,
              void* stream) {
  return dev::flex_decode(*a, user::CappedRelBias{bias, cap, R}, user::WindowGlobal{window, stride},
                          static_cast<cudaStream_t>(stream));
}

}  // extern "C"
