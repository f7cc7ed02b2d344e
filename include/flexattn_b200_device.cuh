// flexattn_b200_device.cuh — the templated entry points for USER mask_mod / score_mod
// functors: the reference's any-callable modifiers (modifiers.hpp:17-40, compose :57-66)
// reach the same sm100a kernels as the built-in ones (include/flexattn_b200/*.cuh), compiled in
// the user's own nvcc translation unit (-gencode arch=compute_100a,code=sm_100a -std=c++17
// --expt-relaxed-constexpr -I include). Header-only: no link dependency on libflexattn_b200.
//
//   A mask functor:   struct M { __device__ bool operator()(int b, int h, int q, int kv) const; };
//   A score functor:  struct S {
//                       __device__ float apply(float s, int b, int h, int q, int kv) const;  // s scaled
//                       __device__ float grad(float s, int b, int h, int q, int kv) const;   // d apply / d s
//                       // optional: static constexpr bool kUnitGrad = true;  (grad == 1 everywhere)
//                     };
//   Both see the already-scaled score and absolute positions; `grad` is the
//   backward's score_mod' (modifiers.hpp:25-28). Functors are passed by value to the kernels, so
//   they hold plain values and device pointers only.
//
//   create_block_mask(mask, b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, bm, ws, ws_bytes, stream)
//                                                 <- create_block_mask + transpose (block_mask.hpp:109-115)
//   flex_attention(args, score, mask, stream)     <- forward<Real>  (engine.hpp:68-71)
//   flex_attention_backward(args, score, mask, stream)  <- backward<Real> (engine.hpp:78-82)
//   flex_decode(args, score, mask, stream)        <- decode<Real>   (engine.hpp:92-96)
// The argument structs are the C ABI's (flexattn_b200.h); their mask/score descriptor fields are
// ignored. Status codes and messages are the C ABI's (flexattn::device::last_error()).
#pragma once

#include "flexattn_b200.h"
#include "flexattn_b200/entry.cuh"

namespace flexattn {
namespace device {

namespace detail {
template <class T, class = void>
struct unit_grad : std::false_type {};
template <class T>
struct unit_grad<T, std::void_t<decltype(T::kUnitGrad)>> : std::integral_constant<bool, T::kUnitGrad> {};
}  // namespace detail

// A user mask as the kernels' mask interface (fa::MaskFn): no closed form over tiles, so the
// BlockMask builder evaluates every tile (with the reference's early exit on mixed tiles), and
// word-level evaluation calls the functor per position. `q_offset` shifts q (offset_mask,
// mask_library.cpp:106-110; used by decode).
template <class F>
struct UserMask {
  F f;
  int q_offset = 0;
  __device__ __forceinline__ bool operator()(int b, int h, int q, int kv) const { return f(b, h, q + q_offset, kv); }
  __device__ __forceinline__ int tile_class(int, int, int, int, int, int, int) const { return fa::kTileMixed; }
  __device__ __forceinline__ uint32_t bits32(int b, int h, int q, int kv0, int kv_lim) const {
    return fa::mask_bits32_generic(*this, b, h, q, kv0, kv_lim);
  }
  __device__ __forceinline__ uint32_t bits32_q(int b, int h, int q0, int kv, int q_lim) const {
    uint32_t bits = 0;
#pragma unroll 4
    for (int i = 0; i < 32; ++i)
      if (q0 + i < q_lim) bits |= static_cast<uint32_t>((*this)(b, h, q0 + i, kv)) << i;
    return bits;
  }
};

// A user score as the kernels' score interface (fa::ScoreFn): the generic kind (not the
// ALiBi / plain fast paths), the log2-domain row / column contexts evaluate the functor per score.
template <class F>
struct UserScore {
  F f;
  int q_offset = 0;  // offset_score (mask_library.cpp:112-119; used by decode)
  static constexpr bool kIdentity = false;
  static constexpr int kKind = 4;  // generic: log2_grad per score in the backward
  static constexpr bool kUnitGrad = detail::unit_grad<F>::value;
  __device__ __forceinline__ float apply(float s, int b, int h, int q, int kv) const {
    return f.apply(s, b, h, q + q_offset, kv);
  }
  __device__ __forceinline__ float grad(float s, int b, int h, int q, int kv) const {
    return f.grad(s, b, h, q + q_offset, kv);
  }
  // positions (q + dq * i, kv + dkv * i) for the i-th score of a row (dq 0, dkv 1) or of a
  // column (dq 1, dkv 0) of a tile
  struct Row {
    F f;
    int b, h, q, kv, dq, dkv;
    float scale;
    float c = 1.f;  // unused (the plain-score path only)
    __device__ __forceinline__ Row shifted(int off) const {
      Row r = *this;
      r.q += dq * off;
      r.kv += dkv * off;
      return r;
    }
    __device__ __forceinline__ float log2(float s_raw, int i) const {
      return 1.4426950408889634f * f.apply(s_raw * scale, b, h, q + dq * i, kv + dkv * i);
    }
    __device__ __forceinline__ float log2_grad(float s_raw, int i, float& g) const {
      const float s = s_raw * scale;
      g = kUnitGrad ? 1.f : f.grad(s, b, h, q + dq * i, kv + dkv * i);
      return 1.4426950408889634f * f.apply(s, b, h, q + dq * i, kv + dkv * i);
    }
  };
  __device__ __forceinline__ Row row(int b, int h, int q, int kv0, float scale) const {
    return Row{f, b, h, q + q_offset, kv0, 0, 1, scale};
  }
  __device__ __forceinline__ Row col(int b, int h, int q0, int kv, float scale) const {
    return Row{f, b, h, q0 + q_offset, kv, 1, 0, scale};
  }
};

inline const char* last_error() { return fa::last_error_ref().c_str(); }

// create_block_mask + transpose for a user mask (bm's arrays caller-allocated, sizes from
// fa_block_mask_geometry; q-side arrays filled when non-NULL)
template <class Mask>
fa_status create_block_mask(const Mask& mask, int64_t b_dims, int64_t h_dims, int64_t q_len, int64_t kv_len,
                            int64_t bs_q, int64_t bs_kv, fa_block_mask* bm, void* workspace, size_t workspace_bytes,
                            cudaStream_t stream) {
  fa::clear_error();
  return fa::bmk::build(UserMask<Mask>{mask}, b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, bm, workspace,
                        workspace_bytes, stream);
}

template <class Score, class Mask>
fa_status flex_attention(const fa_fwd_args& args, const Score& score, const Mask& mask, cudaStream_t stream) {
  fa::clear_error();
  return fa::flex_fwd_t(&args, UserMask<Mask>{mask}, UserScore<Score>{score}, stream);
}

template <class Score, class Mask>
fa_status flex_attention_backward(const fa_bwd_args& args, const Score& score, const Mask& mask,
                                  cudaStream_t stream) {
  fa::clear_error();
  return fa::flex_bwd_t(&args, UserMask<Mask>{mask}, UserScore<Score>{score}, stream);
}

// decode rows [offset, offset + n_new): the functors see absolute positions (the offset shift
// is applied here, engine.cpp:421-424)
template <class Score, class Mask>
fa_status flex_decode(const fa_decode_args& args, const Score& score, const Mask& mask, cudaStream_t stream) {
  fa::clear_error();
  fa::DecodePlan plan;
  fa_status s = fa::prepare_decode(&args, &plan, stream);
  if (s != FA_OK) return s;
  const int off = static_cast<int>(args.offset);
  return fa::flex_decode_t(&args, plan, UserMask<Mask>{mask, off}, UserScore<Score>{score, off}, stream);
}

}  // namespace device
}  // namespace flexattn
