// host.cuh — host-side plumbing shared by every launcher of the kernel templates: the
// thread-local error state and status helpers, launch accounting, small per-(device, stream)
// device scratch words, TMA tensor-map encoding, and the reference's argument checks
// (validate.cpp:16-34, engine.cpp:21-42). Header-only so that the library's C ABI and a user's
// own translation unit (flexattn_b200_device.cuh) share exactly the same code; each shared
// object that includes it gets its own error state and launch counter.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "../flexattn_b200.h"
#include "mods.cuh"

namespace fa {

// ---- error state ------------------------------------------------------------------------------
inline std::string& last_error_ref() {
  static thread_local std::string s;
  return s;
}
inline fa_status set_error(fa_status s, const std::string& msg) {
  last_error_ref() = msg;
  return s;
}
inline void clear_error() { last_error_ref().clear(); }
inline fa_status cuda_status(cudaError_t e, const char* what) {
  return set_error(FA_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

#define FA_CHECK_CUDA(expr)                                          \
  do {                                                               \
    cudaError_t e__ = (expr);                                        \
    if (e__ != cudaSuccess) return ::fa::cuda_status(e__, #expr);    \
  } while (0)

#define FA_REQUIRE(cond, status, msg)                                \
  do {                                                               \
    if (!(cond)) return ::fa::set_error((status), (msg));            \
  } while (0)

// ---- launch accounting, device facts, scratch words -----------------------------------------------
inline std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> n{0};
  return n;
}
inline void count_launch(uint64_t n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }

inline int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// 64 bytes of device scratch per (device, stream, slot): work counters of the persistent
// kernels and device status flags. The launcher zeroes a word on the stream right before the
// kernel, so launches on one stream are ordered and launches on different streams never share
// a word.
enum { kSlotFwdSched = 0, kSlotBwdSched = 1, kSlotConvertErr = 2, kSlotFiniteErr = 3, kSlotCounters = 4, kSlotDqSched = 5 };
inline int* scheduler_counter(int slot, cudaStream_t st) {
  static std::map<std::tuple<int, cudaStream_t, int>, int*> counters;
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  int*& c = counters[std::make_tuple(dev, st, slot)];
  if (c == nullptr && cudaMalloc(&c, 64) != cudaSuccess) c = nullptr;
  return c;
}

// passes of compute_counters (validate.cuh)
enum { kPassForward = 0, kPassBackward = 1 };

// ---- problem geometry shared by the launchers ------------------------------------------------------
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

// Backward options beyond the tensors (ABI v3 fields of fa_bwd_args).
struct BwdOptions {
  uint32_t flags = 0;               // FA_FLAG_*
  cudaEvent_t events[4] = {nullptr, nullptr, nullptr, nullptr};  // phase timing, may be null
  int* dout_nonfinite = nullptr;    // device word set by the preprocess when d_out has NaN/inf
};

// ---- workspace sizes (fa_bwd_workspace_size / fa_decode_workspace_size) ------------------------------
inline size_t bwd_workspace_bytes(int64_t batch, int64_t heads, int64_t q_len, int64_t dim) {
  // dq accumulator (fp32) + delta (fp32) + log2-domain lse (fp32) + one reserved int per
  // (b, h, q block) (kept so the size stays ABI-stable), 256-byte aligned pieces
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t rows = static_cast<size_t>(batch * heads * q_len);
  const size_t prow = static_cast<size_t>(batch * heads * ((q_len + 127) / 128 * 128));
  const size_t qblocks = static_cast<size_t>(batch * heads * ((q_len + 127) / 128));
  return al(rows * dim * 4) + al(prow * 4) + al(prow * 4) + al(qblocks * 4);
}
inline size_t decode_workspace_bytes(int64_t batch, int64_t heads, int64_t n_new, int64_t dim, int32_t num_splits) {
  if (num_splits <= 1) num_splits = 64;  // upper bound of the automatic choice
  return static_cast<size_t>(batch * heads * n_new) * num_splits * (dim + 2) * 4;
}

// ---- TMA tensor maps --------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// 3-D map over a (BH, L, D) bf16 tensor with a (64, box_rows, 1) box and 128-byte swizzle: the
// operand tiles of the tensor-core kernels (box_rows 128) and the target of TMA stores.
inline CUresult encode_store_map(CUtensorMap* map, const void* base, int bh, int len, int d, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (enc == nullptr) return CUDA_ERROR_NOT_SUPPORTED;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(len), static_cast<cuuint64_t>(bh)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * 2, static_cast<cuuint64_t>(len) * d * 2};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}
// 3-D map over a (BH, L, D) bf16 tensor with a (32, 32, 1) box and 64-byte swizzle: the forward's
// epilogue stores O through it, 32 rows x 32 columns per warp (rows past L are clipped).
inline CUresult encode_o32_map(CUtensorMap* map, const void* base, int bh, int len, int d) {
  EncodeTiledFn enc = get_encode();
  if (enc == nullptr) return CUDA_ERROR_NOT_SUPPORTED;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(len), static_cast<cuuint64_t>(bh)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * 2, static_cast<cuuint64_t>(len) * d * 2};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}
inline CUresult encode_tile_map(CUtensorMap* map, const void* base, int bh, int len, int d) {
  return encode_store_map(map, base, bh, len, d, 128);
}
inline fa_status make_map(CUtensorMap* map, const void* base, int bh, int len, int d) {
  FA_REQUIRE(get_encode() != nullptr, FA_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  const CUresult r = encode_tile_map(map, base, bh, len, d);
  FA_REQUIRE(r == CUDA_SUCCESS, FA_CUDA_ERROR,
             "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return FA_OK;
}

// 3-D map over a (BH, L, D) fp32 tensor with a (box_d, box_rows, 1) box and no swizzle: the
// target of the backward's TMA reduce-add of dQ (rows past L are clipped per head).
inline CUresult encode_f32_map(CUtensorMap* map, const void* base, int bh, int len, int d, int box_d,
                               int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (enc == nullptr) return CUDA_ERROR_NOT_SUPPORTED;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(len), static_cast<cuuint64_t>(bh)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * 4, static_cast<cuuint64_t>(len) * d * 4};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_d), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// ---- the reference's argument checks (errors.hpp taxonomy) ------------------------------------------
inline fa_status check_tensor(const fa_tensor& t, const char* name) {
  FA_REQUIRE(t.data != nullptr, FA_SHAPE_MISMATCH, std::string(name) + ": NULL data");
  FA_REQUIRE(t.b > 0 && t.h > 0 && t.l > 0 && t.d > 0, FA_SHAPE_MISMATCH,
             std::string(name) + ": all dims must be positive");
  FA_REQUIRE(t.dtype == FA_F32 || t.dtype == FA_BF16, FA_UNSUPPORTED,
             std::string(name) + ": dtype must be FA_F32 or FA_BF16");
  return FA_OK;
}

inline bool same_shape(const fa_tensor& a, const fa_tensor& b) {
  return a.b == b.b && a.h == b.h && a.l == b.l && a.d == b.d;
}

inline std::string shp(const fa_tensor& t) {
  return "(" + std::to_string(t.b) + "," + std::to_string(t.h) + "," + std::to_string(t.l) + "," +
         std::to_string(t.d) + ")";
}

// validate_shapes (validate.cpp:16-34) + gqa divisibility (config.hpp:33-45)
inline fa_status check_qkv(const fa_tensor& q, const fa_tensor& k, const fa_tensor& v, int64_t gqa) {
  fa_status s;
  if ((s = check_tensor(q, "q")) || (s = check_tensor(k, "k")) || (s = check_tensor(v, "v"))) return s;
  FA_REQUIRE(k.b == v.b && k.h == v.h && k.l == v.l && k.d == v.d, FA_SHAPE_MISMATCH,
             "k " + shp(k) + " and v " + shp(v) + " must have the same shape");
  FA_REQUIRE(q.d == k.d, FA_SHAPE_MISMATCH, "q head dim must match k");
  FA_REQUIRE(k.b == 1 || k.b == q.b, FA_SHAPE_MISMATCH, "kv batch must be 1 or the q batch");
  FA_REQUIRE(gqa >= 1, FA_SHAPE_MISMATCH, "gqa_group must be >= 1");
  FA_REQUIRE(q.h == gqa * k.h, FA_SHAPE_MISMATCH,
             "q heads " + std::to_string(q.h) + " != gqa_group * kv heads " + std::to_string(gqa * k.h));
  FA_REQUIRE(q.dtype == k.dtype && k.dtype == v.dtype, FA_SHAPE_MISMATCH, "q/k/v dtypes differ");
  return FA_OK;
}

// check_block_mask (engine.cpp:21-42)
inline fa_status check_bm(const fa_block_mask* bm, int64_t batch, int64_t heads, int64_t q_len, int64_t kv_len) {
  FA_REQUIRE(bm != nullptr && bm->kv_num_blocks && bm->kv_indices && bm->full_kv_num_blocks && bm->full_kv_indices,
             FA_BLOCK_MASK_MISMATCH, "block mask kv-side arrays missing");
  FA_REQUIRE(bm->q_len == q_len && bm->kv_len == kv_len, FA_BLOCK_MASK_MISMATCH,
             "block mask covers " + std::to_string(bm->q_len) + "x" + std::to_string(bm->kv_len) +
                 " but tensors are " + std::to_string(q_len) + "x" + std::to_string(kv_len));
  FA_REQUIRE(bm->b_dims == 1 || bm->b_dims == batch, FA_BLOCK_MASK_MISMATCH,
             "block mask batch dim must be 1 or " + std::to_string(batch));
  FA_REQUIRE(bm->h_dims == 1 || bm->h_dims == heads, FA_BLOCK_MASK_MISMATCH,
             "block mask head dim must be 1 or " + std::to_string(heads));
  FA_REQUIRE(bm->rows == (bm->q_len + bm->bs_q - 1) / bm->bs_q && bm->cols == (bm->kv_len + bm->bs_kv - 1) / bm->bs_kv,
             FA_BLOCK_MASK_MISMATCH, "block mask rows/cols inconsistent with lengths");
  return FA_OK;
}

inline AttnGeom geom_of(const fa_tensor& q, const fa_tensor& k, const fa_block_mask* bm, double scale,
                        int64_t gqa) {
  AttnGeom g{};
  g.B = (int)q.b; g.Hq = (int)q.h; g.Hkv = (int)k.h; g.Bkv = (int)k.b; g.Lq = (int)q.l;
  g.Lkv = (int)k.l; g.D = (int)q.d; g.G = (int)gqa;
  g.bm_b = (int)bm->b_dims; g.bm_h = (int)bm->h_dims; g.rows = (int)bm->rows; g.cols = (int)bm->cols;
  g.bs_q = (int)bm->bs_q; g.bs_kv = (int)bm->bs_kv;
  g.scale = static_cast<float>(scale > 0 ? scale : 1.0 / std::sqrt(static_cast<double>(q.d)));
  return g;
}

inline BmView kv_view(const fa_block_mask* bm) {
  return BmView{bm->kv_num_blocks, bm->kv_indices, bm->full_kv_num_blocks, bm->full_kv_indices};
}
inline BmView q_view(const fa_block_mask* bm) {
  return BmView{bm->q_num_blocks, bm->q_indices, bm->full_q_num_blocks, bm->full_q_indices};
}

}  // namespace fa
