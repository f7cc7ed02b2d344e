// flexattn_b200.hpp — C++ host API mirroring the reference's blockattn API
// (/root/reference/proj/include/blockattn/*.hpp) over the C ABI in flexattn_b200.h.
//
// Header-only. Same names and argument meaning as the reference, so a blockattn user
// switches by changing the namespace and moving tensors to the device:
//
//   blockattn::create_block_mask(mask, b, h, q, kv, bsq, bskv)  block_mask.hpp:109-110
//   blockattn::transpose(bm)                                   block_mask.hpp:115
//   blockattn::forward<Real>(q, k, v, smod, bm, cfg)            engine.hpp:68-71
//   blockattn::backward<Real>(q, k, v, fwd, dout, smod, bm, bm_t, cfg) engine.hpp:78-82
//   blockattn::decode<Real>(q, k, v, offset, mask, smod, bm, cfg)      engine.hpp:92-96
//   blockattn::convert_block_mask(bm, page_table)               paged_kv.hpp:101
//   blockattn::convert_mods(mask, smod, page_table)             paged_kv.hpp:117
//   blockattn::PagedKVCache                                     paged_kv.hpp:50-89
//   blockattn::OpCounters                                       engine.hpp:21-32
//   blockattn::validate_inputs (finiteness)                     validate.hpp:30-39
//
// Differences by design: tensors are device buffers (bf16 or fp32); every call is
// stream-ordered (default stream unless given); errors are the same exception classes
// (errors.hpp:11-101) raised from the C ABI status codes. No CPU path exists.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <algorithm>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "flexattn_b200.h"

namespace flexattn {

using i64 = std::int64_t;

// ---- errors (errors.hpp:11-101) ------------------------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
#define FLEXATTN_ERROR(Name) \
  class Name : public Error { \
   public:                    \
    using Error::Error;       \
  };
FLEXATTN_ERROR(ShapeMismatch)
FLEXATTN_ERROR(NonFiniteInput)
FLEXATTN_ERROR(IndexOutOfRange)
FLEXATTN_ERROR(NonPositiveCap)
FLEXATTN_ERROR(GeometryMismatch)
FLEXATTN_ERROR(BlockMaskMismatch)
FLEXATTN_ERROR(StaleStatistics)
FLEXATTN_ERROR(OffsetOutOfRange)
FLEXATTN_ERROR(OutOfPages)
FLEXATTN_ERROR(UnmappedBlock)
FLEXATTN_ERROR(UnmappedPhysicalIndex)
FLEXATTN_ERROR(CudaError)
FLEXATTN_ERROR(Unsupported)
#undef FLEXATTN_ERROR

inline void check(fa_status s) {
  if (s == FA_OK) return;
  const std::string m = fa_last_error();
  switch (s) {
    case FA_SHAPE_MISMATCH: throw ShapeMismatch(m);
    case FA_NON_FINITE_INPUT: throw NonFiniteInput(m);
    case FA_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(m);
    case FA_NON_POSITIVE_CAP: throw NonPositiveCap(m);
    case FA_GEOMETRY_MISMATCH: throw GeometryMismatch(m);
    case FA_BLOCK_MASK_MISMATCH: throw BlockMaskMismatch(m);
    case FA_STALE_STATISTICS: throw StaleStatistics(m);
    case FA_OFFSET_OUT_OF_RANGE: throw OffsetOutOfRange(m);
    case FA_OUT_OF_PAGES: throw OutOfPages(m);
    case FA_UNMAPPED_BLOCK: throw UnmappedBlock(m);
    case FA_UNMAPPED_PHYSICAL_INDEX: throw UnmappedPhysicalIndex(m);
    case FA_UNSUPPORTED: throw Unsupported(m);
    default: throw CudaError(m);
  }
}

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- device memory ---------------------------------------------------------------------------
struct DeviceBuffer {
  std::shared_ptr<void> p;
  size_t bytes = 0;
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) : bytes(n) {
    void* raw = nullptr;
    if (n) check_cuda(cudaMalloc(&raw, n), "cudaMalloc");
    p = std::shared_ptr<void>(raw, [](void* x) { if (x) cudaFree(x); });
  }
  void* get() const { return p.get(); }
  template <typename T>
  T* as() const { return static_cast<T*>(p.get()); }
};

enum class DType : int32_t { F32 = FA_F32, BF16 = FA_BF16 };

// Dense device (B, H, L, D) tensor, row-major like Tensor4 (tensor.hpp:20-117).
struct DeviceTensor4 {
  DeviceBuffer buf;
  DType dtype = DType::BF16;
  i64 b = 0, h = 0, l = 0, d = 0;
  DeviceTensor4() = default;
  DeviceTensor4(i64 b_, i64 h_, i64 l_, i64 d_, DType t = DType::BF16)
      : buf(static_cast<size_t>(b_ * h_ * l_ * d_) * (t == DType::F32 ? 4 : 2)), dtype(t), b(b_), h(h_), l(l_), d(d_) {
    if (b_ <= 0 || h_ <= 0 || l_ <= 0 || d_ <= 0) throw ShapeMismatch("Tensor4: all dims must be positive");
  }
  i64 size() const { return b * h * l * d; }
  fa_tensor c() const {
    fa_tensor t{};
    t.data = buf.get();
    t.dtype = static_cast<int32_t>(dtype);
    t.b = b; t.h = h; t.l = l; t.d = d;
    return t;
  }
  bool same_shape(const DeviceTensor4& o) const { return b == o.b && h == o.h && l == o.l && d == o.d; }
};

// random_tensor (random.hpp:41-46), generated on the device.
inline DeviceTensor4 random_tensor(std::uint64_t seed, i64 b, i64 h, i64 l, i64 d, DType t = DType::BF16,
                                   cudaStream_t st = nullptr) {
  DeviceTensor4 x(b, h, l, d, t);
  check(fa_fill_uniform(x.buf.get(), static_cast<int32_t>(t), seed, 0, x.size(), st));
  return x;
}

// ---- modifiers (modifiers.hpp, mask_library.hpp) -------------------------------------------
struct MaskMod {
  fa_mask_desc d{};
  std::shared_ptr<void> keep;        // device doc-id table
  std::shared_ptr<void> keep_remap;  // device remap table
  std::shared_ptr<void> keep_remap_rc;  // device (row, col) table of remapped na_naive
};
struct ScoreMod {
  fa_score_desc d{};
  std::shared_ptr<void> keep;  // device slopes
  bool identity() const { return d.terms == 0; }
};

inline MaskMod noop_mask() { return MaskMod{}; }
inline MaskMod causal() { MaskMod m; m.d.terms = FA_MASK_CAUSAL; return m; }
inline MaskMod sliding_window(i64 w) {
  if (w < 0) throw IndexOutOfRange("sliding_window: window must be >= 0, got " + std::to_string(w));
  MaskMod m; m.d.terms = FA_MASK_SLIDING_WINDOW; m.d.window = w; return m;
}
inline MaskMod prefix_lm(i64 p) {
  if (p < 0) throw IndexOutOfRange("prefix_lm: prefix_len must be >= 0, got " + std::to_string(p));
  MaskMod m; m.d.terms = FA_MASK_PREFIX_LM; m.d.prefix = p; return m;
}
inline MaskMod document_mask(const std::vector<i64>& ids) {
  std::vector<int32_t> ids32(ids.begin(), ids.end());
  DeviceBuffer buf(ids32.size() * 4);
  check_cuda(cudaMemcpy(buf.get(), ids32.data(), ids32.size() * 4, cudaMemcpyHostToDevice), "doc ids");
  MaskMod m; m.d.terms = FA_MASK_DOCUMENT; m.d.doc_ids = buf.as<int32_t>();
  m.d.doc_len = static_cast<i64>(ids.size()); m.keep = buf.p; return m;
}
inline MaskMod and_mask(const MaskMod& a, const MaskMod& b) {
  MaskMod m = a;
  m.d.terms |= b.d.terms;
  if (b.d.terms & FA_MASK_SLIDING_WINDOW) m.d.window = b.d.window;
  if (b.d.terms & FA_MASK_PREFIX_LM) m.d.prefix = b.d.prefix;
  if (b.d.terms & FA_MASK_DOCUMENT) { m.d.doc_ids = b.d.doc_ids; m.d.doc_len = b.d.doc_len; m.keep = b.keep; }
  if (b.d.terms & FA_MASK_HASH) { m.d.hash_seed = b.d.hash_seed; m.d.hash_density = b.d.hash_density; }
  if (b.d.terms & FA_MASK_NATTEN) {
    m.d.na_height = b.d.na_height; m.d.na_width = b.d.na_width; m.d.na_kernel = b.d.na_kernel;
  }
  return m;
}
inline MaskMod offset_mask(MaskMod m, i64 off) { m.d.q_offset += off; return m; }

// or_mask (mask_library.cpp:100-104) of two single-group masks: the device evaluates
// (AND of a's terms) OR (AND of b's terms), parameters shared between the groups.
inline MaskMod or_mask(const MaskMod& a, const MaskMod& b) {
  if (a.d.or_terms || b.d.or_terms) throw Unsupported("or_mask: operands that are already OR-combinations");
  if (a.d.remap_len || b.d.remap_len) throw Unsupported("or_mask: remapped operands (apply remap_mask last)");
  if (a.d.q_offset != b.d.q_offset) throw Unsupported("or_mask: operands with different offsets");
  if (a.d.terms == 0 || b.d.terms == 0) return noop_mask();  // or with noop is noop
  MaskMod m = and_mask(a, b);  // merges the parameters of both groups
  m.d.terms = a.d.terms;
  m.d.or_terms = b.d.terms;
  if (b.d.terms & FA_MASK_NATTEN) {
    m.d.na_height = b.d.na_height; m.d.na_width = b.d.na_width; m.d.na_kernel = b.d.na_kernel;
  }
  return m;
}

// Neighbourhood attention on a canvas_h x canvas_w row-major canvas (mask_library.cpp:121-215).
struct NAGeometry {
  i64 canvas_h, canvas_w, kernel;
  NAGeometry(i64 h, i64 w, i64 k) : canvas_h(h), canvas_w(w), kernel(k) {
    if (h < 1 || w < 1) throw GeometryMismatch("NAGeometry: canvas dims must be >= 1");
    if (k < 1 || k % 2 == 0) throw GeometryMismatch("NAGeometry: kernel must be odd and >= 1");
    if (k > std::min(h, w)) throw GeometryMismatch("NAGeometry: kernel exceeds canvas");
  }
  i64 tokens() const { return canvas_h * canvas_w; }
};
inline MaskMod na_naive(const NAGeometry& g) {
  MaskMod m;
  m.d.terms = FA_MASK_NATTEN;
  m.d.na_height = g.canvas_h; m.d.na_width = g.canvas_w; m.d.na_kernel = static_cast<int32_t>(g.kernel);
  return m;
}
struct Permutation {
  std::vector<i64> forward;  // slot -> pixel
};
inline Permutation tile_permutation(const NAGeometry& g, i64 tile) {
  if (tile < 1 || g.canvas_h % tile != 0 || g.canvas_w % tile != 0)
    throw GeometryMismatch("tile_permutation: tile must divide the canvas");
  Permutation p;
  for (i64 tr = 0; tr < g.canvas_h; tr += tile)
    for (i64 tc = 0; tc < g.canvas_w; tc += tile)
      for (i64 r = tr; r < tr + tile; ++r)
        for (i64 c = tc; c < tc + tile; ++c) p.forward.push_back(r * g.canvas_w + c);
  return p;
}
inline Permutation morton_permutation(const NAGeometry& g) {
  const i64 n = g.canvas_h;
  if (g.canvas_h != g.canvas_w || (n & (n - 1)) != 0)
    throw GeometryMismatch("morton_permutation: canvas must be square with power-of-two side");
  Permutation p;
  p.forward.assign(static_cast<size_t>(n * n), 0);
  for (i64 r = 0; r < n; ++r)
    for (i64 c = 0; c < n; ++c) {
      i64 slot = 0;
      for (i64 bit = 0; (i64(1) << bit) < n; ++bit) {
        slot |= ((c >> bit) & 1) << (2 * bit);
        slot |= ((r >> bit) & 1) << (2 * bit + 1);
      }
      p.forward[static_cast<size_t>(slot)] = r * n + c;
    }
  return p;
}
// mask(q, kv) = base(fwd[q], fwd[kv]) (mask_library.cpp:203-215)
inline MaskMod remap_mask(MaskMod base, const Permutation& p) {
  std::vector<i64> sorted = p.forward;
  std::sort(sorted.begin(), sorted.end());
  for (size_t i = 0; i < sorted.size(); ++i)
    if (sorted[i] != static_cast<i64>(i)) throw GeometryMismatch("Permutation: forward is not a bijection");
  if (base.d.remap_len) throw Unsupported("remap_mask: base is already remapped");
  std::vector<int32_t> t32(p.forward.begin(), p.forward.end());
  DeviceBuffer buf(t32.size() * 4);
  check_cuda(cudaMemcpy(buf.get(), t32.data(), t32.size() * 4, cudaMemcpyHostToDevice), "remap table");
  base.d.remap = buf.as<int32_t>();
  base.d.remap_len = static_cast<i64>(t32.size());
  base.keep_remap = buf.p;
  if (base.d.terms == FA_MASK_NATTEN && base.d.or_terms == 0 && base.d.na_width > 0 && base.d.na_width < 65536 &&
      base.d.na_height < 65536) {
    // (row << 16) | col of every slot's token: the kernels skip the per-position division
    std::vector<int32_t> rc(t32.size());
    for (size_t i = 0; i < t32.size(); ++i)
      rc[i] = static_cast<int32_t>(((t32[i] / base.d.na_width) << 16) | (t32[i] % base.d.na_width));
    DeviceBuffer rbuf(rc.size() * 4);
    check_cuda(cudaMemcpy(rbuf.get(), rc.data(), rc.size() * 4, cudaMemcpyHostToDevice), "remap rc table");
    base.d.remap_rc = rbuf.as<int32_t>();
    base.keep_remap_rc = rbuf.p;
  }
  return base;
}

inline ScoreMod noop_score() { return ScoreMod{}; }
inline std::vector<double> alibi_slopes(i64 heads) {
  if (heads < 1) throw IndexOutOfRange("alibi_slopes: heads must be >= 1");
  std::vector<double> s(static_cast<size_t>(heads));
  for (i64 h = 0; h < heads; ++h) s[h] = -std::exp2(-8.0 * static_cast<double>(h + 1) / static_cast<double>(heads));
  return s;
}
inline ScoreMod alibi(const std::vector<double>& slopes) {
  std::vector<float> f(slopes.begin(), slopes.end());
  DeviceBuffer buf(f.size() * 4);
  check_cuda(cudaMemcpy(buf.get(), f.data(), f.size() * 4, cudaMemcpyHostToDevice), "slopes");
  ScoreMod s; s.d.terms = FA_SCORE_ALIBI; s.d.slopes = buf.as<float>();
  s.d.num_slopes = static_cast<int32_t>(f.size()); s.keep = buf.p; return s;
}
inline ScoreMod soft_cap(double cap) {
  if (!(cap > 0.0) || !std::isfinite(cap)) throw NonPositiveCap("soft_cap: cap must be finite and > 0");
  ScoreMod s; s.d.terms = FA_SCORE_SOFT_CAP; s.d.cap = cap; return s;
}
inline ScoreMod compose(const ScoreMod& outer, const ScoreMod& inner) {
  if (outer.identity()) return inner;
  if (inner.identity()) return outer;
  if (outer.d.terms == FA_SCORE_SOFT_CAP && inner.d.terms == FA_SCORE_ALIBI) {
    ScoreMod s = inner; s.d.terms |= FA_SCORE_SOFT_CAP; s.d.cap = outer.d.cap; return s;
  }
  throw Unsupported("compose: only soft_cap(alibi(s)) is compiled");
}
inline ScoreMod offset_score(ScoreMod s, i64 off) { s.d.q_offset += off; return s; }

// ---- config (config.hpp:16-45) ---------------------------------------------------------------
struct AttentionConfig {
  std::optional<double> scale;
  i64 gqa_group = 1;
  i64 block_size_q = 128;
  i64 block_size_kv = 128;
  // Not in the reference config: the reference always runs its data-dependent validation
  // (NaN/inf scans -> NonFiniteInput, foreign pages -> UnmappedPhysicalIndex); here it costs an
  // extra pass and a stream synchronisation, so it is opt-in.
  bool validate = false;
  // Backward: ordered dQ additions, bitwise reproducible gradients (README.md:104-106).
  bool deterministic = false;
  double scale_or_default() const { return scale.has_value() ? *scale : 0.0; }
  uint32_t flags() const {
    return (validate ? FA_FLAG_VALIDATE : 0u) | (deterministic ? FA_FLAG_DETERMINISTIC : 0u);
  }
};

// OpCounters (engine.hpp:21-32); calls add into it like the reference. madds omit the
// reference's data-dependent rescale term (see fa_op_counters in flexattn_b200.h).
struct OpCounters {
  std::uint64_t madds = 0;
  std::uint64_t mask_evals = 0;
  std::uint64_t score_evals = 0;
  OpCounters& operator+=(const fa_op_counters& o) {
    madds += o.madds;
    mask_evals += o.mask_evals;
    score_evals += o.score_evals;
    return *this;
  }
};

// validate_inputs' finiteness part (validate.hpp:36-38): throws NonFiniteInput.
inline void check_finite(const std::vector<std::pair<std::string, const DeviceTensor4*>>& ts,
                         cudaStream_t st = nullptr) {
  std::vector<fa_tensor> c;
  std::vector<const char*> names;
  for (const auto& t : ts) {
    c.push_back(t.second->c());
    names.push_back(t.first.c_str());
  }
  check(fa_check_finite(c.data(), names.data(), static_cast<int32_t>(c.size()), st));
}

// ---- BlockMask (block_mask.hpp:35-79) --------------------------------------------------------
struct BlockMask {
  fa_block_mask c{};
  DeviceBuffer kv_num, kv_idx, full_num, full_idx, q_num, q_idx, fq_num, fq_idx;
  MaskMod runtime_mask;
  bool has_runtime_mask = false;
  i64 rows() const { return c.rows; }
  i64 cols() const { return c.cols; }
};

inline BlockMask create_block_mask(const MaskMod& mask, i64 b_dims, i64 h_dims, i64 q_len, i64 kv_len,
                                   i64 bs_q = 128, i64 bs_kv = 128, cudaStream_t st = nullptr) {
  i64 rows = 0, cols = 0;
  size_t ws = 0;
  check(fa_block_mask_geometry(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, &rows, &cols, &ws));
  BlockMask bm;
  const size_t nr = static_cast<size_t>(b_dims * h_dims * rows), nc = static_cast<size_t>(b_dims * h_dims * cols);
  const size_t cells = nr * static_cast<size_t>(cols);
  bm.kv_num = DeviceBuffer(nr * 4); bm.full_num = DeviceBuffer(nr * 4);
  bm.kv_idx = DeviceBuffer(cells * 4); bm.full_idx = DeviceBuffer(cells * 4);
  bm.q_num = DeviceBuffer(nc * 4); bm.fq_num = DeviceBuffer(nc * 4);
  bm.q_idx = DeviceBuffer(cells * 4); bm.fq_idx = DeviceBuffer(cells * 4);
  bm.c.kv_num_blocks = bm.kv_num.as<int32_t>(); bm.c.kv_indices = bm.kv_idx.as<int32_t>();
  bm.c.full_kv_num_blocks = bm.full_num.as<int32_t>(); bm.c.full_kv_indices = bm.full_idx.as<int32_t>();
  bm.c.q_num_blocks = bm.q_num.as<int32_t>(); bm.c.q_indices = bm.q_idx.as<int32_t>();
  bm.c.full_q_num_blocks = bm.fq_num.as<int32_t>(); bm.c.full_q_indices = bm.fq_idx.as<int32_t>();
  DeviceBuffer work(ws ? ws : 1);
  check(fa_create_block_mask(&mask.d, b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, &bm.c, work.get(), ws, st));
  check_cuda(cudaStreamSynchronize(st), "create_block_mask");  // workspace freed on return
  bm.runtime_mask = mask;
  bm.has_runtime_mask = true;
  return bm;
}

// transpose (block_mask.cpp:161-178): the q-side arrays of `bm` viewed as a kv-side mask.
inline BlockMask transpose(const BlockMask& bm) {
  BlockMask t = bm;
  t.c.rows = bm.c.cols; t.c.cols = bm.c.rows; t.c.bs_q = bm.c.bs_kv; t.c.bs_kv = bm.c.bs_q;
  t.c.q_len = bm.c.kv_len; t.c.kv_len = bm.c.q_len;
  std::swap(t.c.kv_num_blocks, t.c.q_num_blocks); std::swap(t.c.kv_indices, t.c.q_indices);
  std::swap(t.c.full_kv_num_blocks, t.c.full_q_num_blocks); std::swap(t.c.full_kv_indices, t.c.full_q_indices);
  t.has_runtime_mask = false;
  return t;
}

// Host copies of the kv-side arrays (for inspection / parity), widened to i64 like the reference.
struct HostBlockMask {
  std::vector<i64> partial_num, partial_idx, full_num, full_idx;
};
inline HostBlockMask to_host(const BlockMask& bm) {
  auto copy = [](const int32_t* p, size_t n) {
    std::vector<int32_t> v(n);
    check_cuda(cudaMemcpy(v.data(), p, n * 4, cudaMemcpyDeviceToHost), "to_host");
    return std::vector<i64>(v.begin(), v.end());
  };
  const size_t nr = static_cast<size_t>(bm.c.b_dims * bm.c.h_dims * bm.c.rows);
  const size_t cells = nr * static_cast<size_t>(bm.c.cols);
  return HostBlockMask{copy(bm.c.kv_num_blocks, nr), copy(bm.c.kv_indices, cells),
                       copy(bm.c.full_kv_num_blocks, nr), copy(bm.c.full_kv_indices, cells)};
}

// ---- attention (engine.hpp) --------------------------------------------------------------------
struct AttentionOutput {
  DeviceTensor4 out;
  DeviceBuffer lse;  // (B, H, L) fp32, natural log
};
struct Gradients {
  DeviceTensor4 dq, dk, dv;
};

inline AttentionOutput forward(const DeviceTensor4& q, const DeviceTensor4& k, const DeviceTensor4& v,
                               const ScoreMod& smod, const BlockMask& bm, const AttentionConfig& cfg = {},
                               OpCounters* counters = nullptr, cudaStream_t st = nullptr) {
  if (!bm.has_runtime_mask) throw BlockMaskMismatch("forward: block mask has no runtime mask attached");
  if (bm.c.bs_q != cfg.block_size_q || bm.c.bs_kv != cfg.block_size_kv)
    throw BlockMaskMismatch("block mask block sizes disagree with config");
  AttentionOutput res{DeviceTensor4(q.b, q.h, q.l, q.d, q.dtype), DeviceBuffer(static_cast<size_t>(q.b * q.h * q.l) * 4)};
  fa_fwd_args a{};
  a.q = q.c(); a.k = k.c(); a.v = v.c(); a.out = res.out.c();
  a.lse = res.lse.as<float>();
  a.bm = &bm.c;
  a.mask = bm.runtime_mask.d;
  a.score = smod.d;
  a.scale = cfg.scale_or_default();
  a.gqa_group = cfg.gqa_group;
  a.flags = cfg.flags() & FA_FLAG_VALIDATE;
  fa_op_counters cc{};
  if (counters) a.counters = &cc;
  check(fa_flex_fwd(&a, st));
  if (counters) *counters += cc;
  return res;
}

inline Gradients backward(const DeviceTensor4& q, const DeviceTensor4& k, const DeviceTensor4& v,
                          const AttentionOutput& fwd, const DeviceTensor4& d_out, const ScoreMod& smod,
                          const BlockMask& bm, const BlockMask& /*bm_t: q side lives in bm*/,
                          const AttentionConfig& cfg = {}, OpCounters* counters = nullptr,
                          cudaStream_t st = nullptr) {
  if (!bm.has_runtime_mask) throw BlockMaskMismatch("backward: block mask has no runtime mask attached");
  Gradients g{DeviceTensor4(q.b, q.h, q.l, q.d, q.dtype), DeviceTensor4(k.b, k.h, k.l, k.d, k.dtype),
              DeviceTensor4(v.b, v.h, v.l, v.d, v.dtype)};
  const size_t ws = fa_bwd_workspace_size(q.b, q.h, q.l, q.d);
  DeviceBuffer work(ws);
  fa_bwd_args a{};
  a.q = q.c(); a.k = k.c(); a.v = v.c(); a.out = fwd.out.c(); a.d_out = d_out.c();
  a.lse = fwd.lse.as<float>();
  a.dq = g.dq.c(); a.dk = g.dk.c(); a.dv = g.dv.c();
  a.bm = &bm.c;
  a.mask = bm.runtime_mask.d;
  a.score = smod.d;
  a.scale = cfg.scale_or_default();
  a.gqa_group = cfg.gqa_group;
  a.workspace = work.get();
  a.workspace_bytes = ws;
  a.flags = cfg.flags();
  fa_op_counters cc{};
  if (counters) a.counters = &cc;
  check(fa_flex_bwd(&a, st));
  if (counters) *counters += cc;
  check_cuda(cudaStreamSynchronize(st), "backward");  // workspace freed on return
  return g;
}

inline AttentionOutput decode(const DeviceTensor4& q_step, const DeviceTensor4& k_cache,
                              const DeviceTensor4& v_cache, i64 offset, const MaskMod& mask,
                              const ScoreMod& smod, const BlockMask& bm, const AttentionConfig& cfg = {},
                              const fa_page_table* pt = nullptr, OpCounters* counters = nullptr,
                              cudaStream_t st = nullptr) {
  AttentionOutput res{DeviceTensor4(q_step.b, q_step.h, q_step.l, q_step.d, q_step.dtype),
                      DeviceBuffer(static_cast<size_t>(q_step.b * q_step.h * q_step.l) * 4)};
  const size_t ws = fa_decode_workspace_size(q_step.b, q_step.h, q_step.l, q_step.d, 0);
  DeviceBuffer work(ws);
  fa_decode_args a{};
  a.q = q_step.c(); a.k_cache = k_cache.c(); a.v_cache = v_cache.c(); a.out = res.out.c();
  a.lse = res.lse.as<float>();
  a.bm = &bm.c;
  a.pt = pt;
  a.offset = offset;
  a.mask = mask.d;
  a.score = smod.d;
  a.scale = cfg.scale_or_default();
  a.gqa_group = cfg.gqa_group;
  a.workspace = work.get();
  a.workspace_bytes = ws;
  a.flags = cfg.flags() & FA_FLAG_VALIDATE;
  fa_op_counters cc{};
  if (counters) a.counters = &cc;
  check(fa_flex_decode(&a, st));
  if (counters) *counters += cc;
  check_cuda(cudaStreamSynchronize(st), "decode");
  return res;
}

// convert_block_mask (paged_kv.cpp:154-228); page-table arrays on the device.
inline BlockMask convert_block_mask(const BlockMask& bm, const fa_page_table& pt, cudaStream_t st = nullptr) {
  BlockMask out;
  const size_t nr = static_cast<size_t>(pt.batches * bm.c.h_dims * bm.c.rows);
  const size_t cells = nr * static_cast<size_t>(pt.num_physical_pages);
  out.kv_num = DeviceBuffer(nr * 4); out.full_num = DeviceBuffer(nr * 4);
  out.kv_idx = DeviceBuffer(cells * 4); out.full_idx = DeviceBuffer(cells * 4);
  out.c.kv_num_blocks = out.kv_num.as<int32_t>(); out.c.kv_indices = out.kv_idx.as<int32_t>();
  out.c.full_kv_num_blocks = out.full_num.as<int32_t>(); out.c.full_kv_indices = out.full_idx.as<int32_t>();
  check(fa_convert_block_mask(&bm.c, &pt, &out.c, st));
  out.runtime_mask = bm.runtime_mask;
  out.has_runtime_mask = bm.has_runtime_mask;
  return out;
}

// ---- paged KV cache (paged_kv.hpp:18-89, paged_kv.cpp:13-152) --------------------------------
// PageTable with host arrays (the reference's value type) and device mirrors for the kernels.
struct PageTable {
  static constexpr std::int32_t kSentinel = -1;
  i64 batches = 0, max_logical_pages = 0, num_physical_pages = 0, page_size = 0;
  std::vector<std::int32_t> table, phys_to_logical, owner, seq_len;
  i64 lookup(i64 b, i64 lp) const { return table[static_cast<size_t>(b * max_logical_pages + lp)]; }
  // device snapshot (convert_mods snapshots the table by value, paged_kv.hpp:115-116)
  struct Device {
    DeviceBuffer table, p2l, owner, seq;
    fa_page_table c{};
  };
  std::shared_ptr<Device> to_device(cudaStream_t st = nullptr) const {
    auto d = std::make_shared<Device>();
    auto up = [st](const std::vector<std::int32_t>& v, DeviceBuffer& buf) {
      buf = DeviceBuffer(std::max<size_t>(v.size(), 1) * 4);
      if (!v.empty())
        check_cuda(cudaMemcpyAsync(buf.get(), v.data(), v.size() * 4, cudaMemcpyHostToDevice, st), "page table");
    };
    up(table, d->table); up(phys_to_logical, d->p2l); up(owner, d->owner); up(seq_len, d->seq);
    check_cuda(cudaStreamSynchronize(st), "page table");
    d->c.batches = batches; d->c.max_logical_pages = max_logical_pages;
    d->c.num_physical_pages = num_physical_pages; d->c.page_size = page_size;
    d->c.table = d->table.as<int32_t>(); d->c.phys_to_logical = d->p2l.as<int32_t>();
    d->c.owner = d->owner.as<int32_t>(); d->c.seq_len = d->seq.as<int32_t>();
    d->c.max_seq_len = seq_len.empty() ? 0 : *std::max_element(seq_len.begin(), seq_len.end());
    return d;
  }
};

// PagedKVCache (paged_kv.hpp:50-89) with the allocator on the device (fa_page_pool: LIFO free
// stack with page 0 on top, deterministic shuffle, capacity-checked assign / append, idempotent
// erase; paged_kv.cpp:13-152) over device K/V of shape (1, kv_heads, num_pages * page_size, dim).
// Single-sequence calls throw like the reference; the *_batch calls apply many requests in
// order in one launch (device int32 arrays, one request per sequence) and, with sync = false,
// leave the outcome on the device for status() (CUDA-graph serving loops).
class PagedKVCache {
 public:
  PagedKVCache(i64 batches, i64 num_pages, i64 page_size, i64 kv_heads, i64 dim, DType t = DType::BF16,
               cudaStream_t st = nullptr)
      : k_(1, kv_heads, num_pages * page_size, dim, t), v_(1, kv_heads, num_pages * page_size, dim, t) {
    if (batches < 1 || num_pages < 1 || page_size < 1)
      throw ShapeMismatch("PagedKVCache: batches, num_pages and page_size must be >= 1");
    const size_t bytes = fa_page_pool_bytes(batches, num_pages);
    mem_ = DeviceBuffer(bytes);
    check(fa_page_pool_init(&pool_, mem_.get(), bytes, batches, num_pages, page_size, st));
    check_cuda(cudaMemsetAsync(k_.buf.get(), 0, k_.buf.bytes, st), "cache");
    check_cuda(cudaMemsetAsync(v_.buf.get(), 0, v_.buf.bytes, st), "cache");
    ids_ = DeviceBuffer(static_cast<size_t>(batches) * 4);
    ntok_ = DeviceBuffer(static_cast<size_t>(batches) * 4);
  }

  // assign (paged_kv.cpp:72-98): tokens (1, kv_heads, n, dim) on the device
  void assign(i64 b, const DeviceTensor4& k_tokens, const DeviceTensor4& v_tokens, cudaStream_t st = nullptr) {
    one(FA_PAGE_ASSIGN, b, k_tokens.l, &k_tokens, &v_tokens, st);
  }
  // append_tokens (paged_kv.cpp:100-126), at any position (fills the slack of the last page)
  void append_tokens(i64 b, const DeviceTensor4& k_new, const DeviceTensor4& v_new, cudaStream_t st = nullptr) {
    one(FA_PAGE_APPEND, b, k_new.l, &k_new, &v_new, st);
  }
  // erase (paged_kv.cpp:128-141): idempotent
  void erase(i64 b, cudaStream_t st = nullptr) { one(FA_PAGE_ERASE, b, 0, nullptr, nullptr, st); }
  // batched updates: device int32 batch_ids[n] / n_tokens[n]; tokens packed along L (or null)
  void update_batch(int32_t op, const int32_t* batch_ids, const int32_t* n_tokens, int32_t n,
                    const DeviceTensor4* k_tokens, const DeviceTensor4* v_tokens, bool sync = true,
                    cudaStream_t st = nullptr) {
    fa_tensor kt{}, vt{}, kc = k_.c(), vc = v_.c();
    if (k_tokens != nullptr) { kt = k_tokens->c(); vt = v_tokens->c(); }
    check(fa_page_pool_update(&pool_, op, batch_ids, n_tokens, n, k_tokens ? &kt : nullptr,
                              v_tokens ? &vt : nullptr, &kc, &vc, sync ? 0u : uint32_t(FA_FLAG_NO_SYNC), st));
  }
  // outcome of the last update (synchronises); returns the number of requests applied
  int32_t status(cudaStream_t st = nullptr) const {
    int32_t applied = 0;
    check(fa_page_pool_status(&pool_, &applied, st));
    return applied;
  }
  // shuffle_free_pages (paged_kv.cpp:143-146, deterministic_shuffle random.hpp:49-56)
  void shuffle_free_pages(std::uint64_t seed, cudaStream_t st = nullptr) {
    check(fa_page_pool_shuffle(&pool_, seed, st));
  }
  const DeviceTensor4& k_phys() const { return k_; }
  const DeviceTensor4& v_phys() const { return v_; }
  // live device page table (no copy) for convert_block_mask / decode
  fa_page_table device_table() const {
    fa_page_table t = fa_page_pool_table(&pool_);
    t.max_seq_len = max_seq_len();
    return t;
  }
  // host snapshot of the page table (paged_kv.hpp:18-41)
  PageTable table() const {
    PageTable pt;
    pt.batches = pool_.batches;
    pt.max_logical_pages = pt.num_physical_pages = pool_.num_pages;
    pt.page_size = pool_.page_size;
    pt.table = down(pool_.table, pool_.batches * pool_.num_pages);
    pt.phys_to_logical = down(pool_.phys_to_logical, pool_.num_pages);
    pt.owner = down(pool_.owner, pool_.num_pages);
    pt.seq_len = down(pool_.seq_len, pool_.batches);
    return pt;
  }
  i64 page_size() const { return pool_.page_size; }
  i64 max_tokens() const { return pool_.num_pages * pool_.page_size; }
  i64 seq_len(i64 b) const {
    check_batch(b);
    std::int32_t v = 0;
    check_cuda(cudaMemcpy(&v, pool_.seq_len + b, 4, cudaMemcpyDeviceToHost), "seq_len");
    return v;
  }
  i64 free_pages() const { return down(pool_.free_count, 1)[0]; }
  const fa_page_pool& pool() const { return pool_; }

 private:
  static std::vector<std::int32_t> down(const std::int32_t* p, i64 n) {
    std::vector<std::int32_t> v(static_cast<size_t>(n));
    if (n) check_cuda(cudaMemcpy(v.data(), p, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost), "page pool");
    return v;
  }
  i64 max_seq_len() const {
    const auto s = down(pool_.seq_len, pool_.batches);
    return s.empty() ? 0 : *std::max_element(s.begin(), s.end());
  }
  void check_batch(i64 b) const {
    if (b < 0 || b >= pool_.batches)
      throw IndexOutOfRange("PagedKVCache: batch " + std::to_string(b) + " outside [0, " +
                            std::to_string(pool_.batches) + ")");
  }
  void one(int32_t op, i64 b, i64 n, const DeviceTensor4* kt, const DeviceTensor4* vt, cudaStream_t st) {
    if (kt != nullptr && (!kt->same_shape(*vt) || kt->dtype != vt->dtype))
      throw ShapeMismatch("PagedKVCache: k and v tokens must agree");
    const std::int32_t req[2] = {static_cast<std::int32_t>(b), static_cast<std::int32_t>(n)};
    check_cuda(cudaMemcpyAsync(ids_.get(), &req[0], 4, cudaMemcpyHostToDevice, st), "request");
    check_cuda(cudaMemcpyAsync(ntok_.get(), &req[1], 4, cudaMemcpyHostToDevice, st), "request");
    update_batch(op, ids_.as<int32_t>(), ntok_.as<int32_t>(), 1, kt, vt, true, st);
  }

  DeviceTensor4 k_, v_;
  DeviceBuffer mem_, ids_, ntok_;
  fa_page_pool pool_{};
};

// convert_block_mask over a host PageTable (uploads a device snapshot).
inline BlockMask convert_block_mask(const BlockMask& bm, const PageTable& pt, cudaStream_t st = nullptr) {
  const auto d = pt.to_device(st);
  return convert_block_mask(bm, d->c, st);
}

// convert_mods (paged_kv.hpp:117, paged_kv.cpp:230-310): the reference bakes a
// (batch, physical index) -> logical index table into new callables. Here the mods stay the
// user's (written in logical positions) and carry a device snapshot of the page table; the
// decode kernel recovers logical positions per page (phys_to_logical, owner, seq_len), masks
// slack, and with cfg.validate reports foreign pages as UnmappedPhysicalIndex.
struct ConvertedMods {
  MaskMod mask;
  ScoreMod score;
  std::shared_ptr<PageTable::Device> table;
};
inline ConvertedMods convert_mods(const MaskMod& mask, const ScoreMod& smod, const PageTable& pt,
                                  cudaStream_t st = nullptr) {
  return ConvertedMods{mask, smod, pt.to_device(st)};
}
// decode over a paged cache with converted mods (the reference passes cm.mask / cm.score).
inline AttentionOutput decode(const DeviceTensor4& q_step, const PagedKVCache& cache, i64 offset,
                              const ConvertedMods& cm, const BlockMask& physical_bm,
                              const AttentionConfig& cfg = {}, OpCounters* counters = nullptr,
                              cudaStream_t st = nullptr) {
  return decode(q_step, cache.k_phys(), cache.v_phys(), offset, cm.mask, cm.score, physical_bm, cfg,
                &cm.table->c, counters, st);
}

}  // namespace flexattn
