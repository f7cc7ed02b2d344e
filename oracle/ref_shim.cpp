// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. A C-ABI shim over the UNMODIFIED
// reference library (/root/reference/proj/src/*.cpp, compiled from where the
// sources lie by oracle/Makefile into oracle/_ref/libblockattn_ref.so). It lets
// pytest (ctypes) run the reference's own create_block_mask / transpose /
// forward / backward / decode / PagedKVCache / convert_block_mask on the same
// synthetic inputs the GPU path sees, and lets bench.py time the reference
// CPU path (`--impl reference`, cpu_baseline kind "reference").
//
// No reference source is copied here; the shim only calls the public API
// declared in /root/reference/proj/include/blockattn/*.hpp.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <blockattn/block_mask.hpp>
#include <blockattn/engine.hpp>
#include <blockattn/errors.hpp>
#include <blockattn/mask_library.hpp>
#include <blockattn/paged_kv.hpp>
#include <blockattn/parallel.hpp>
#include <blockattn/random.hpp>

#include "test_support.hpp"  // reference tests/test_support.hpp (hash_mask, never_mask)

using namespace blockattn;

namespace {

thread_local std::string g_err;

struct RefMask {  // same field order as fo_mask (oracle/flex_oracle.h)
  uint32_t terms;
  int32_t hash_density;
  int64_t window;
  int64_t prefix;
  int64_t q_offset;
  uint64_t hash_seed;
  const int64_t* doc_ids;
  int64_t doc_len;
  int64_t bound_q;
  int64_t bound_kv;
  uint32_t or_terms;
  int32_t na_kernel;
  int64_t na_height;
  int64_t na_width;
  const int64_t* remap;
  int64_t remap_len;
};

struct RefScore {  // same field order as fo_score
  uint32_t terms;
  int32_t num_slopes;
  double cap;
  const double* slopes;
  int64_t q_offset;
};

// Build the user mask as the reference library would: and_mask of the terms, or_mask with the
// second term group, remap_mask around both, offset_mask outermost.
MaskMod make_group(const RefMask& d, uint32_t terms) {
  MaskMod m = noop_mask();
  bool have = false;
  auto add = [&](MaskMod t) {
    m = have ? and_mask(m, t) : t;
    have = true;
  };
  if (terms & 32u) add(testsupport::never_mask());
  if (terms & 1u) add(causal());
  if (terms & 2u) add(sliding_window(d.window));
  if (terms & 64u) add(na_naive(NAGeometry(d.na_height, d.na_width, d.na_kernel)));
  if (terms & 4u) add(document_mask(std::vector<i64>(d.doc_ids, d.doc_ids + d.doc_len)));
  if (terms & 8u) add(prefix_lm(d.prefix));
  if (terms & 16u) add(testsupport::hash_mask(d.hash_seed, d.hash_density));
  return m;
}

MaskMod make_mask(const RefMask& d, bool with_offset = true) {
  MaskMod m = make_group(d, d.terms);
  if (d.or_terms != 0) m = or_mask(m, make_group(d, d.or_terms));
  if (d.remap_len > 0) {
    Permutation p;
    p.forward.assign(d.remap, d.remap + d.remap_len);
    m = remap_mask(m, p);
  }
  if (with_offset && d.q_offset != 0) m = offset_mask(m, d.q_offset);
  return m;
}

ScoreMod make_score(const RefScore& d, bool with_offset = true) {
  ScoreMod s = noop_score();
  const bool al = (d.terms & 1u) != 0, sc = (d.terms & 2u) != 0;
  if (al && sc) {
    s = compose(soft_cap(d.cap), alibi(std::vector<double>(d.slopes, d.slopes + d.num_slopes)));
  } else if (al) {
    s = alibi(std::vector<double>(d.slopes, d.slopes + d.num_slopes));
  } else if (sc) {
    s = soft_cap(d.cap);
  }
  if (with_offset && d.q_offset != 0) s = offset_score(s, d.q_offset);
  return s;
}

int status_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ShapeMismatch*>(&e)) return 1;
  if (dynamic_cast<const NonFiniteInput*>(&e)) return 2;
  if (dynamic_cast<const IndexOutOfRange*>(&e)) return 3;
  if (dynamic_cast<const NonPositiveCap*>(&e)) return 4;
  if (dynamic_cast<const GeometryMismatch*>(&e)) return 5;
  if (dynamic_cast<const BlockMaskMismatch*>(&e)) return 6;
  if (dynamic_cast<const StaleStatistics*>(&e)) return 7;
  if (dynamic_cast<const OffsetOutOfRange*>(&e)) return 8;
  if (dynamic_cast<const OutOfPages*>(&e)) return 9;
  if (dynamic_cast<const UnmappedBlock*>(&e)) return 10;
  if (dynamic_cast<const UnmappedPhysicalIndex*>(&e)) return 11;
  return 99;
}

template <typename Real>
Tensor4<Real> tensor_from(const Real* p, i64 b, i64 h, i64 l, i64 d) {
  return Tensor4<Real>(b, h, l, d, std::vector<Real>(p, p + b * h * l * d));
}

void copy_bm(const BlockMask& bm, int64_t* pn, int64_t* pi, int64_t* fn, int64_t* fi, int64_t* vn,
             int64_t* vi, uint8_t* vf) {
  std::memcpy(pn, bm.partial_num.data(), bm.partial_num.size() * 8);
  std::memcpy(pi, bm.partial_idx.data(), bm.partial_idx.size() * 8);
  std::memcpy(fn, bm.full_num.data(), bm.full_num.size() * 8);
  std::memcpy(fi, bm.full_idx.data(), bm.full_idx.size() * 8);
  if (vn) std::memcpy(vn, bm.visit_num.data(), bm.visit_num.size() * 8);
  if (vi) std::memcpy(vi, bm.visit_idx.data(), bm.visit_idx.size() * 8);
  if (vf) std::memcpy(vf, bm.visit_full_flag.data(), bm.visit_full_flag.size());
}

template <typename Real>
int do_forward(const Real* q, const Real* k, const Real* v, int64_t B, int64_t Hq, int64_t Hkv,
               int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D, double scale, int64_t gqa,
               const RefScore* s, const RefMask* m, int64_t mb, int64_t mh, int64_t bs,
               Real* out, Real* lse) {
  try {
    AttentionConfig cfg;
    if (scale > 0) cfg.scale = scale;
    cfg.gqa_group = gqa;
    cfg.block_size_q = cfg.block_size_kv = bs;
    const auto bm = create_block_mask(make_mask(*m), mb, mh, Lq, Lkv, bs, bs);
    const auto res = forward(tensor_from(q, B, Hq, Lq, D), tensor_from(k, Bkv, Hkv, Lkv, D),
                             tensor_from(v, Bkv, Hkv, Lkv, D), make_score(*s), bm, cfg);
    std::memcpy(out, res.out.data().data(), res.out.data().size() * sizeof(Real));
    std::memcpy(lse, res.lse.data(), res.lse.size() * sizeof(Real));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

template <typename Real>
int do_backward(const Real* q, const Real* k, const Real* v, const Real* dout, int64_t B,
                int64_t Hq, int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D,
                double scale, int64_t gqa, const RefScore* s, const RefMask* m, int64_t mb,
                int64_t mh, int64_t bs, Real* out, Real* lse, Real* dq, Real* dk, Real* dv) {
  try {
    AttentionConfig cfg;
    if (scale > 0) cfg.scale = scale;
    cfg.gqa_group = gqa;
    cfg.block_size_q = cfg.block_size_kv = bs;
    const auto bm = create_block_mask(make_mask(*m), mb, mh, Lq, Lkv, bs, bs);
    const auto bm_t = transpose(bm);
    const auto qt = tensor_from(q, B, Hq, Lq, D);
    const auto kt = tensor_from(k, Bkv, Hkv, Lkv, D);
    const auto vt = tensor_from(v, Bkv, Hkv, Lkv, D);
    const auto smod = make_score(*s);
    const auto fwd = forward(qt, kt, vt, smod, bm, cfg);
    const auto g = backward(qt, kt, vt, fwd, tensor_from(dout, B, Hq, Lq, D), smod, bm, bm_t, cfg);
    std::memcpy(out, fwd.out.data().data(), fwd.out.data().size() * sizeof(Real));
    std::memcpy(lse, fwd.lse.data(), fwd.lse.size() * sizeof(Real));
    std::memcpy(dq, g.dq.data().data(), g.dq.data().size() * sizeof(Real));
    std::memcpy(dk, g.dk.data().data(), g.dk.data().size() * sizeof(Real));
    std::memcpy(dv, g.dv.data().data(), g.dv.data().size() * sizeof(Real));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// save_block_mask / render_ppm / save_tensor of the reference, for byte-level comparisons
int ref_save_block_mask(const RefMask* m, int64_t bd, int64_t hd, int64_t ql, int64_t kl, int64_t bsq,
                        int64_t bskv, const char* path) {
  try {
    save_block_mask(path, create_block_mask(make_mask(*m), bd, hd, ql, kl, bsq, bskv));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
// load a BlockMask file with the reference and return its kv-side arrays (sizes from the header)
int ref_load_block_mask(const char* path, int64_t* hdr8, int64_t* pn, int64_t* pi, int64_t* fn,
                        int64_t* fi, int64_t cap_rows, int64_t cap_cells) {
  try {
    const BlockMask bm = load_block_mask(path);
    const int64_t v[8] = {bm.b_dims, bm.h_dims, bm.rows, bm.cols, bm.bs_q, bm.bs_kv, bm.q_len, bm.kv_len};
    std::copy(v, v + 8, hdr8);
    if (static_cast<int64_t>(bm.partial_num.size()) > cap_rows ||
        static_cast<int64_t>(bm.partial_idx.size()) > cap_cells)
      return 1;
    std::copy(bm.partial_num.begin(), bm.partial_num.end(), pn);
    std::copy(bm.partial_idx.begin(), bm.partial_idx.end(), pi);
    std::copy(bm.full_num.begin(), bm.full_num.end(), fn);
    std::copy(bm.full_idx.begin(), bm.full_idx.end(), fi);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
int ref_write_ppm(const RefMask* m, int64_t ql, int64_t kl, int64_t bs, const char* path) {
  try {
    write_ppm(path, create_block_mask(make_mask(*m), 1, 1, ql, kl, bs, bs), 0, 0);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
int ref_save_tensor_f32(const float* x, int64_t B, int64_t H, int64_t L, int64_t D, const char* path) {
  try {
    save_tensor(path, Tensor4<float>(B, H, L, D, std::vector<float>(x, x + B * H * L * D)));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
int ref_load_tensor_f32(const char* path, float* out, int64_t cap) {
  try {
    const auto t = load_tensor<float>(path);
    if (static_cast<int64_t>(t.data().size()) > cap) return 1;
    std::copy(t.data().begin(), t.data().end(), out);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// tile_permutation / morton_permutation (mask_library.cpp:164-201): forward table into out[h*w]
int ref_tile_permutation(int64_t h, int64_t w, int64_t k, int64_t tile, int64_t* out) {
  try {
    const auto p = tile_permutation(NAGeometry(h, w, k), tile);
    std::copy(p.forward.begin(), p.forward.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
int ref_morton_permutation(int64_t h, int64_t w, int64_t k, int64_t* out) {
  try {
    const auto p = morton_permutation(NAGeometry(h, w, k));
    std::copy(p.forward.begin(), p.forward.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
int ref_worker_count() { return worker_count(); }

// create_block_mask (+ transpose) with all seven arrays (block_mask.hpp:109-115).
int ref_create_block_mask(const RefMask* m, int64_t bd, int64_t hd, int64_t ql, int64_t kl,
                          int64_t bsq, int64_t bskv, int64_t* pn, int64_t* pi, int64_t* fn,
                          int64_t* fi, int64_t* vn, int64_t* vi, uint8_t* vf, int64_t* tpn,
                          int64_t* tpi, int64_t* tfn, int64_t* tfi) {
  try {
    const auto bm = create_block_mask(make_mask(*m), bd, hd, ql, kl, bsq, bskv);
    copy_bm(bm, pn, pi, fn, fi, vn, vi, vf);
    if (tpn) {
      const auto t = transpose(bm);
      copy_bm(t, tpn, tpi, tfn, tfi, nullptr, nullptr, nullptr);
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_forward_f32(const float* q, const float* k, const float* v, int64_t B, int64_t Hq,
                    int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D, double scale,
                    int64_t gqa, const RefScore* s, const RefMask* m, int64_t mb, int64_t mh,
                    int64_t bs, float* out, float* lse) {
  return do_forward<float>(q, k, v, B, Hq, Hkv, Bkv, Lq, Lkv, D, scale, gqa, s, m, mb, mh, bs,
                           out, lse);
}

int ref_forward_f64(const double* q, const double* k, const double* v, int64_t B, int64_t Hq,
                    int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D, double scale,
                    int64_t gqa, const RefScore* s, const RefMask* m, int64_t mb, int64_t mh,
                    int64_t bs, double* out, double* lse) {
  return do_forward<double>(q, k, v, B, Hq, Hkv, Bkv, Lq, Lkv, D, scale, gqa, s, m, mb, mh, bs,
                            out, lse);
}

int ref_backward_f32(const float* q, const float* k, const float* v, const float* dout,
                     int64_t B, int64_t Hq, int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv,
                     int64_t D, double scale, int64_t gqa, const RefScore* s, const RefMask* m,
                     int64_t mb, int64_t mh, int64_t bs, float* out, float* lse, float* dq,
                     float* dk, float* dv) {
  return do_backward<float>(q, k, v, dout, B, Hq, Hkv, Bkv, Lq, Lkv, D, scale, gqa, s, m, mb, mh,
                            bs, out, lse, dq, dk, dv);
}

int ref_backward_f64(const double* q, const double* k, const double* v, const double* dout,
                     int64_t B, int64_t Hq, int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv,
                     int64_t D, double scale, int64_t gqa, const RefScore* s, const RefMask* m,
                     int64_t mb, int64_t mh, int64_t bs, double* out, double* lse, double* dq,
                     double* dk, double* dv) {
  return do_backward<double>(q, k, v, dout, B, Hq, Hkv, Bkv, Lq, Lkv, D, scale, gqa, s, m, mb, mh,
                             bs, out, lse, dq, dk, dv);
}

// decode (engine.cpp:403-427): q_step rows [offset, offset+n_new); bm built the
// way bench.cpp:518-519 does (offset_mask of the user mask at q_len = n_new).
int ref_decode_f32(const float* q_step, const float* k, const float* v, int64_t B, int64_t Hq,
                   int64_t Hkv, int64_t Bkv, int64_t n_new, int64_t Lkv, int64_t D, int64_t offset,
                   double scale, int64_t gqa, const RefScore* s, const RefMask* m, int64_t bs,
                   float* out, float* lse) {
  try {
    AttentionConfig cfg;
    if (scale > 0) cfg.scale = scale;
    cfg.gqa_group = gqa;
    cfg.block_size_q = cfg.block_size_kv = bs;
    const MaskMod user = make_mask(*m, /*with_offset=*/false);
    const auto bm = create_block_mask(offset_mask(user, offset), 1, 1, n_new, Lkv, bs, bs);
    const auto res = decode(tensor_from(q_step, B, Hq, n_new, D), tensor_from(k, Bkv, Hkv, Lkv, D),
                            tensor_from(v, Bkv, Hkv, Lkv, D), offset, user,
                            make_score(*s, false), bm, cfg);
    std::memcpy(out, res.out.data().data(), res.out.data().size() * sizeof(float));
    std::memcpy(lse, res.lse.data(), res.lse.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// Paged decode the way the reference composes it (bench.cpp:546-589 with the
// decode geometry of :512-545): PagedKVCache with batch*pages_per_seq+batch
// pages, shuffled free list, assign per batch, convert_block_mask +
// convert_mods, forward over the physical buffer with the shifted mask.
// Outputs the physical page table so the GPU path can reuse the same layout.
int ref_paged_decode_f32(const float* q_step, const float* k, const float* v, int64_t B,
                         int64_t Hq, int64_t Hkv, int64_t n_new, int64_t Lkv, int64_t D,
                         int64_t offset, double scale, int64_t gqa, const RefScore* s,
                         const RefMask* m, int64_t page_size, uint64_t shuffle_seed, float* out,
                         float* lse, int32_t* table_out, int64_t* num_pages_out) {
  try {
    AttentionConfig cfg;
    if (scale > 0) cfg.scale = scale;
    cfg.gqa_group = gqa;
    cfg.block_size_q = cfg.block_size_kv = page_size;
    const i64 pages_per_seq = (Lkv + page_size - 1) / page_size;
    const i64 num_pages = B * pages_per_seq + B;
    PagedKVCache<float> cache(B, num_pages, page_size, Hkv, D);
    cache.shuffle_free_pages(shuffle_seed);
    for (i64 b = 0; b < B; ++b) {
      std::vector<float> kb(k + b * Hkv * Lkv * D, k + (b + 1) * Hkv * Lkv * D);
      std::vector<float> vb(v + b * Hkv * Lkv * D, v + (b + 1) * Hkv * Lkv * D);
      cache.assign(b, Tensor4<float>(1, Hkv, Lkv, D, std::move(kb)),
                   Tensor4<float>(1, Hkv, Lkv, D, std::move(vb)));
    }
    // decode's offset shift (engine.cpp:418-424) composed with paging the way
    // bench.cpp:562-566 composes it: the bounded runtime mask of the logical
    // BlockMask is carried through convert_block_mask -> convert_mods.
    const MaskMod shifted = offset_mask(make_mask(*m, false), offset);
    const ScoreMod score_shifted = offset_score(make_score(*s, false), offset);
    const auto bm = create_block_mask(shifted, 1, 1, n_new, Lkv, page_size, page_size);
    const BlockMask bm_phys = convert_block_mask(bm, cache.table());
    const ConvertedMods mods = convert_mods(shifted, score_shifted, cache.table());
    const auto res = forward(tensor_from(q_step, B, Hq, n_new, D), cache.k_phys(), cache.v_phys(),
                             mods.score, bm_phys, cfg);
    std::memcpy(out, res.out.data().data(), res.out.data().size() * sizeof(float));
    std::memcpy(lse, res.lse.data(), res.lse.size() * sizeof(float));
    if (table_out) {
      const auto& t = cache.table().table;
      std::memcpy(table_out, t.data(), t.size() * sizeof(int32_t));
    }
    if (num_pages_out) *num_pages_out = num_pages;
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// convert_block_mask (paged_kv.cpp:154-228) on a logical mask built from `m`
// with an explicit page table (batches x max_logical_pages, -1 = unmapped).
int ref_convert_block_mask(const RefMask* m, int64_t bd, int64_t hd, int64_t ql, int64_t kl,
                           int64_t bs, int64_t batches, int64_t max_logical_pages,
                           int64_t num_physical_pages, const int32_t* table, int64_t* pn,
                           int64_t* pi, int64_t* fn, int64_t* fi) {
  try {
    const auto bm = create_block_mask(make_mask(*m), bd, hd, ql, kl, bs, bs);
    PageTable pt;
    pt.batches = batches;
    pt.max_logical_pages = max_logical_pages;
    pt.num_physical_pages = num_physical_pages;
    pt.page_size = bs;
    pt.table.assign(table, table + batches * max_logical_pages);
    pt.phys_to_logical.assign(static_cast<std::size_t>(num_physical_pages), -1);
    pt.owner.assign(static_cast<std::size_t>(num_physical_pages), -1);
    pt.seq_len.assign(static_cast<std::size_t>(batches), 0);
    const auto out = convert_block_mask(bm, pt);
    copy_bm(out, pn, pi, fn, fi, nullptr, nullptr, nullptr);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// PagedKVCache page table after construction, shuffle and assigning
// `tokens_per_batch` tokens to each batch (paged_kv.cpp:14-98, 143-146).
int ref_paged_layout(int64_t B, int64_t num_pages, int64_t page_size, uint64_t shuffle_seed,
                     int64_t tokens_per_batch, int32_t* table, int32_t* phys_to_logical,
                     int32_t* owner) {
  try {
    PagedKVCache<float> cache(B, num_pages, page_size, 1, 1);
    cache.shuffle_free_pages(shuffle_seed);
    Tensor4<float> t(1, 1, tokens_per_batch, 1);
    for (i64 b = 0; b < B; ++b) cache.assign(b, t, t);
    const auto& pt = cache.table();
    std::memcpy(table, pt.table.data(), pt.table.size() * sizeof(int32_t));
    std::memcpy(phys_to_logical, pt.phys_to_logical.data(), pt.phys_to_logical.size() * 4);
    std::memcpy(owner, pt.owner.data(), pt.owner.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// A script of PagedKVCache calls on the reference (paged_kv.cpp:13-152): op[i] 0 = assign,
// 1 = append_tokens, 2 = erase, 3 = shuffle_free_pages(seed[i]); n[i] tokens whose element
// (h, t, d) of the token tensor is tok[base + (h * n + t) * dim + d] (base = running sum of
// n * heads * dim over the token-carrying calls). status[i] = the call's error status (0 = ok;
// a failing call is caught and the script goes on). Outputs the final table, p2l, owner,
// seq_len, free page count and the physical K and V buffers (V = -K).
int ref_paged_script(int64_t B, int64_t num_pages, int64_t page_size, int64_t heads, int64_t dim,
                     int64_t n_ops, const int32_t* op, const int64_t* bat, const int64_t* n,
                     const uint64_t* seed, const float* tok, int32_t* status, int32_t* table,
                     int32_t* p2l, int32_t* owner, int64_t* seq, int64_t* free_pages, float* k_out,
                     float* v_out) {
  try {
    PagedKVCache<float> cache(B, num_pages, page_size, heads, dim);
    int64_t base = 0;
    for (int64_t i = 0; i < n_ops; ++i) {
      status[i] = 0;
      try {
        if (op[i] == 3) {
          cache.shuffle_free_pages(seed[i]);
        } else if (op[i] == 2) {
          cache.erase(bat[i]);
        } else {
          Tensor4<float> kt(1, heads, n[i], dim), vt(1, heads, n[i], dim);
          for (int64_t h = 0; h < heads; ++h)
            for (int64_t t = 0; t < n[i]; ++t)
              for (int64_t d = 0; d < dim; ++d) {
                const float x = tok[base + (h * n[i] + t) * dim + d];
                kt.at(0, h, t, d) = x;
                vt.at(0, h, t, d) = -x;
              }
          base += n[i] * heads * dim;
          if (op[i] == 0) cache.assign(bat[i], kt, vt);
          else cache.append_tokens(bat[i], kt, vt);
        }
      } catch (const std::exception& e) {
        status[i] = status_of(e);
      }
    }
    const auto& pt = cache.table();
    std::memcpy(table, pt.table.data(), pt.table.size() * sizeof(int32_t));
    std::memcpy(p2l, pt.phys_to_logical.data(), pt.phys_to_logical.size() * 4);
    std::memcpy(owner, pt.owner.data(), pt.owner.size() * 4);
    for (int64_t b = 0; b < B; ++b) seq[b] = cache.seq_len(b);
    *free_pages = cache.free_pages();
    const auto& kp = cache.k_phys();
    const auto& vp = cache.v_phys();
    std::memcpy(k_out, kp.data().data(), kp.data().size() * sizeof(float));
    std::memcpy(v_out, vp.data().data(), vp.data().size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

}  // extern "C"

// Timing entry for bench.py's CPU legs: the reference forward and backward on
// prebuilt masks (create_block_mask/transpose outside the timed region, as
// bench.cpp:412-426 builds them in build_point), each timed with steady_clock.
#include <chrono>
extern "C" int ref_time_fwd_bwd_f32(const float* q, const float* k, const float* v,
                                    const float* dout, int64_t B, int64_t Hq, int64_t Hkv,
                                    int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D, double scale,
                                    int64_t gqa, const RefScore* s, const RefMask* m, int64_t bs,
                                    int do_bwd, double* fwd_s, double* bwd_s) {
  try {
    AttentionConfig cfg;
    if (scale > 0) cfg.scale = scale;
    cfg.gqa_group = gqa;
    cfg.block_size_q = cfg.block_size_kv = bs;
    const auto bm = create_block_mask(make_mask(*m), 1, 1, Lq, Lkv, bs, bs);
    const auto bm_t = transpose(bm);
    const auto qt = tensor_from(q, B, Hq, Lq, D);
    const auto kt = tensor_from(k, Bkv, Hkv, Lkv, D);
    const auto vt = tensor_from(v, Bkv, Hkv, Lkv, D);
    const auto dot = tensor_from(dout, B, Hq, Lq, D);
    const auto smod = make_score(*s);
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const auto fwd = forward(qt, kt, vt, smod, bm, cfg);
    const auto t1 = clk::now();
    *fwd_s = std::chrono::duration<double>(t1 - t0).count();
    *bwd_s = 0.0;
    if (do_bwd) {
      const auto g = backward(qt, kt, vt, fwd, dot, smod, bm, bm_t, cfg);
      *bwd_s = std::chrono::duration<double>(clk::now() - t1).count();
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// OpCounters of the reference forward and backward (engine.hpp:21-32) on one problem:
// out6 = {fwd madds, fwd mask_evals, fwd score_evals, bwd madds, bwd mask_evals, bwd score_evals}.
extern "C" int ref_counters_f32(const float* q, const float* k, const float* v, const float* dout,
                                int64_t B, int64_t Hq, int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv,
                                int64_t D, double scale, int64_t gqa, const RefScore* s, const RefMask* m,
                                int64_t bs, uint64_t* out6) {
  try {
    AttentionConfig cfg;
    if (scale > 0) cfg.scale = scale;
    cfg.gqa_group = gqa;
    cfg.block_size_q = cfg.block_size_kv = bs;
    const auto bm = create_block_mask(make_mask(*m), 1, 1, Lq, Lkv, bs, bs);
    const auto bm_t = transpose(bm);
    const auto qt = tensor_from(q, B, Hq, Lq, D);
    const auto kt = tensor_from(k, Bkv, Hkv, Lkv, D);
    const auto vt = tensor_from(v, Bkv, Hkv, Lkv, D);
    const auto smod = make_score(*s);
    OpCounters cf, cb;
    const auto fwd = forward(qt, kt, vt, smod, bm, cfg, &cf);
    backward(qt, kt, vt, fwd, tensor_from(dout, B, Hq, Lq, D), smod, bm, bm_t, cfg, &cb);
    const uint64_t v6[6] = {cf.madds, cf.mask_evals, cf.score_evals, cb.madds, cb.mask_evals, cb.score_evals};
    std::copy(v6, v6 + 6, out6);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
