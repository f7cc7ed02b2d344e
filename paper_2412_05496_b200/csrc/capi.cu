// capi.cu — the extern "C" boundary (include/flexattn_b200.h): argument
// validation with the reference's error taxonomy (errors.hpp, engine.cpp:21-42,
// validate.cpp:16-34), dispatch of mask/score descriptors to the precompiled
// functor instantiations, synthetic-input generation and paged-KV scatter.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "internal.h"

namespace fa {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

fa_status set_error(fa_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
void clear_error() { g_last_error.clear(); }
fa_status cuda_status(cudaError_t e, const char* what) {
  return set_error(FA_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// Small device scratch words (dynamic tile-scheduler counters, device status flags), one
// 64-byte slot per (device, stream, slot id): the launcher zeroes it on the stream right before
// the kernel, so launches on one stream are ordered and launches on different streams never
// share a word.
int* scheduler_counter(int slot, cudaStream_t st) {
  static std::map<std::tuple<int, cudaStream_t, int>, int*> counters;
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  int*& c = counters[std::make_tuple(dev, st, slot)];
  if (c == nullptr && cudaMalloc(&c, 64) != cudaSuccess) c = nullptr;
  return c;
}

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

MaskParams to_mask_params(const fa_mask_desc& d) {
  MaskParams m{};
  m.terms = d.terms;
  m.hash_density = d.hash_density;
  m.window = static_cast<int32_t>(d.window);
  m.prefix = static_cast<int32_t>(d.prefix);
  m.q_offset = static_cast<int32_t>(d.q_offset);
  m.doc_len = static_cast<int32_t>(d.doc_len);
  m.hash_seed = d.hash_seed;
  m.doc_ids = d.doc_ids;
  m.or_terms = d.or_terms;
  m.na_w = static_cast<int32_t>(d.na_width);
  m.na_n = static_cast<int32_t>(d.na_height * d.na_width);
  m.na_radius = d.na_kernel / 2;
  m.remap = d.remap_len > 0 ? d.remap : nullptr;
  return m;
}

ScoreParams to_score_params(const fa_score_desc& d) {
  ScoreParams s{};
  s.terms = d.terms;
  s.q_offset = static_cast<int32_t>(d.q_offset);
  s.cap = static_cast<float>(d.cap);
  s.inv_cap = d.cap > 0 ? static_cast<float>(1.0 / d.cap) : 0.f;
  s.slopes = d.slopes;
  return s;
}

int mask_kind_of(const fa_mask_desc& d) {
  if (d.or_terms != 0 || d.remap_len > 0) return kMaskDynamic;
  const uint32_t terms = d.terms;
  if (terms == 0) return kMaskNoop;
  if (terms == kMaskCausal) return kMaskCausalOnly;
  if (terms == kMaskSliding || terms == (kMaskSliding | kMaskCausal)) return kMaskSlidingOnly;
  if (terms == (kMaskDocument | kMaskCausal)) return kMaskDocCausal;
  return kMaskDynamic;
}

// Checks of the mask terms that the reference performs when it builds or evaluates the
// mask (GeometryMismatch / IndexOutOfRange): positions q in [q_offset, q_len + q_offset),
// kv in [0, kv_len) must be inside every table the terms index.
fa_status check_mask_desc(const fa_mask_desc& m, int64_t q_len, int64_t kv_len) {
  FA_REQUIRE(!(m.terms & ~0x7Fu) && !(m.or_terms & ~0x7Fu), FA_SHAPE_MISMATCH, "mask: unknown term bits");
  const uint32_t all = m.terms | m.or_terms;
  if (all & kMaskSliding)
    FA_REQUIRE(m.window >= 0, FA_INDEX_OUT_OF_RANGE, "sliding_window: window must be >= 0");
  if (all & kMaskPrefix)
    FA_REQUIRE(m.prefix >= 0, FA_INDEX_OUT_OF_RANGE, "prefix_lm: prefix_len must be >= 0");
  const int64_t q_end = q_len + m.q_offset;
  if (m.remap_len > 0) {  // remap_mask range check, mask_library.cpp:208-211
    FA_REQUIRE(m.remap != nullptr, FA_SHAPE_MISMATCH, "remap_mask: table is NULL");
    FA_REQUIRE(m.q_offset >= 0 && q_end <= m.remap_len && kv_len <= m.remap_len, FA_INDEX_OUT_OF_RANGE,
               "remap_mask: slot index outside permutation of size " + std::to_string(m.remap_len));
  }
  // with a remap the terms see permuted tokens in [0, remap_len)
  const int64_t q_hi = m.remap_len > 0 ? m.remap_len : q_end;
  const int64_t kv_hi = m.remap_len > 0 ? m.remap_len : kv_len;
  if (all & kMaskDocument) {
    FA_REQUIRE(m.doc_ids != nullptr, FA_SHAPE_MISMATCH, "document_mask: doc_ids is NULL");
    // the reference throws IndexOutOfRange on the first out-of-table index (mask_library.cpp:27-31)
    FA_REQUIRE(m.doc_len >= q_hi && m.doc_len >= kv_hi && q_end > 0, FA_INDEX_OUT_OF_RANGE,
               "document_mask: token index outside id table of size " + std::to_string(m.doc_len));
  }
  if (all & kMaskNatten) {  // NAGeometry, mask_library.cpp:121-135; na_naive range :141-144
    FA_REQUIRE(m.na_height >= 1 && m.na_width >= 1, FA_GEOMETRY_MISMATCH,
               "NAGeometry: canvas dims must be >= 1");
    FA_REQUIRE(m.na_kernel >= 1 && m.na_kernel % 2 == 1, FA_GEOMETRY_MISMATCH,
               "NAGeometry: kernel must be odd and >= 1");
    FA_REQUIRE(m.na_kernel <= std::min(m.na_height, m.na_width), FA_GEOMETRY_MISMATCH,
               "NAGeometry: kernel exceeds canvas");
    const int64_t n = m.na_height * m.na_width;
    FA_REQUIRE(q_hi <= n && kv_hi <= n && m.q_offset >= 0, FA_INDEX_OUT_OF_RANGE,
               "na_naive: token index outside canvas of " + std::to_string(n) + " pixels");
  }
  return FA_OK;
}

}  // namespace fa

using namespace fa;

namespace {

fa_status check_tensor(const fa_tensor& t, const char* name) {
  FA_REQUIRE(t.data != nullptr, FA_SHAPE_MISMATCH, std::string(name) + ": NULL data");
  FA_REQUIRE(t.b > 0 && t.h > 0 && t.l > 0 && t.d > 0, FA_SHAPE_MISMATCH,
             std::string(name) + ": all dims must be positive");
  FA_REQUIRE(t.dtype == FA_F32 || t.dtype == FA_BF16, FA_UNSUPPORTED,
             std::string(name) + ": dtype must be FA_F32 or FA_BF16");
  return FA_OK;
}

bool same_shape(const fa_tensor& a, const fa_tensor& b) {
  return a.b == b.b && a.h == b.h && a.l == b.l && a.d == b.d;
}

std::string shp(const fa_tensor& t) {
  return "(" + std::to_string(t.b) + "," + std::to_string(t.h) + "," + std::to_string(t.l) + "," +
         std::to_string(t.d) + ")";
}

// validate_shapes (validate.cpp:16-34) + gqa divisibility (config.hpp:33-45)
fa_status check_qkv(const fa_tensor& q, const fa_tensor& k, const fa_tensor& v, int64_t gqa) {
  fa_status s;
  if ((s = check_tensor(q, "q")) || (s = check_tensor(k, "k")) || (s = check_tensor(v, "v"))) return s;
  FA_REQUIRE(k.b == v.b && k.h == v.h && k.l == v.l && k.d == v.d, FA_SHAPE_MISMATCH,
             "k " + shp(k) + " and v " + shp(v) + " must have the same shape");
  FA_REQUIRE(q.d == k.d, FA_SHAPE_MISMATCH, "q head dim must match k");
  FA_REQUIRE(k.b == 1 || k.b == q.b, FA_SHAPE_MISMATCH, "kv batch must be 1 or the q batch");
  FA_REQUIRE(gqa >= 1, FA_SHAPE_MISMATCH, "gqa_group must be >= 1");
  FA_REQUIRE(q.h == gqa * k.h, FA_SHAPE_MISMATCH,
             "q heads " + std::to_string(q.h) + " != gqa_group * kv heads " +
                 std::to_string(gqa * k.h));
  FA_REQUIRE(q.dtype == k.dtype && k.dtype == v.dtype, FA_SHAPE_MISMATCH, "q/k/v dtypes differ");
  return FA_OK;
}

// check_block_mask (engine.cpp:21-42)
fa_status check_bm(const fa_block_mask* bm, int64_t batch, int64_t heads, int64_t q_len,
                   int64_t kv_len) {
  FA_REQUIRE(bm != nullptr && bm->kv_num_blocks && bm->kv_indices && bm->full_kv_num_blocks &&
                 bm->full_kv_indices,
             FA_BLOCK_MASK_MISMATCH, "block mask kv-side arrays missing");
  FA_REQUIRE(bm->q_len == q_len && bm->kv_len == kv_len, FA_BLOCK_MASK_MISMATCH,
             "block mask covers " + std::to_string(bm->q_len) + "x" + std::to_string(bm->kv_len) +
                 " but tensors are " + std::to_string(q_len) + "x" + std::to_string(kv_len));
  FA_REQUIRE(bm->b_dims == 1 || bm->b_dims == batch, FA_BLOCK_MASK_MISMATCH,
             "block mask batch dim must be 1 or " + std::to_string(batch));
  FA_REQUIRE(bm->h_dims == 1 || bm->h_dims == heads, FA_BLOCK_MASK_MISMATCH,
             "block mask head dim must be 1 or " + std::to_string(heads));
  FA_REQUIRE(bm->rows == (bm->q_len + bm->bs_q - 1) / bm->bs_q &&
                 bm->cols == (bm->kv_len + bm->bs_kv - 1) / bm->bs_kv,
             FA_BLOCK_MASK_MISMATCH, "block mask rows/cols inconsistent with lengths");
  return FA_OK;
}

fa_status check_mods(const fa_mask_desc& m, const fa_score_desc& s, int64_t heads, int64_t q_len,
                     int64_t kv_len) {
  FA_REQUIRE(!(s.terms & ~0x3u), FA_SHAPE_MISMATCH, "score: unknown term bits");
  fa_status st;
  if ((st = check_mask_desc(m, q_len, kv_len)) != FA_OK) return st;
  if (s.terms & kScoreAlibi) {
    FA_REQUIRE(s.slopes != nullptr, FA_SHAPE_MISMATCH, "alibi: slopes is NULL");
    FA_REQUIRE(s.num_slopes >= heads, FA_INDEX_OUT_OF_RANGE,
               "alibi: head " + std::to_string(heads - 1) + " outside slope table of size " +
                   std::to_string(s.num_slopes));
  }
  if (s.terms & kScoreSoftCap)
    FA_REQUIRE(s.cap > 0 && std::isfinite(s.cap), FA_NON_POSITIVE_CAP,
               "soft_cap: cap must be finite and > 0");
  return FA_OK;
}

AttnGeom geom_of(const fa_tensor& q, const fa_tensor& k, const fa_block_mask* bm, double scale,
                 int64_t gqa) {
  AttnGeom g{};
  g.B = (int)q.b; g.Hq = (int)q.h; g.Hkv = (int)k.h; g.Bkv = (int)k.b; g.Lq = (int)q.l;
  g.Lkv = (int)k.l; g.D = (int)q.d; g.G = (int)gqa;
  g.bm_b = (int)bm->b_dims; g.bm_h = (int)bm->h_dims; g.rows = (int)bm->rows; g.cols = (int)bm->cols;
  g.bs_q = (int)bm->bs_q; g.bs_kv = (int)bm->bs_kv;
  g.scale = static_cast<float>(scale > 0 ? scale : 1.0 / std::sqrt(static_cast<double>(q.d)));
  return g;
}

BmView kv_view(const fa_block_mask* bm) {
  return BmView{bm->kv_num_blocks, bm->kv_indices, bm->full_kv_num_blocks, bm->full_kv_indices};
}

}  // namespace

extern "C" {

const char* fa_last_error(void) { return g_last_error.c_str(); }
int32_t fa_abi_version(void) { return 4; }  // v3: flags, counters, phase events, fa_check_finite; v4: device page pool
uint64_t fa_launch_count(void) { return g_launches.load(); }

const char* fa_status_name(fa_status s) {
  switch (s) {
    case FA_OK: return "OK";
    case FA_SHAPE_MISMATCH: return "ShapeMismatch";
    case FA_NON_FINITE_INPUT: return "NonFiniteInput";
    case FA_INDEX_OUT_OF_RANGE: return "IndexOutOfRange";
    case FA_NON_POSITIVE_CAP: return "NonPositiveCap";
    case FA_GEOMETRY_MISMATCH: return "GeometryMismatch";
    case FA_BLOCK_MASK_MISMATCH: return "BlockMaskMismatch";
    case FA_STALE_STATISTICS: return "StaleStatistics";
    case FA_OFFSET_OUT_OF_RANGE: return "OffsetOutOfRange";
    case FA_OUT_OF_PAGES: return "OutOfPages";
    case FA_UNMAPPED_BLOCK: return "UnmappedBlock";
    case FA_UNMAPPED_PHYSICAL_INDEX: return "UnmappedPhysicalIndex";
    case FA_CUDA_ERROR: return "CudaError";
    case FA_UNSUPPORTED: return "Unsupported";
    default: return "Unknown";
  }
}

fa_status fa_flex_fwd(const fa_fwd_args* a, void* stream) {
  clear_error();
  FA_REQUIRE(a != nullptr, FA_SHAPE_MISMATCH, "forward: NULL args");
  fa_status s;
  if ((s = check_qkv(a->q, a->k, a->v, a->gqa_group))) return s;
  if ((s = check_tensor(a->out, "out"))) return s;
  FA_REQUIRE(a->out.b == a->q.b && a->out.h == a->q.h && a->out.l == a->q.l && a->out.d == a->q.d &&
                 a->out.dtype == a->q.dtype,
             FA_SHAPE_MISMATCH, "out must match q");
  FA_REQUIRE(a->lse != nullptr, FA_SHAPE_MISMATCH, "forward: NULL lse");
  if ((s = check_bm(a->bm, a->q.b, a->q.h, a->q.l, a->k.l))) return s;
  if ((s = check_mods(a->mask, a->score, a->q.h, a->q.l, a->k.l))) return s;
  const AttnGeom g = geom_of(a->q, a->k, a->bm, a->scale, a->gqa_group);
  const MaskParams mp = to_mask_params(a->mask);
  const ScoreParams sp = to_score_params(a->score);
  const int mk = mask_kind_of(a->mask);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  FA_REQUIRE(!(a->flags & ~uint32_t(FA_FLAG_VALIDATE)), FA_SHAPE_MISMATCH, "forward: unknown flags");
  if (a->flags & FA_FLAG_VALIDATE) {  // validate_inputs (validate.hpp:36-38)
    const fa_tensor ts[3] = {a->q, a->k, a->v};
    const char* names[3] = {"q", "k", "v"};
    if ((s = check_finite_list(ts, names, 3, st)) != FA_OK) return s;
  }
  if (a->q.dtype == FA_BF16 && fwd_sm100_supported(g))
    s = launch_fwd_sm100(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, kv_view(a->bm),
                         mp, mk, sp, (int)a->score.terms, st);
  else
    s = launch_fwd_simt(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, a->q.dtype,
                        kv_view(a->bm), mp, mk, sp, (int)a->score.terms, st);
  if (s != FA_OK || a->counters == nullptr) return s;
  return compute_counters(g, kv_view(a->bm), mp, mk, nullptr, g.Lkv, kPassForward, a->counters, st);
}

size_t fa_bwd_workspace_size(int64_t batch, int64_t heads, int64_t q_len, int64_t dim) {
  // dq accumulator (fp32) + delta (fp32) + log2-domain lse (fp32), 256-byte aligned pieces
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t rows = static_cast<size_t>(batch * heads * q_len);
  const size_t prow = static_cast<size_t>(batch * heads * ((q_len + 127) / 128 * 128));
  const size_t qblocks = static_cast<size_t>(batch * heads * ((q_len + 127) / 128));
  // + per-(b, h, q block) turn counters of the deterministic dQ order
  return al(rows * dim * 4) + al(prow * 4) + al(prow * 4) + al(qblocks * 4);
}

fa_status fa_flex_bwd(const fa_bwd_args* a, void* stream) {
  clear_error();
  FA_REQUIRE(a != nullptr, FA_SHAPE_MISMATCH, "backward: NULL args");
  fa_status s;
  if ((s = check_qkv(a->q, a->k, a->v, a->gqa_group))) return s;
  if ((s = check_tensor(a->out, "out")) || (s = check_tensor(a->d_out, "d_out")) ||
      (s = check_tensor(a->dq, "dq")) || (s = check_tensor(a->dk, "dk")) ||
      (s = check_tensor(a->dv, "dv")))
    return s;
  FA_REQUIRE(same_shape(a->d_out, a->q) && a->d_out.dtype == a->q.dtype, FA_SHAPE_MISMATCH,
             "backward: d_out " + shp(a->d_out) + " must match q " + shp(a->q));
  FA_REQUIRE(same_shape(a->dq, a->q) && a->dq.dtype == a->q.dtype, FA_SHAPE_MISMATCH,
             "backward: dq " + shp(a->dq) + " must match q " + shp(a->q));
  FA_REQUIRE(same_shape(a->dk, a->k) && same_shape(a->dv, a->k) && a->dk.dtype == a->q.dtype &&
                 a->dv.dtype == a->q.dtype,
             FA_SHAPE_MISMATCH, "backward: dk/dv must match k " + shp(a->k));
  FA_REQUIRE(a->out.dtype == a->q.dtype, FA_STALE_STATISTICS,
             "backward: saved forward output has another dtype than q");
  FA_REQUIRE(a->out.b == a->q.b && a->out.h == a->q.h && a->out.l == a->q.l && a->out.d == a->q.d,
             FA_STALE_STATISTICS, "backward: saved forward statistics do not match these tensors");
  FA_REQUIRE(a->lse != nullptr, FA_STALE_STATISTICS, "backward: NULL lse");
  if ((s = check_bm(a->bm, a->q.b, a->q.h, a->q.l, a->k.l))) return s;
  FA_REQUIRE(a->bm->q_num_blocks && a->bm->q_indices && a->bm->full_q_num_blocks &&
                 a->bm->full_q_indices,
             FA_BLOCK_MASK_MISMATCH, "backward: q-side (transposed) arrays required");
  if ((s = check_mods(a->mask, a->score, a->q.h, a->q.l, a->k.l))) return s;
  FA_REQUIRE(a->workspace != nullptr &&
                 a->workspace_bytes >= fa_bwd_workspace_size(a->q.b, a->q.h, a->q.l, a->q.d),
             FA_SHAPE_MISMATCH, "backward: workspace too small");
  FA_REQUIRE(!(a->flags & ~uint32_t(FA_FLAG_VALIDATE | FA_FLAG_DETERMINISTIC)), FA_SHAPE_MISMATCH,
             "backward: unknown flags");
  const AttnGeom g = geom_of(a->q, a->k, a->bm, a->scale, a->gqa_group);
  const BmView bmt{a->bm->q_num_blocks, a->bm->q_indices, a->bm->full_q_num_blocks,
                   a->bm->full_q_indices};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool tc_path = a->q.dtype == FA_BF16 && bwd_sm100_supported(g);
  BwdOptions opt;
  opt.flags = a->flags;
  for (int i = 0; i < 4; ++i) opt.events[i] = static_cast<cudaEvent_t>(a->phase_events[i]);
  if (a->flags & FA_FLAG_VALIDATE) {
    // q/k/v as validate_inputs; d_out (engine.cpp:196) is checked inside the tensor-core
    // path's preprocess read of d_out, else scanned here
    const fa_tensor ts[4] = {a->q, a->k, a->v, a->d_out};
    const char* names[4] = {"q", "k", "v", "d_out"};
    if ((s = check_finite_list(ts, names, tc_path ? 3 : 4, st)) != FA_OK) return s;
    if (tc_path) {
      opt.dout_nonfinite = scheduler_counter(kSlotFiniteErr, st);
      FA_REQUIRE(opt.dout_nonfinite != nullptr, FA_CUDA_ERROR, "backward: status word");
      FA_CHECK_CUDA(cudaMemsetAsync(opt.dout_nonfinite, 0, sizeof(int), st));
    }
  }
  const MaskParams mp = to_mask_params(a->mask);
  const int mk = mask_kind_of(a->mask);
  s = launch_bwd(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, a->d_out.data, a->dq.data,
                 a->dk.data, a->dv.data, a->q.dtype, kv_view(a->bm), bmt, mp, mk,
                 to_score_params(a->score), (int)a->score.terms, a->workspace, opt, st);
  if (s != FA_OK) return s;
  if (opt.dout_nonfinite != nullptr) {
    int bad = 0;
    FA_CHECK_CUDA(cudaMemcpyAsync(&bad, opt.dout_nonfinite, sizeof(int), cudaMemcpyDeviceToHost, st));
    FA_CHECK_CUDA(cudaStreamSynchronize(st));
    FA_REQUIRE(bad == 0, FA_NON_FINITE_INPUT, "backward: d_out contains NaN or inf");
  }
  if (a->counters == nullptr) return FA_OK;
  return compute_counters(g, kv_view(a->bm), mp, mk, nullptr, g.Lkv, kPassBackward, a->counters, st);
}

size_t fa_decode_workspace_size(int64_t batch, int64_t heads, int64_t n_new, int64_t dim,
                                int32_t num_splits) {
  if (num_splits <= 1) num_splits = 64;  // upper bound of the automatic choice
  return static_cast<size_t>(batch * heads * n_new) * num_splits * (dim + 2) * 4;
}

fa_status fa_flex_decode(const fa_decode_args* a, void* stream) {
  clear_error();
  FA_REQUIRE(a != nullptr, FA_SHAPE_MISMATCH, "decode: NULL args");
  FA_REQUIRE(a->bm != nullptr, FA_BLOCK_MASK_MISMATCH, "decode: NULL block mask");
  fa_status s;
  if ((s = check_qkv(a->q, a->k_cache, a->v_cache, a->gqa_group))) return s;
  if ((s = check_tensor(a->out, "out"))) return s;
  FA_REQUIRE(same_shape(a->out, a->q) && a->out.dtype == a->q.dtype, FA_SHAPE_MISMATCH,
             "decode: out " + shp(a->out) + " must match q " + shp(a->q));
  FA_REQUIRE(a->lse != nullptr, FA_SHAPE_MISMATCH, "decode: NULL lse");
  FA_REQUIRE(a->q.dtype == FA_BF16 || a->pt == nullptr, FA_UNSUPPORTED,
             "decode: a paged cache needs bf16 (float32 decode is unpaged)");
  const int64_t n_new = a->q.l;
  int64_t logical_kv = a->k_cache.l;
  if (a->pt != nullptr) {
    const fa_page_table* pt = a->pt;
    FA_REQUIRE(pt->table && pt->phys_to_logical && pt->owner && pt->seq_len, FA_SHAPE_MISMATCH,
               "decode: page table arrays missing");
    FA_REQUIRE(a->k_cache.b == 1, FA_SHAPE_MISMATCH, "decode: paged cache must have batch 1");
    FA_REQUIRE(pt->batches == a->q.b, FA_SHAPE_MISMATCH, "decode: page table batches must equal q batch");
    FA_REQUIRE(pt->page_size == a->bm->bs_kv, FA_BLOCK_MASK_MISMATCH,
               "decode: page size must equal bs_kv");
    FA_REQUIRE(a->k_cache.l == pt->num_physical_pages * pt->page_size, FA_SHAPE_MISMATCH,
               "decode: physical cache length must be pages * page_size");
    // a converted mask (convert_block_mask): batch materialised, one column per physical page
    FA_REQUIRE(a->bm->b_dims == a->q.b, FA_BLOCK_MASK_MISMATCH,
               "decode: converted block mask must materialise the batch");
    FA_REQUIRE(a->bm->h_dims == 1 || a->bm->h_dims == a->q.h, FA_BLOCK_MASK_MISMATCH,
               "decode: block mask head dim must be 1 or " + std::to_string(a->q.h));
    FA_REQUIRE(a->bm->q_len == n_new && a->bm->kv_len == a->k_cache.l && a->bm->bs_q >= 1 &&
                   a->bm->rows == (n_new + a->bm->bs_q - 1) / a->bm->bs_q &&
                   a->bm->cols == pt->num_physical_pages,
               FA_BLOCK_MASK_MISMATCH,
               "decode: converted block mask geometry does not match the physical cache");
    FA_REQUIRE(a->bm->kv_num_blocks && a->bm->kv_indices && a->bm->full_kv_num_blocks &&
                   a->bm->full_kv_indices,
               FA_BLOCK_MASK_MISMATCH, "decode: block mask kv-side arrays missing");
    logical_kv = pt->max_logical_pages * pt->page_size;
    FA_REQUIRE(pt->max_seq_len >= 0 && pt->max_seq_len <= logical_kv, FA_SHAPE_MISMATCH,
               "decode: page table max_seq_len outside [0, max_logical_pages * page_size]");
  }
  // kv positions the mask can be evaluated at (the paged kernel also stops at each seq_len)
  const int64_t mask_kv = (a->pt && a->pt->max_seq_len > 0) ? a->pt->max_seq_len : logical_kv;
  // engine.cpp:410-414
  FA_REQUIRE(a->offset >= 0 && a->offset + n_new <= logical_kv, FA_OFFSET_OUT_OF_RANGE,
             "decode: rows [" + std::to_string(a->offset) + ", " + std::to_string(a->offset + n_new) +
                 ") fall outside cache");
  if (a->pt == nullptr) {
    if ((s = check_bm(a->bm, a->q.b, a->q.h, n_new, a->k_cache.l))) return s;
  }
  fa_mask_desc m = a->mask;
  fa_score_desc sc = a->score;
  m.q_offset += a->offset;  // offset_mask / offset_score (mask_library.cpp:106-119)
  sc.q_offset += a->offset;
  // the kernels evaluate the mask at logical kv positions up to logical_kv - 1
  if ((s = check_mods(m, sc, a->q.h, n_new, mask_kv))) return s;
  FA_REQUIRE(!(a->flags & ~uint32_t(FA_FLAG_VALIDATE)), FA_SHAPE_MISMATCH, "decode: unknown flags");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a->flags & FA_FLAG_VALIDATE) {  // decode -> forward_impl -> validate_inputs
    const fa_tensor ts[3] = {a->q, a->k_cache, a->v_cache};
    const char* names[3] = {"q", "k", "v"};
    if ((s = check_finite_list(ts, names, 3, st)) != FA_OK) return s;
  }
  if (a->q.dtype == FA_F32) {
    // decode<float> is forward_impl over the shifted mask (engine.cpp:403-427): the fp32
    // CUDA-core forward with q_offset applied to the mask and score terms
    const AttnGeom ga = geom_of(a->q, a->k_cache, a->bm, a->scale, a->gqa_group);
    s = launch_fwd_simt(ga, a->q.data, a->k_cache.data, a->v_cache.data, a->out.data, a->lse, FA_F32,
                        kv_view(a->bm), to_mask_params(m), mask_kind_of(m), to_score_params(sc),
                        (int)sc.terms, st);
    if (s != FA_OK || a->counters == nullptr) return s;
    return compute_counters(ga, kv_view(a->bm), to_mask_params(m), mask_kind_of(m), nullptr, (int)ga.Lkv,
                            kPassForward, a->counters, st);
  }
  DecodeGeom g{};
  g.a = geom_of(a->q, a->k_cache, a->bm, a->scale, a->gqa_group);
  g.logical_kv = (int)mask_kv;
  int splits = a->num_splits;
  if (splits <= 0) {
    const int64_t rows_total = a->q.b * a->q.h * n_new;
    const int64_t want = (2LL * num_sms() + rows_total - 1) / rows_total;
    splits = (int)std::max<int64_t>(1, std::min<int64_t>(want, std::min<int64_t>(64, a->bm->cols)));
  }
  g.num_splits = splits;
  if (splits > 1)
    FA_REQUIRE(a->workspace != nullptr &&
                   a->workspace_bytes >= fa_decode_workspace_size(a->q.b, a->q.h, n_new, a->q.d, splits),
               FA_SHAPE_MISMATCH, "decode: workspace too small");
  PageView pv{};
  if (a->pt) {
    pv.phys_to_logical = a->pt->phys_to_logical;
    pv.owner = a->pt->owner;
    pv.seq_len = a->pt->seq_len;
    pv.page_size = (int)a->pt->page_size;
    pv.enabled = 1;
    if (a->flags & FA_FLAG_VALIDATE) {  // foreign pages -> UnmappedPhysicalIndex (paged_kv.cpp:265-269)
      pv.foreign = scheduler_counter(kSlotConvertErr, st);
      FA_REQUIRE(pv.foreign != nullptr, FA_CUDA_ERROR, "decode: status word");
      FA_CHECK_CUDA(cudaMemsetAsync(pv.foreign, 0, sizeof(int), st));
    }
  }
  const MaskParams mp = to_mask_params(m);
  const int mk = mask_kind_of(m);
  s = launch_decode(g, a->q.data, a->k_cache.data, a->v_cache.data, a->out.data, a->lse, kv_view(a->bm),
                    pv, mp, mk, to_score_params(sc), (int)sc.terms, a->workspace, st);
  if (s != FA_OK) return s;
  if (pv.foreign != nullptr) {
    int bad = 0;
    FA_CHECK_CUDA(cudaMemcpyAsync(&bad, pv.foreign, sizeof(int), cudaMemcpyDeviceToHost, st));
    FA_CHECK_CUDA(cudaStreamSynchronize(st));
    FA_REQUIRE(bad == 0, FA_UNMAPPED_PHYSICAL_INDEX,
               "converted modifier: a visited physical page is not mapped for its batch element");
  }
  if (a->counters == nullptr) return FA_OK;
  return compute_counters(g.a, kv_view(a->bm), mp, mk, &pv, g.logical_kv, kPassForward, a->counters, st);
}

}  // extern "C"

// ---- synthetic inputs and paged scatter ---------------------------------------
namespace {

__global__ void fill_uniform_kernel(void* dst, int dtype, uint64_t seed, long long first,
                                    long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    // SplitMix64 draw (first + i): state = seed + (first + i + 1) * golden (random.hpp:21-26)
    uint64_t z = seed + static_cast<uint64_t>(first + i + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    const double unit = static_cast<double>(z >> 11) * 0x1.0p-53;  // next_unit (random.hpp:29)
    const float f = static_cast<float>(unit * 2.0 - 1.0);          // next_pm1 -> (Real)
    if (dtype == FA_F32) static_cast<float*>(dst)[i] = f;
    else static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(f);
  }
}

// PagedKVCache::write_tokens (paged_kv.cpp:54-70): 16-byte chunks.
__global__ void paged_write_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int B,
                                   int H, int L, int chunks_per_row, const int32_t* __restrict__ table,
                                   int max_logical_pages, int page_size, long long phys_len) {
  const long long total = (long long)B * H * L * chunks_per_row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(i % chunks_per_row);
    const long long tok = i / chunks_per_row;
    const int t = (int)(tok % L);
    const int h = (int)((tok / L) % H);
    const int b = (int)(tok / ((long long)L * H));
    const int page = table[(long long)b * max_logical_pages + t / page_size];
    if (page < 0) continue;
    const long long phys = (long long)page * page_size + t % page_size;
    dst[((long long)h * phys_len + phys) * chunks_per_row + ch] = src[i];
  }
}

}  // namespace

extern "C" fa_status fa_fill_uniform(void* dst, int32_t dtype, uint64_t seed, int64_t first,
                                     int64_t n, void* stream) {
  clear_error();
  FA_REQUIRE(dst != nullptr && n >= 0 && first >= 0, FA_SHAPE_MISMATCH, "fill_uniform: bad args");
  FA_REQUIRE(dtype == FA_F32 || dtype == FA_BF16, FA_UNSUPPORTED, "fill_uniform: dtype");
  if (n == 0) return FA_OK;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 32);
  fill_uniform_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, dtype, seed,
                                                                              first, n);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

extern "C" fa_status fa_paged_write(const fa_tensor* lg, const fa_page_table* pt, fa_tensor* ph,
                                    void* stream) {
  clear_error();
  FA_REQUIRE(lg && pt && ph && lg->data && ph->data, FA_SHAPE_MISMATCH, "paged_write: NULL argument");
  FA_REQUIRE(lg->dtype == ph->dtype && lg->d == ph->d && lg->h == ph->h && ph->b == 1,
             FA_SHAPE_MISMATCH, "paged_write: physical must be (1, H, pages*ps, D) like logical");
  FA_REQUIRE(ph->l == pt->num_physical_pages * pt->page_size, FA_SHAPE_MISMATCH,
             "paged_write: physical length must be pages * page_size");
  FA_REQUIRE(lg->b == pt->batches && lg->l <= pt->max_logical_pages * pt->page_size,
             FA_SHAPE_MISMATCH, "paged_write: logical tokens exceed the page table");
  const int esz = lg->dtype == FA_F32 ? 4 : 2;
  FA_REQUIRE((lg->d * esz) % 16 == 0, FA_UNSUPPORTED, "paged_write: row bytes must be a multiple of 16");
  const int cpr = (int)(lg->d * esz / 16);
  const long long total = lg->b * lg->h * lg->l * cpr;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  paged_write_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(lg->data), static_cast<uint4*>(ph->data), (int)lg->b, (int)lg->h,
      (int)lg->l, cpr, pt->table, (int)pt->max_logical_pages, (int)pt->page_size, ph->l);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}
