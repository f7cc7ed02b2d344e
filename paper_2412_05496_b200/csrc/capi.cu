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
#include "flexattn_b200/entry.cuh"

namespace fa {

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
  m.remap_rc = (m.remap != nullptr && d.terms == kMaskNatten && d.or_terms == 0) ? d.remap_rc : nullptr;
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
  FA_REQUIRE(m.remap_rc == nullptr || m.remap_len > 0, FA_SHAPE_MISMATCH, "remap_mask: remap_rc without a remap");
  if (m.remap_rc != nullptr)
    FA_REQUIRE(m.na_width < 65536 && m.na_height < 65536, FA_UNSUPPORTED,
               "remap_mask: the (row, col) table needs canvas dims < 65536");
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

namespace capi_detail {

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

}  // namespace capi_detail

using namespace capi_detail;

extern "C" {

const char* fa_last_error(void) { return last_error_ref().c_str(); }
int32_t fa_abi_version(void) { return 6; }  // v3: flags, counters, phase events, fa_check_finite; v4: device page pool; v5: remap_rc; v6: async convert
uint64_t fa_launch_count(void) { return launch_counter().load(); }

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
  AttnGeom g;
  fa_status s;
  if ((s = prepare_fwd(a, &g)) != FA_OK) return s;
  if ((s = check_mods(a->mask, a->score, a->q.h, a->q.l, a->k.l))) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((s = begin_fwd(a, st)) != FA_OK) return s;
  const MaskParams mp = to_mask_params(a->mask);
  const ScoreParams sp = to_score_params(a->score);
  const int mk = mask_kind_of(a->mask);
  if (a->q.dtype == FA_BF16 && fwd_sm100_supported(g))
    s = launch_fwd_sm100(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, kv_view(a->bm),
                         mp, mk, sp, (int)a->score.terms, st);
  else
    s = launch_fwd_simt(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, a->q.dtype,
                        kv_view(a->bm), mp, mk, sp, (int)a->score.terms, st);
  if (s != FA_OK || a->counters == nullptr) return s;
  return counters_by_desc(g, kv_view(a->bm), mp, mk, nullptr, g.Lkv, kPassForward, a->counters, st);
}

size_t fa_bwd_workspace_size(int64_t batch, int64_t heads, int64_t q_len, int64_t dim) {
  return bwd_workspace_bytes(batch, heads, q_len, dim);
}

fa_status fa_flex_bwd(const fa_bwd_args* a, void* stream) {
  clear_error();
  AttnGeom g;
  fa_status s;
  if ((s = prepare_bwd(a, &g)) != FA_OK) return s;
  if ((s = check_mods(a->mask, a->score, a->q.h, a->q.l, a->k.l))) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool tc_path = a->q.dtype == FA_BF16 && bwd_sm100_supported(g);
  BwdOptions opt;
  if ((s = begin_bwd(a, tc_path, &opt, st)) != FA_OK) return s;
  const MaskParams mp = to_mask_params(a->mask);
  const int mk = mask_kind_of(a->mask);
  s = launch_bwd(g, a->q.data, a->k.data, a->v.data, a->out.data, a->lse, a->d_out.data, a->dq.data,
                 a->dk.data, a->dv.data, a->q.dtype, kv_view(a->bm), q_view(a->bm), mp, mk,
                 to_score_params(a->score), (int)a->score.terms, a->workspace, opt, st);
  if (s != FA_OK) return s;
  if ((s = end_bwd(opt, st)) != FA_OK) return s;
  if (a->counters == nullptr) return FA_OK;
  return counters_by_desc(g, kv_view(a->bm), mp, mk, nullptr, g.Lkv, kPassBackward, a->counters, st);
}

size_t fa_decode_workspace_size(int64_t batch, int64_t heads, int64_t n_new, int64_t dim,
                                int32_t num_splits) {
  return decode_workspace_bytes(batch, heads, n_new, dim, num_splits);
}

fa_status fa_flex_decode(const fa_decode_args* a, void* stream) {
  clear_error();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DecodePlan plan;
  fa_status s;
  if ((s = prepare_decode(a, &plan, st)) != FA_OK) return s;
  fa_mask_desc m = a->mask;
  fa_score_desc sc = a->score;
  m.q_offset += a->offset;  // offset_mask / offset_score (mask_library.cpp:106-119)
  sc.q_offset += a->offset;
  // the kernels evaluate the mask at logical kv positions up to logical_kv - 1
  if ((s = check_mods(m, sc, a->q.h, a->q.l, plan.mask_kv))) return s;
  if ((s = begin_decode(a, &plan, st)) != FA_OK) return s;
  const MaskParams mp = to_mask_params(m);
  const int mk = mask_kind_of(m);
  if (a->q.dtype == FA_F32) {
    // decode<float> is forward_impl over the shifted mask (engine.cpp:403-427): the fp32
    // CUDA-core forward with q_offset applied to the mask and score terms
    s = launch_fwd_simt(plan.g.a, a->q.data, a->k_cache.data, a->v_cache.data, a->out.data, a->lse, FA_F32,
                        kv_view(a->bm), mp, mk, to_score_params(sc), (int)sc.terms, st);
    if (s != FA_OK || a->counters == nullptr) return s;
    return counters_by_desc(plan.g.a, kv_view(a->bm), mp, mk, nullptr, plan.g.a.Lkv, kPassForward, a->counters, st);
  }
  s = launch_decode(plan.g, a->q.data, a->k_cache.data, a->v_cache.data, a->out.data, a->lse, kv_view(a->bm),
                    plan.pv, mp, mk, to_score_params(sc), (int)sc.terms, a->workspace, st);
  if (s != FA_OK) return s;
  if ((s = end_decode(plan, st)) != FA_OK) return s;
  if (a->counters == nullptr) return FA_OK;
  return counters_by_desc(plan.g.a, kv_view(a->bm), mp, mk, &plan.pv, plan.g.logical_kv, kPassForward, a->counters, st);
}

}  // extern "C"

// ---- synthetic inputs and paged scatter ---------------------------------------
namespace capi_detail {

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
