/*
 * flexattn_b200.h — C ABI of the B200-native FlexAttention hot path.
 *
 * This is the drop-in boundary for the reference's block-sparse attention
 * library (`blockattn`, /root/reference/proj/include/blockattn/*.hpp). The
 * reference has no FFI of its own: its boundary is the C++ API. Each entry
 * point below replaces one reference function and cites it:
 *
 *   fa_create_block_mask   <- create_block_mask   block_mask.hpp:109-110 (+ transpose :115)
 *   fa_transpose_block_mask<- transpose           block_mask.hpp:115, block_mask.cpp:161-178
 *   fa_convert_block_mask  <- convert_block_mask  paged_kv.hpp:101, paged_kv.cpp:154-228
 *   fa_flex_fwd            <- forward<Real>       engine.hpp:68-71, engine.cpp:46-172
 *   fa_flex_bwd            <- backward<Real>      engine.hpp:78-82, engine.cpp:174-401
 *   fa_flex_decode         <- decode<Real>        engine.hpp:92-96, engine.cpp:403-427
 *                             (+ convert_mods     paged_kv.hpp:117, paged_kv.cpp:230-310
 *                                when a page table is given)
 *   fa_fill_uniform        <- random_tensor<Real> random.hpp:41-46 (SplitMix64 [-1,1))
 *   fa_check_finite        <- validate_inputs     validate.hpp:30-39 (finiteness part)
 *   fa_*_args.counters     <- OpCounters*         engine.hpp:21-32, 68-96
 *
 * Conventions (all entry points):
 *   - Caller-owned DEVICE buffers; plain pointers + sizes, no library types.
 *   - Stream-ordered and asynchronous on the `stream` argument (a cudaStream_t
 *     passed as void*; NULL = legacy default stream). No internal host threads.
 *   - No CPU fallback: a missing/unsupported GPU returns FA_CUDA_ERROR or
 *     FA_UNSUPPORTED, never a silent host computation.
 *   - Errors map 1:1 onto the reference exception classes (errors.hpp:11-101);
 *     fa_last_error() returns the thread-local message of the last failure.
 *   - Tensors are dense row-major (B, H, L, D) as reference Tensor4
 *     (tensor.hpp:20-117). BlockMask indices are int32 (the reference uses
 *     i64; values are identical, widening is exact).
 */
#ifndef FLEXATTN_B200_H_
#define FLEXATTN_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FA_API __attribute__((visibility("default")))
#else
#define FA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception class (errors.hpp) ------- */
typedef int32_t fa_status;
enum {
  FA_OK = 0,
  FA_SHAPE_MISMATCH = 1,          /* ShapeMismatch          errors.hpp:18 */
  FA_NON_FINITE_INPUT = 2,        /* NonFiniteInput         errors.hpp:24 */
  FA_INDEX_OUT_OF_RANGE = 3,      /* IndexOutOfRange        errors.hpp:30 */
  FA_NON_POSITIVE_CAP = 4,        /* NonPositiveCap         errors.hpp:36 */
  FA_GEOMETRY_MISMATCH = 5,       /* GeometryMismatch       errors.hpp:42 */
  FA_BLOCK_MASK_MISMATCH = 6,     /* BlockMaskMismatch      errors.hpp:48 */
  FA_STALE_STATISTICS = 7,        /* StaleStatistics        errors.hpp:55 */
  FA_OFFSET_OUT_OF_RANGE = 8,     /* OffsetOutOfRange       errors.hpp:61 */
  FA_OUT_OF_PAGES = 9,            /* OutOfPages             errors.hpp:67 */
  FA_UNMAPPED_BLOCK = 10,         /* UnmappedBlock          errors.hpp:73 */
  FA_UNMAPPED_PHYSICAL_INDEX = 11,/* UnmappedPhysicalIndex  errors.hpp:80 */
  FA_CUDA_ERROR = 100,            /* CUDA runtime/driver failure            */
  FA_UNSUPPORTED = 101            /* shape/dtype not compiled for sm_100a   */
};

/* ---- element types -------------------------------------------------------- */
enum { FA_F32 = 0, FA_BF16 = 1 };

/* ---- mask_mod descriptor ----------------------------------------------------
 * A mask is the AND of the primitive terms whose bit is set in `terms`
 * (and_mask, mask_library.cpp:94-98). An empty term set is noop_mask
 * (mask_library.cpp:43-45). A non-zero `or_terms` adds a second AND-group
 * evaluated with the same parameters and ORed with the first (or_mask,
 * mask_library.cpp:100-104). Every term sees q + q_offset (offset_mask,
 * mask_library.cpp:106-110); with a `remap` table the terms see
 * (remap[q + q_offset], remap[kv]) (remap_mask, mask_library.cpp:203-215; the
 * table must be a bijection on [0, remap_len), which the host layers check).
 */
enum {
  FA_MASK_CAUSAL = 1u << 0,       /* q >= kv                        mask_library.cpp:13-15 */
  FA_MASK_SLIDING_WINDOW = 1u << 1,/* q >= kv && q - kv <= window   mask_library.cpp:17-22 */
  FA_MASK_DOCUMENT = 1u << 2,     /* ids[q] == ids[kv]              mask_library.cpp:24-34 */
  FA_MASK_PREFIX_LM = 1u << 3,    /* kv < prefix || q >= kv         mask_library.cpp:36-41 */
  FA_MASK_HASH = 1u << 4,         /* test aid hash_mask             tests/test_support.hpp:16-29 */
  FA_MASK_NEVER = 1u << 5,        /* test aid never_mask            tests/test_support.hpp:31-35 */
  FA_MASK_NATTEN = 1u << 6        /* 2-D neighbourhood: max(|dr|,|dc|) <= kernel/2 on a
                                     na_height x na_width canvas      mask_library.cpp:137-149 */
};

typedef struct fa_mask_desc {
  uint32_t terms;          /* OR of FA_MASK_* bits; 0 = noop */
  int32_t hash_density;    /* FA_MASK_HASH: true for density/256 of positions */
  int64_t window;          /* FA_MASK_SLIDING_WINDOW (>= 0) */
  int64_t prefix;          /* FA_MASK_PREFIX_LM (>= 0) */
  int64_t q_offset;        /* offset_mask shift (decode); 0 otherwise */
  uint64_t hash_seed;      /* FA_MASK_HASH */
  const int32_t* doc_ids;  /* FA_MASK_DOCUMENT: device int32[doc_len] */
  int64_t doc_len;
  uint32_t or_terms;       /* second AND-group, ORed with `terms`; 0 = none (ABI v2) */
  int32_t na_kernel;       /* FA_MASK_NATTEN: odd, 1 <= kernel <= min(height, width) */
  int64_t na_height;       /* FA_MASK_NATTEN canvas (tokens = height * width, row-major) */
  int64_t na_width;
  const int32_t* remap;    /* optional device int32[remap_len] slot -> token permutation */
  int64_t remap_len;
  /* optional (ABI v5), with a remap and FA_MASK_NATTEN as the only term: device
   * int32[remap_len], (row << 16) | col of token remap[slot] on the na canvas, which replaces
   * the per-position division of the remapped neighbourhood test (the host layers build it) */
  const int32_t* remap_rc;
} fa_mask_desc;

/* ---- score_mod descriptor ---------------------------------------------------
 * noop_score (mask_library.cpp:47-51) when `terms` == 0; FA_SCORE_ALIBI adds
 * slopes[h]*(q-kv) (mask_library.cpp:53-69); FA_SCORE_SOFT_CAP applies
 * cap*tanh(s/cap) (mask_library.cpp:83-92). Both set = compose(soft_cap, alibi)
 * (modifiers.hpp:57-66): soft_cap(alibi(s)). Every term sees q + q_offset
 * (offset_score, mask_library.cpp:112-119).
 */
enum { FA_SCORE_ALIBI = 1u << 0, FA_SCORE_SOFT_CAP = 1u << 1 };

typedef struct fa_score_desc {
  uint32_t terms;          /* OR of FA_SCORE_* bits; 0 = noop */
  int32_t num_slopes;      /* length of slopes (indexed by q-head) */
  double cap;              /* FA_SCORE_SOFT_CAP: finite, > 0 */
  const float* slopes;     /* FA_SCORE_ALIBI: device float[num_slopes] */
  int64_t q_offset;        /* offset_score shift (decode); 0 otherwise */
} fa_score_desc;

/* ---- BlockMask (device) -----------------------------------------------------
 * Layout of reference BlockMask (block_mask.hpp:35-79) with the FlexAttention
 * names: kv_num_blocks == partial_num, kv_indices == partial_idx,
 * full_kv_* == full_*; q-side arrays == the same fields of transpose(bm).
 * Counts (b_dims, h_dims, rows); indices (b_dims, h_dims, rows, cols);
 * q-side counts (b_dims, h_dims, cols); q-side indices (b_dims, h_dims, cols, rows).
 * Lists are ascending and compacted; slots past the count are 0
 * (block_mask.cpp:50-52). The merged visit order of the reference is the
 * ascending merge of the two lists (block_mask.hpp:26-31).
 */
typedef struct fa_block_mask {
  int64_t b_dims, h_dims, rows, cols, bs_q, bs_kv, q_len, kv_len;
  int32_t* kv_num_blocks;
  int32_t* kv_indices;
  int32_t* full_kv_num_blocks;
  int32_t* full_kv_indices;
  int32_t* q_num_blocks;       /* may be NULL when only the kv side is needed */
  int32_t* q_indices;
  int32_t* full_q_num_blocks;
  int32_t* full_q_indices;
} fa_block_mask;

/* ---- dense (B, H, L, D) tensor view -------------------------------------- */
typedef struct fa_tensor {
  void* data;
  int32_t dtype;           /* FA_F32 | FA_BF16 */
  int32_t _pad;
  int64_t b, h, l, d;
} fa_tensor;

/* ---- paged KV page table (device), reference PageTable paged_kv.hpp:18-41 --- */
typedef struct fa_page_table {
  int64_t batches, max_logical_pages, num_physical_pages, page_size;
  const int32_t* table;            /* (batches, max_logical_pages), -1 = unmapped */
  const int32_t* phys_to_logical;  /* (num_physical_pages), -1 = free */
  const int32_t* owner;            /* (num_physical_pages), -1 = free */
  const int32_t* seq_len;          /* (batches) tokens stored per sequence */
  int64_t max_seq_len;             /* host copy of max(seq_len) (ABI v3); 0 = unknown, then
                                      max_logical_pages * page_size bounds the mask's kv range */
} fa_page_table;

/* ---- misc ------------------------------------------------------------------ */
FA_API const char* fa_last_error(void);
FA_API const char* fa_status_name(fa_status s);
FA_API int32_t fa_abi_version(void);
/* Number of kernel launches issued by this library since load (per process). */
FA_API uint64_t fa_launch_count(void);

/* ---- BlockMask ---------------------------------------------------------------
 * Sizes the caller must allocate: rows/cols, element counts of each count and
 * index array, and the scratch bytes create/transpose need.
 */
FA_API fa_status fa_block_mask_geometry(int64_t b_dims, int64_t h_dims, int64_t q_len, int64_t kv_len,
                                 int64_t bs_q, int64_t bs_kv, int64_t* rows, int64_t* cols,
                                 size_t* workspace_bytes);

/* create_block_mask + transpose in one pass. `bm` holds the caller-allocated
 * arrays; geometry fields are written. q-side arrays are filled when non-NULL. */
FA_API fa_status fa_create_block_mask(const fa_mask_desc* mask, int64_t b_dims, int64_t h_dims,
                               int64_t q_len, int64_t kv_len, int64_t bs_q, int64_t bs_kv,
                               fa_block_mask* bm, void* workspace, size_t workspace_bytes,
                               void* stream);

/* q-side arrays of `bm` from its kv-side arrays (transpose, block_mask.cpp:161-178). */
FA_API fa_status fa_transpose_block_mask(fa_block_mask* bm, void* workspace, size_t workspace_bytes,
                                  void* stream);

/* Rewrites every logical kv block index through the page table
 * (convert_block_mask, paged_kv.cpp:154-228): out has b_dims = pt->batches,
 * cols = num_physical_pages, kv_len = pages * page_size. `out` arrays are
 * caller-allocated; q-side arrays of `out` are ignored. Unmapped blocks are
 * reported with FA_UNMAPPED_BLOCK after the stream is synchronised by the call. */
FA_API fa_status fa_convert_block_mask(const fa_block_mask* logical, const fa_page_table* pt,
                                fa_block_mask* out, void* stream);
/* The same without a host round trip (ABI v6): the device int32 *status is zeroed and then set
 * to 1 when a referenced logical block has no physical page (the caller checks it when it
 * synchronises anyway), so a serving step can be captured in a CUDA graph. */
FA_API fa_status fa_convert_block_mask_async(const fa_block_mask* logical, const fa_page_table* pt,
                                             fa_block_mask* out, int32_t* status, void* stream);

/* ---- attention ---------------------------------------------------------------- */
/* Work counters of the reference (OpCounters, engine.hpp:21-32), computed on the device from the
 * BlockMask and the mask (not by instrumenting the kernels):
 *   mask_evals  = positions of the visited partial tiles inside [0,Q_LEN) x [0,KV_LEN), per (b, h)
 *                 walk (backward: both passes, rows with lse = -inf skipped, engine.cpp:257-260);
 *   score_evals = live (mask-true) positions, one score_mod application each (backward: x2);
 *   madds       = forward: 2*D per live position (q.k dot + p.v); backward: D per q row (Δ)
 *                 + 7*D per live position (dq pass 3*D, dk/dv pass 4*D).
 * The reference's forward madds additionally count D per running-max increase (accumulator
 * rescales, engine.cpp:128-133); that term depends on the data and on the visit order and is
 * not included. */
typedef struct fa_op_counters {
  uint64_t madds;
  uint64_t mask_evals;
  uint64_t score_evals;
} fa_op_counters;

/* Per-call flags (ABI v3). */
enum {
  /* Data-dependent validation of the reference, at the cost of one extra read of the inputs
   * and a stream synchronisation at the end of the call: NaN/inf in q/k/v
   * (validate_inputs, validate.hpp:36-38) and d_out (engine.cpp:196) -> FA_NON_FINITE_INPUT;
   * a paged decode that visits a page not owned by the row's batch element
   * (convert_mods, paged_kv.cpp:259-272) -> FA_UNMAPPED_PHYSICAL_INDEX. */
  FA_FLAG_VALIDATE = 1u << 0,
  /* Backward only: the split backward — a dK/dV kernel plus a separate dQ pass that
   * accumulates each q tile's dQ in TMEM over its kv blocks in one fixed order (the reference's
   * separate dq pass, engine.cpp:237-305) — so dq/dk/dv are bitwise reproducible run to run (the
   * reference's worker-count independence, README.md:104-106). Without it dk/dv are still
   * reproducible but the fused kernel adds fp32 dQ partial sums in arrival order. */
  FA_FLAG_DETERMINISTIC = 1u << 1
};

typedef struct fa_fwd_args {
  fa_tensor q, k, v;       /* q (B,Hq,Q,D); k,v (B or 1, Hkv, KV, D) */
  fa_tensor out;           /* (B,Hq,Q,D), dtype of q */
  float* lse;              /* (B,Hq,Q) natural-log logsumexp; -inf on empty rows */
  const fa_block_mask* bm; /* kv side required */
  fa_mask_desc mask;
  fa_score_desc score;
  double scale;            /* <= 0 selects 1/sqrt(D) (config.hpp:28-31) */
  int64_t gqa_group;       /* Hq == gqa_group * Hkv */
  uint32_t flags;          /* FA_FLAG_VALIDATE (ABI v3) */
  int32_t _pad1;
  fa_op_counters* counters;/* host out-param or NULL; non-NULL synchronises the stream */
} fa_fwd_args;

typedef struct fa_bwd_args {
  fa_tensor q, k, v, out, d_out;
  const float* lse;        /* from fa_flex_fwd on the same tensors */
  fa_tensor dq, dk, dv;    /* dq like q; dk/dv like k */
  const fa_block_mask* bm; /* kv side and q side both required */
  fa_mask_desc mask;
  fa_score_desc score;
  double scale;
  int64_t gqa_group;
  void* workspace;         /* fa_bwd_workspace_size bytes */
  size_t workspace_bytes;
  uint32_t flags;          /* FA_FLAG_VALIDATE | FA_FLAG_DETERMINISTIC (ABI v3) */
  int32_t _pad1;
  fa_op_counters* counters;/* host out-param or NULL; non-NULL synchronises the stream */
  /* optional cudaEvent_t (as void*) recorded on the stream before the preprocess kernel, before
   * the main kernel, before the dQ conversion and after it (per-kernel timing); NULL = none */
  void* phase_events[4];
} fa_bwd_args;

typedef struct fa_decode_args {
  fa_tensor q;             /* (B,Hq,n_new,D): rows [offset, offset+n_new) */
  fa_tensor k_cache, v_cache; /* logical (B|1,Hkv,L,D) or physical (1,Hkv,pages*ps,D) */
  fa_tensor out;
  float* lse;
  const fa_block_mask* bm; /* bm for the shifted mask at q_len == n_new (physical if pt) */
  const fa_page_table* pt; /* NULL: unpaged; else logical positions recovered per page */
  int64_t offset;
  fa_mask_desc mask;       /* written in absolute positions (offset applied here) */
  fa_score_desc score;
  double scale;
  int64_t gqa_group;
  int32_t num_splits;      /* split-KV factor; <= 0 picks one */
  int32_t _pad;
  void* workspace;         /* fa_decode_workspace_size bytes */
  size_t workspace_bytes;
  uint32_t flags;          /* FA_FLAG_VALIDATE (ABI v3) */
  int32_t _pad2;
  fa_op_counters* counters;/* host out-param or NULL; non-NULL synchronises the stream */
} fa_decode_args;

FA_API fa_status fa_flex_fwd(const fa_fwd_args* args, void* stream);
FA_API size_t fa_bwd_workspace_size(int64_t batch, int64_t heads, int64_t q_len, int64_t dim);
FA_API fa_status fa_flex_bwd(const fa_bwd_args* args, void* stream);
FA_API size_t fa_decode_workspace_size(int64_t batch, int64_t heads, int64_t n_new, int64_t dim,
                                int32_t num_splits);
FA_API fa_status fa_flex_decode(const fa_decode_args* args, void* stream);

/* NaN/inf scan of up to 8 tensors in one pass (validate_inputs' finiteness checks,
 * validate.hpp:36-38, tensor.hpp:38-42). Synchronises the stream; FA_NON_FINITE_INPUT names the
 * first offending tensor (names[i], or its index). */
FA_API fa_status fa_check_finite(const fa_tensor* tensors, const char* const* names, int32_t n,
                                 void* stream);

/* ---- synthetic inputs ------------------------------------------------------------
 * Element i of random_tensor(seed, ...) (random.hpp:41-46):
 * (float)(SplitMix64(seed) i-th draw in [-1,1)), rounded to bf16 (RNE) when dtype is bf16.
 * Elements [first, first + n) are written to dst[0..n). */
FA_API fa_status fa_fill_uniform(void* dst, int32_t dtype, uint64_t seed, int64_t first, int64_t n,
                          void* stream);

/* Scatter logical tokens (B, Hkv, L, D) into a physical paged buffer
 * (1, Hkv, pages*ps, D) through `pt` (PagedKVCache::write_tokens, paged_kv.cpp:54-70). */
FA_API fa_status fa_paged_write(const fa_tensor* logical, const fa_page_table* pt, fa_tensor* physical,
                         void* stream);

/* ---- device page pool (ABI v4) ------------------------------------------------------
 * The PagedKVCache allocator (paged_kv.hpp:50-89, paged_kv.cpp:13-152) with ALL of its state
 * in device memory, so a serving step (append -> convert -> decode) runs without a host round
 * trip and can be captured in a CUDA graph. Same semantics as the reference, bit for bit:
 * LIFO free stack with page 0 on top (paged_kv.cpp:27-31), deterministic_shuffle
 * (random.hpp:49-56), assign = capacity check, erase, pop `needed` pages (:72-98), append_tokens
 * pops the extra pages (:100-126), erase pushes the owned pages in logical order (:128-141);
 * max_logical_pages == num_pages (:20).
 *
 * A batched update applies its requests IN ORDER, exactly as the same sequence of reference
 * calls; the first failing request (batch outside [0, batches) -> IndexOutOfRange, not enough
 * pages -> OutOfPages, a batch id repeated in one call -> ShapeMismatch) stops the batch:
 * requests before it are applied, it and the ones after are not (the reference's exception
 * leaves earlier calls applied and the failing one without effect). */
typedef struct fa_page_pool {
  int64_t batches, num_pages, page_size;
  /* device arrays, laid out by fa_page_pool_init in one caller-owned allocation */
  int32_t* table;            /* (batches, num_pages), -1 = unmapped */
  int32_t* phys_to_logical;  /* (num_pages), -1 = free */
  int32_t* owner;            /* (num_pages), -1 = free */
  int32_t* seq_len;          /* (batches) */
  int32_t* free_stack;       /* (num_pages): free pages, top = free_stack[*free_count - 1] */
  int32_t* free_count;       /* device scalar */
  int32_t* status;           /* device int32[8]: fa_status, failing request (= applied count),
                                needed, available, tokens, op, batch id of the failure */
  int32_t* scratch;          /* per-request bookkeeping of the last update */
} fa_page_pool;

enum { FA_PAGE_ASSIGN = 0, FA_PAGE_APPEND = 1, FA_PAGE_ERASE = 2 };
/* Update flag: do not synchronise; the outcome stays in pool->status (fa_page_pool_status). */
enum { FA_FLAG_NO_SYNC = 1u << 2 };

/* Device bytes fa_page_pool_init needs for (batches, num_pages). */
FA_API size_t fa_page_pool_bytes(int64_t batches, int64_t num_pages);
/* Lays the pool out in `device_mem` and resets it (every page free, page 0 on top, all
 * sequences empty), stream-ordered. */
FA_API fa_status fa_page_pool_init(fa_page_pool* pool, void* device_mem, size_t bytes, int64_t batches,
                                   int64_t num_pages, int64_t page_size, void* stream);
/* shuffle_free_pages(seed) (paged_kv.cpp:143-146) on the device free stack. */
FA_API fa_status fa_page_pool_shuffle(const fa_page_pool* pool, uint64_t seed, void* stream);
/* n requests (device int32 batch_ids[n], n_tokens[n]; n_tokens ignored for FA_PAGE_ERASE) of
 * one kind. With k_tokens/v_tokens given (packed (1, Hkv, sum(n_tokens), D), request i's tokens
 * at offset sum_{j<i} n_tokens[j]) the applied requests' tokens are written into
 * k_cache/v_cache (1, Hkv, num_pages * page_size, D) at their logical positions
 * (write_tokens, paged_kv.cpp:54-70): assign from 0, append from the old length. Unless
 * FA_FLAG_NO_SYNC, the call synchronises the stream and returns the first failure. */
FA_API fa_status fa_page_pool_update(const fa_page_pool* pool, int32_t op, const int32_t* batch_ids,
                                     const int32_t* n_tokens, int32_t n, const fa_tensor* k_tokens,
                                     const fa_tensor* v_tokens, fa_tensor* k_cache, fa_tensor* v_cache,
                                     uint32_t flags, void* stream);
/* Reads pool->status (synchronises): the outcome of the last update, as its fa_status with the
 * reference's message in fa_last_error(); *applied = number of requests applied. */
FA_API fa_status fa_page_pool_status(const fa_page_pool* pool, int32_t* applied, void* stream);
/* The pool as a page table for fa_convert_block_mask / fa_flex_decode (max_seq_len = 0). */
FA_API fa_page_table fa_page_pool_table(const fa_page_pool* pool);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* FLEXATTN_B200_H_ */
