/*
 * flex_oracle.h — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference
 * block-sparse attention path (/root/reference/proj) used as the parity checker
 * for the sm_100a kernels. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product path never does.
 *
 * Parity pinned: tests/test_oracle_pin.py checks this restatement against the
 * reference itself (oracle/_ref, built from /root/reference sources by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 *
 * Every function cites the reference file:line it restates.
 */
#ifndef FLEX_ORACLE_H_
#define FLEX_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* mask terms: identical bit values to fa_mask_desc (include/flexattn_b200.h) */
typedef struct fo_mask {
  uint32_t terms;
  int32_t hash_density;
  int64_t window;
  int64_t prefix;
  int64_t q_offset;
  uint64_t hash_seed;
  const int64_t* doc_ids;   /* host */
  int64_t doc_len;
  int64_t bound_q;          /* > 0: runtime mask adds q < bound_q (bound_mask, block_mask.cpp:14-19) */
  int64_t bound_kv;         /* > 0: ... && kv < bound_kv */
  uint32_t or_terms;        /* second AND-group, ORed (or_mask) */
  int32_t na_kernel;        /* term 64: na_naive on a na_height x na_width canvas */
  int64_t na_height;
  int64_t na_width;
  const int64_t* remap;     /* host; remap_mask slot -> token, or NULL */
  int64_t remap_len;
} fo_mask;

typedef struct fo_score {
  uint32_t terms;           /* 1 = alibi, 2 = soft_cap, 3 = soft_cap(alibi(s)) */
  int32_t num_slopes;
  double cap;
  const double* slopes;     /* host, indexed by q-head */
  int64_t q_offset;
} fo_score;

/* Status: 0 ok, else the fa_status code of the reference exception. */
int fo_mask_eval(const fo_mask* m, int64_t b, int64_t h, int64_t q, int64_t kv, int* out);
int fo_score_apply(const fo_score* s, double x, int64_t b, int64_t h, int64_t q, int64_t kv,
                   double* out);
int fo_score_dapply(const fo_score* s, double x, int64_t b, int64_t h, int64_t q, int64_t kv,
                    double* out);
void fo_alibi_slopes(int64_t heads, double* out);

/* create_block_mask (block_mask.cpp:79-115). Arrays caller-allocated, int64,
 * counts (b,h,rows), indices (b,h,rows,cols). Bounds are applied from q_len/kv_len. */
int fo_create_block_mask(const fo_mask* m, int64_t b_dims, int64_t h_dims, int64_t q_len,
                         int64_t kv_len, int64_t bs_q, int64_t bs_kv, int64_t* partial_num,
                         int64_t* partial_idx, int64_t* full_num, int64_t* full_idx);

/* transpose (block_mask.cpp:161-178): kv-side lists (rows x cols) -> q-side (cols x rows). */
void fo_transpose(int64_t b_dims, int64_t h_dims, int64_t rows, int64_t cols,
                  const int64_t* partial_num, const int64_t* partial_idx, const int64_t* full_num,
                  const int64_t* full_idx, int64_t* t_partial_num, int64_t* t_partial_idx,
                  int64_t* t_full_num, int64_t* t_full_idx);

/* Block mask geometry as consumed by the engine. */
typedef struct fo_bm {
  int64_t b_dims, h_dims, rows, cols, bs_q, bs_kv;
  const int64_t* partial_num;
  const int64_t* partial_idx;
  const int64_t* full_num;
  const int64_t* full_idx;
} fo_bm;

/* forward_impl (engine.cpp:46-163), Real = float / double. `mask` is the runtime
 * mask evaluated in partial blocks (bounds included via bound_q/bound_kv).
 * Visit order = ascending merge of partial and full lists (block_mask.cpp:57-69). */
int fo_forward_f32(const float* q, const float* k, const float* v, int64_t B, int64_t Hq,
                   int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D, double scale,
                   int64_t gqa_group, const fo_score* s, const fo_mask* mask, const fo_bm* bm,
                   float* out, float* lse);
int fo_forward_f64(const double* q, const double* k, const double* v, int64_t B, int64_t Hq,
                   int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D, double scale,
                   int64_t gqa_group, const fo_score* s, const fo_mask* mask, const fo_bm* bm,
                   double* out, double* lse);

/* backward (engine.cpp:174-401), double accumulators; bm_t = transpose(bm). */
int fo_backward_f32(const float* q, const float* k, const float* v, const float* out,
                    const float* lse, const float* dout, int64_t B, int64_t Hq, int64_t Hkv,
                    int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D, double scale,
                    int64_t gqa_group, const fo_score* s, const fo_mask* mask, const fo_bm* bm,
                    const fo_bm* bm_t, float* dq, float* dk, float* dv);
int fo_backward_f64(const double* q, const double* k, const double* v, const double* out,
                    const double* lse, const double* dout, int64_t B, int64_t Hq, int64_t Hkv,
                    int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D, double scale,
                    int64_t gqa_group, const fo_score* s, const fo_mask* mask, const fo_bm* bm,
                    const fo_bm* bm_t, double* dq, double* dk, double* dv);

/* dense_forward (oracle.cpp:13-76): materialised scores, no block mask. */
int fo_dense_forward_f64(const double* q, const double* k, const double* v, int64_t B,
                         int64_t Hq, int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D,
                         double scale, int64_t gqa_group, const fo_score* s, const fo_mask* mask,
                         double* out, double* lse);

/* convert_block_mask (paged_kv.cpp:154-228) on the kv side. table (batches, max_logical_pages)
 * int32 with -1 sentinel. Output b_dims = batches, cols = num_physical_pages. Returns
 * FA_UNMAPPED_BLOCK (10) if a referenced logical block is unmapped. */
int fo_convert_block_mask(int64_t b_dims, int64_t h_dims, int64_t rows, int64_t cols,
                          const int64_t* partial_num, const int64_t* partial_idx,
                          const int64_t* full_num, const int64_t* full_idx, int64_t batches,
                          int64_t max_logical_pages, int64_t num_physical_pages,
                          const int32_t* table, int64_t* o_partial_num, int64_t* o_partial_idx,
                          int64_t* o_full_num, int64_t* o_full_idx);

/* random_tensor<float> (random.hpp:41-46): element i in [first, first+n). */
void fo_random_f32(uint64_t seed, int64_t first, int64_t n, float* out);
/* SplitMix64 next_u64 sequence (random.hpp:21-26), used by make_doc_ids / shuffles. */
uint64_t fo_splitmix_next(uint64_t* state);

#ifdef __cplusplus
}
#endif

#endif /* FLEX_ORACLE_H_ */
