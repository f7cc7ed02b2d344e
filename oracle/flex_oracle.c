/*
 * flex_oracle.c — TEST INFRASTRUCTURE ONLY (see flex_oracle.h). A line-by-line
 * restatement, in C, of the reference algorithms the sm_100a kernels replace.
 * It is the checker; nothing in the product path links it.
 *
 * Compiled with -O3 -std=c11 and no -ffast-math / -mfma so the float path
 * performs the same IEEE operations in the same order as the reference
 * (compiled -O3 -DNDEBUG, CMakeLists.txt:23), which lets tests pin it
 * bit-for-bit against oracle/_ref.
 */
#include "flex_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, E_SHAPE = 1, E_INDEX = 3, E_CAP = 4, E_BM = 6, E_UNMAPPED_BLOCK = 10 };

/* ---- SplitMix64 (random.hpp:15-38) --------------------------------------- */
uint64_t fo_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* random_tensor (random.hpp:41-46): v = (Real)(next_unit()*2-1); draw i uses
 * state seed + (i+1)*golden, so element i is computable independently. */
void fo_random_f32(uint64_t seed, int64_t first, int64_t n, float* out) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t st = seed + (uint64_t)(first + i) * 0x9e3779b97f4a7c15ull;
    const uint64_t u = fo_splitmix_next(&st);
    const double unit = (double)(u >> 11) * 0x1.0p-53;
    out[i] = (float)(unit * 2.0 - 1.0);
  }
}

/* ---- mask_mod (mask_library.cpp, tests/test_support.hpp) ----------------- */
/* AND of the primitive terms in t at positions (q, kv) (and_mask, mask_library.cpp:94-98) */
static int mask_group(const fo_mask* m, uint32_t t, int64_t b, int64_t h, int64_t qq, int64_t kv,
                      int* out) {
  if (t & (1u << 5)) { *out = 0; return OK; } /* never_mask, test_support.hpp:31-35 */
  if ((t & 1u) && !(qq >= kv)) { *out = 0; return OK; }                       /* causal :13-15 */
  if ((t & 2u) && !(qq >= kv && qq - kv <= m->window)) { *out = 0; return OK; } /* sliding :17-22 */
  if (t & 64u) {                                                              /* na_naive :137-149 */
    const int64_t w = m->na_width, n = m->na_height * m->na_width, rad = m->na_kernel / 2;
    if (qq < 0 || qq >= n || kv < 0 || kv >= n) return E_INDEX;
    const int64_t dr = qq / w - kv / w, dc = qq % w - kv % w;
    const int64_t adr = dr < 0 ? -dr : dr, adc = dc < 0 ? -dc : dc;
    if (!((adr > adc ? adr : adc) <= rad)) { *out = 0; return OK; }
  }
  if (t & 4u) {                                                                 /* document :24-34 */
    const int64_t n = m->doc_len;
    if (qq < 0 || qq >= n || kv < 0 || kv >= n) return E_INDEX;
    if (m->doc_ids[qq] != m->doc_ids[kv]) { *out = 0; return OK; }
  }
  if ((t & 8u) && !(kv < m->prefix || qq >= kv)) { *out = 0; return OK; }      /* prefix_lm :36-41 */
  if (t & 16u) {                                            /* hash_mask test_support.hpp:16-29 */
    uint64_t x = m->hash_seed;
    x ^= 0x9e3779b97f4a7c15ull * (uint64_t)(b + 1);
    x ^= 0xc2b2ae3d27d4eb4full * (uint64_t)(h + 1);
    x ^= 0x165667b19e3779f9ull * (uint64_t)(qq + 1);
    x ^= 0x27d4eb2f165667c5ull * (uint64_t)(kv + 1);
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    x ^= x >> 31;
    if (!((int)(x & 0xff) < m->hash_density)) { *out = 0; return OK; }
  }
  *out = 1;
  return OK;
}

int fo_mask_eval(const fo_mask* m, int64_t b, int64_t h, int64_t q, int64_t kv, int* out) {
  /* bound_mask (block_mask.cpp:14-19) is applied on the UNshifted q, then the
   * user mask sees q + offset (decode runtime mask, engine.cpp:421-424). */
  if (m->bound_q > 0 && !(q < m->bound_q)) { *out = 0; return OK; }
  if (m->bound_kv > 0 && !(kv < m->bound_kv)) { *out = 0; return OK; }
  int64_t qq = q + m->q_offset; /* offset_mask (mask_library.cpp:106-110) */
  if (m->remap_len > 0) {      /* remap_mask (mask_library.cpp:203-215) */
    if (qq < 0 || qq >= m->remap_len || kv < 0 || kv >= m->remap_len) return E_INDEX;
    qq = m->remap[qq];
    kv = m->remap[kv];
  }
  int st = mask_group(m, m->terms, b, h, qq, kv, out);
  if (st != OK) return st;
  if (!*out && m->or_terms != 0) st = mask_group(m, m->or_terms, b, h, qq, kv, out); /* or_mask :100-104 */
  return st;
}

/* ---- score_mod (mask_library.cpp:47-92, modifiers.hpp:57-66) ------------ */
static int slope_at(const fo_score* s, int64_t h, double* out) {
  if (h < 0 || h >= s->num_slopes) return E_INDEX; /* alibi slope_at :56-60 */
  *out = s->slopes[h];
  return OK;
}

int fo_score_apply(const fo_score* s, double x, int64_t b, int64_t h, int64_t q, int64_t kv,
                   double* out) {
  (void)b;
  const int64_t qq = q + s->q_offset; /* offset_score :112-119 */
  if (s->terms & 1u) {                /* alibi :61-63 */
    double sl;
    int st = slope_at(s, h, &sl);
    if (st) return st;
    x = x + sl * (double)(qq - kv);
  }
  if (s->terms & 2u) { /* soft_cap :88 */
    if (!(s->cap > 0.0) || !isfinite(s->cap)) return E_CAP;
    x = s->cap * tanh(x / s->cap);
  }
  *out = x;
  return OK;
}

int fo_score_dapply(const fo_score* s, double x, int64_t b, int64_t h, int64_t q, int64_t kv,
                    double* out) {
  (void)b;
  const int64_t qq = q + s->q_offset;
  double d = 1.0;
  double inner = x;
  if (s->terms & 1u) { /* alibi dapply :64-67 (domain check, derivative 1) */
    double sl;
    int st = slope_at(s, h, &sl);
    if (st) return st;
    inner = x + sl * (double)(qq - kv);
  }
  if (s->terms & 2u) { /* soft_cap dapply :89-91, chained via compose :61-65 */
    const double t = tanh(inner / s->cap);
    d = (1.0 - t * t) * d;
  }
  *out = d;
  return OK;
}

void fo_alibi_slopes(int64_t heads, double* out) { /* alibi_slopes :71-81 */
  for (int64_t h = 0; h < heads; ++h) out[h] = -exp2(-8.0 * (double)(h + 1) / (double)heads);
}

/* ---- create_block_mask (block_mask.cpp:79-115) --------------------------- */
int fo_create_block_mask(const fo_mask* m_in, int64_t b_dims, int64_t h_dims, int64_t q_len,
                         int64_t kv_len, int64_t bs_q, int64_t bs_kv, int64_t* partial_num,
                         int64_t* partial_idx, int64_t* full_num, int64_t* full_idx) {
  if (b_dims < 1 || h_dims < 1) return E_SHAPE;                               /* :30-32 */
  if (q_len < 1 || kv_len < 1 || bs_q < 1 || bs_kv < 1) return E_SHAPE;       /* :33-35 */
  const int64_t rows = (q_len + bs_q - 1) / bs_q, cols = (kv_len + bs_kv - 1) / bs_kv;
  const int64_t nrows = b_dims * h_dims * rows;
  memset(partial_num, 0, sizeof(int64_t) * (size_t)nrows); /* make_empty zero fill :45-52 */
  memset(full_num, 0, sizeof(int64_t) * (size_t)nrows);
  memset(partial_idx, 0, sizeof(int64_t) * (size_t)(nrows * cols));
  memset(full_idx, 0, sizeof(int64_t) * (size_t)(nrows * cols));
  fo_mask m = *m_in;
  m.bound_q = 0; /* the builder evaluates the user mask over in-range positions only */
  m.bound_kv = 0;
  for (int64_t b = 0; b < b_dims; ++b)
    for (int64_t h = 0; h < h_dims; ++h)
      for (int64_t r = 0; r < rows; ++r) {
        const int64_t q0 = r * bs_q;
        const int64_t q1 = q0 + bs_q < q_len ? q0 + bs_q : q_len;
        const int64_t row = (b * h_dims + h) * rows + r;
        for (int64_t c = 0; c < cols; ++c) {
          const int64_t k0 = c * bs_kv;
          const int64_t k1 = k0 + bs_kv < kv_len ? k0 + bs_kv : kv_len;
          const int ragged = (q1 - q0 != bs_q) || (k1 - k0 != bs_kv); /* :91-94 */
          int any = 0, all = 1;
          for (int64_t q = q0; q < q1 && !(any && !all); ++q) {      /* early exit :96-105 */
            for (int64_t kv = k0; kv < k1; ++kv) {
              int v;
              const int st = fo_mask_eval(&m, b, h, q, kv, &v);
              if (st) return st;
              if (v) {
                any = 1;
              } else {
                all = 0;
                if (any) break;
              }
            }
          }
          if (!any) continue;                                        /* kEmpty */
          if (all && !ragged) full_idx[row * cols + full_num[row]++] = c; /* push_block :62-64 */
          else partial_idx[row * cols + partial_num[row]++] = c;        /* :65-66 */
        }
      }
  return OK;
}

/* ---- transpose (block_mask.cpp:161-178, via to_dense :117-138) --------- */
void fo_transpose(int64_t b_dims, int64_t h_dims, int64_t rows, int64_t cols,
                  const int64_t* partial_num, const int64_t* partial_idx, const int64_t* full_num,
                  const int64_t* full_idx, int64_t* t_partial_num, int64_t* t_partial_idx,
                  int64_t* t_full_num, int64_t* t_full_idx) {
  unsigned char* g = (unsigned char*)calloc((size_t)(rows * cols), 1);
  for (int64_t b = 0; b < b_dims; ++b)
    for (int64_t h = 0; h < h_dims; ++h) {
      memset(g, 0, (size_t)(rows * cols));
      for (int64_t r = 0; r < rows; ++r) {
        const int64_t row = (b * h_dims + h) * rows + r;
        for (int64_t i = 0; i < partial_num[row]; ++i) g[r * cols + partial_idx[row * cols + i]] = 1;
        for (int64_t i = 0; i < full_num[row]; ++i) g[r * cols + full_idx[row * cols + i]] = 2;
      }
      for (int64_t c = 0; c < cols; ++c) {
        const int64_t trow = (b * h_dims + h) * cols + c;
        t_partial_num[trow] = 0;
        t_full_num[trow] = 0;
        for (int64_t r = 0; r < rows; ++r) {
          t_partial_idx[trow * rows + r] = 0;
          t_full_idx[trow * rows + r] = 0;
        }
        for (int64_t r = 0; r < rows; ++r) {
          const unsigned char k = g[r * cols + c];
          if (k == 2) t_full_idx[trow * rows + t_full_num[trow]++] = r;
          else if (k == 1) t_partial_idx[trow * rows + t_partial_num[trow]++] = r;
        }
      }
    }
  free(g);
}

/* Merged visit entry n of a row: ascending merge of the two lists, which is the
 * order push_block recorded at build time (block_mask.cpp:57-69, load :251-268). */
typedef struct { int64_t c; int full; } visit_t;
static int64_t merged_visits(const fo_bm* bm, int64_t mb, int64_t mh, int64_t r, visit_t* out) {
  const int64_t row = (mb * bm->h_dims + mh) * bm->rows + r;
  const int64_t np = bm->partial_num[row], nf = bm->full_num[row];
  const int64_t* pi = bm->partial_idx + row * bm->cols;
  const int64_t* fi = bm->full_idx + row * bm->cols;
  int64_t p = 0, f = 0, n = 0;
  while (p < np || f < nf) {
    const int take_full = p >= np || (f < nf && fi[f] < pi[p]);
    if (take_full) { out[n].c = fi[f++]; out[n].full = 1; }
    else { out[n].c = pi[p++]; out[n].full = 0; }
    ++n;
  }
  return n;
}

/* ---- forward_impl (engine.cpp:46-163) ------------------------------------ */
#define FO_FORWARD(NAME, Real, EXP, LOG)                                                        \
  int NAME(const Real* q, const Real* k, const Real* v, int64_t B, int64_t Hq, int64_t Hkv,    \
           int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D, double scale, int64_t gqa_group,   \
           const fo_score* s, const fo_mask* mask, const fo_bm* bm, Real* out, Real* lse) {    \
    if (Hq != gqa_group * Hkv) return E_SHAPE;                                                 \
    if (Bkv != 1 && Bkv != B) return E_SHAPE;                                                  \
    if (bm->b_dims != 1 && bm->b_dims != B) return E_BM;                                        \
    if (bm->h_dims != 1 && bm->h_dims != Hq) return E_BM;                                       \
    const Real scale_r = (Real)scale;                                                          \
    const Real NEG = -(Real)INFINITY;                                                          \
    const int64_t bs_q = bm->bs_q, bs_kv = bm->bs_kv;                                          \
    Real* sbuf = (Real*)malloc(sizeof(Real) * (size_t)bs_kv);                                  \
    Real* acc = (Real*)malloc(sizeof(Real) * (size_t)D);                                       \
    visit_t* vis = (visit_t*)malloc(sizeof(visit_t) * (size_t)bm->cols);                       \
    int st = OK;                                                                               \
    for (int64_t i = 0; i < B * Hq * Lq; ++i) lse[i] = NEG;                                    \
    for (int64_t task = 0; task < B * Hq * bm->rows && st == OK; ++task) {                    \
      const int64_t r = task % bm->rows; /* :75-82 */                                          \
      const int64_t h = (task / bm->rows) % Hq;                                                \
      const int64_t b = task / (bm->rows * Hq);                                                \
      const int64_t mb = bm->b_dims == 1 ? 0 : b, mh = bm->h_dims == 1 ? 0 : h;                \
      const int64_t kb = Bkv == 1 ? 0 : b, kh = h / gqa_group;                                 \
      const int64_t nvisit = merged_visits(bm, mb, mh, r, vis);                                \
      const int64_t q_end = (r + 1) * bs_q < Lq ? (r + 1) * bs_q : Lq;                         \
      for (int64_t iq = r * bs_q; iq < q_end && st == OK; ++iq) {                              \
        const Real* qrow = q + ((b * Hq + h) * Lq + iq) * D;                                   \
        Real run_max = NEG, run_sum = (Real)0;                                                 \
        for (int64_t d = 0; d < D; ++d) acc[d] = (Real)0;                                      \
        for (int64_t vi = 0; vi < nvisit && st == OK; ++vi) { /* :91-95 */                     \
          const int64_t c = vis[vi].c;                                                         \
          const int full = vis[vi].full;                                                       \
          const int64_t j0 = c * bs_kv;                                                        \
          const int64_t j1 = j0 + bs_kv < Lkv ? j0 + bs_kv : Lkv;                              \
          Real block_max = NEG;                                                                \
          for (int64_t j = j0; j < j1; ++j) { /* :98-119 */                                    \
            if (!full) {                                                                       \
              int mv;                                                                          \
              st = fo_mask_eval(mask, b, h, iq, j, &mv);                                       \
              if (st) break;                                                                   \
              if (!mv) { sbuf[j - j0] = NEG; continue; }                                       \
            }                                                                                  \
            const Real* krow = k + ((kb * Hkv + kh) * Lkv + j) * D;                            \
            Real dot = (Real)0;                                                                \
            for (int64_t d = 0; d < D; ++d) dot += qrow[d] * krow[d];                          \
            const Real s_scaled = dot * scale_r;                                               \
            double sm;                                                                         \
            st = fo_score_apply(s, (double)s_scaled, b, h, iq, j, &sm);                        \
            if (st) break;                                                                     \
            const Real sv = (Real)sm;                                                          \
            sbuf[j - j0] = sv;                                                                 \
            if (sv > block_max) block_max = sv;                                                \
          }                                                                                    \
          if (st) break;                                                                       \
          const Real new_max = run_max > block_max ? run_max : block_max; /* :121-134 */       \
          if (new_max == NEG) continue;                                                        \
          if (new_max > run_max) {                                                             \
            if (run_max != NEG) {                                                              \
              const Real alpha = EXP(run_max - new_max);                                       \
              run_sum *= alpha;                                                                \
              for (int64_t d = 0; d < D; ++d) acc[d] *= alpha;                                 \
            }                                                                                  \
            run_max = new_max;                                                                 \
          }                                                                                    \
          for (int64_t j = j0; j < j1; ++j) { /* :135-143 */                                   \
            const Real sv = sbuf[j - j0];                                                      \
            if (sv == NEG) continue;                                                           \
            const Real p = EXP(sv - run_max);                                                  \
            run_sum += p;                                                                      \
            const Real* vrow = v + ((kb * Hkv + kh) * Lkv + j) * D;                            \
            for (int64_t d = 0; d < D; ++d) acc[d] += p * vrow[d];                             \
          }                                                                                    \
        }                                                                                      \
        Real* orow = out + ((b * Hq + h) * Lq + iq) * D; /* :146-154 */                        \
        const int64_t slot = (b * Hq + h) * Lq + iq;                                           \
        if (run_sum > (Real)0) {                                                               \
          for (int64_t d = 0; d < D; ++d) orow[d] = acc[d] / run_sum;                          \
          lse[slot] = run_max + LOG(run_sum);                                                  \
        } else {                                                                               \
          for (int64_t d = 0; d < D; ++d) orow[d] = (Real)0;                                   \
          lse[slot] = NEG;                                                                     \
        }                                                                                      \
      }                                                                                        \
    }                                                                                          \
    /* rows beyond the mask (none when bm covers Lq) keep zero output */                       \
    free(sbuf);                                                                                \
    free(acc);                                                                                 \
    free(vis);                                                                                 \
    return st;                                                                                 \
  }

FO_FORWARD(fo_forward_f32, float, expf, logf)
FO_FORWARD(fo_forward_f64, double, exp, log)

/* ---- backward (engine.cpp:174-401) ---------------------------------------- */
#define FO_BACKWARD(NAME, Real)                                                                 \
  int NAME(const Real* q, const Real* k, const Real* v, const Real* out, const Real* lse,      \
           const Real* dout, int64_t B, int64_t Hq, int64_t Hkv, int64_t Bkv, int64_t Lq,      \
           int64_t Lkv, int64_t D, double scale, int64_t gqa_group, const fo_score* s,         \
           const fo_mask* mask, const fo_bm* bm, const fo_bm* bm_t, Real* dq, Real* dk,        \
           Real* dv) {                                                                         \
    if (Hq != gqa_group * Hkv) return E_SHAPE;                                                 \
    if (bm_t->rows != bm->cols || bm_t->cols != bm->rows) return E_BM; /* :188-193 */          \
    const Real scale_r = (Real)scale;                                                          \
    const int64_t bs_q = bm->bs_q, bs_kv = bm->bs_kv;                                          \
    double* row_dot = (double*)malloc(sizeof(double) * (size_t)(B * Hq * Lq));                 \
    for (int64_t idx = 0; idx < B * Hq * Lq; ++idx) { /* :218-235 */                            \
      double a = 0.0;                                                                          \
      for (int64_t d = 0; d < D; ++d) a += (double)dout[idx * D + d] * (double)out[idx * D + d]; \
      row_dot[idx] = a;                                                                        \
    }                                                                                          \
    visit_t* vis = (visit_t*)malloc(sizeof(visit_t) * (size_t)(bm->cols > bm->rows ? bm->cols : bm->rows)); \
    double* dq_acc = (double*)malloc(sizeof(double) * (size_t)D);                              \
    int st = OK;                                                                               \
    /* pass 1: dq (:237-305) */                                                                \
    for (int64_t task = 0; task < B * Hq * bm->rows && st == OK; ++task) {                    \
      const int64_t r = task % bm->rows, h = (task / bm->rows) % Hq, b = task / (bm->rows * Hq); \
      const int64_t mb = bm->b_dims == 1 ? 0 : b, mh = bm->h_dims == 1 ? 0 : h;                \
      const int64_t kb = Bkv == 1 ? 0 : b, kh = h / gqa_group;                                 \
      const int64_t nvisit = merged_visits(bm, mb, mh, r, vis);                                \
      const int64_t q_end = (r + 1) * bs_q < Lq ? (r + 1) * bs_q : Lq;                         \
      for (int64_t iq = r * bs_q; iq < q_end && st == OK; ++iq) {                              \
        Real* dqrow = dq + ((b * Hq + h) * Lq + iq) * D;                                       \
        const int64_t slot = (b * Hq + h) * Lq + iq;                                           \
        const double lse_i = (double)lse[slot];                                                \
        if (lse_i == -INFINITY) { for (int64_t d = 0; d < D; ++d) dqrow[d] = (Real)0; continue; } \
        const Real* qrow = q + slot * D;                                                       \
        const Real* dorow = dout + slot * D;                                                   \
        const double di = row_dot[slot];                                                       \
        for (int64_t d = 0; d < D; ++d) dq_acc[d] = 0.0;                                       \
        for (int64_t vi = 0; vi < nvisit && st == OK; ++vi) {                                  \
          const int64_t c = vis[vi].c;                                                         \
          const int full = vis[vi].full;                                                       \
          const int64_t j0 = c * bs_kv, j1 = j0 + bs_kv < Lkv ? j0 + bs_kv : Lkv;              \
          for (int64_t j = j0; j < j1; ++j) {                                                  \
            if (!full) {                                                                       \
              int mv;                                                                          \
              st = fo_mask_eval(mask, b, h, iq, j, &mv);                                       \
              if (st) break;                                                                   \
              if (!mv) continue;                                                               \
            }                                                                                  \
            const Real* krow = k + ((kb * Hkv + kh) * Lkv + j) * D;                            \
            Real dot = (Real)0;                                                                \
            for (int64_t d = 0; d < D; ++d) dot += qrow[d] * krow[d];                          \
            const Real s_scaled = dot * scale_r;                                               \
            double s_mod, dap;                                                                 \
            st = fo_score_apply(s, (double)s_scaled, b, h, iq, j, &s_mod);                     \
            if (st) break;                                                                     \
            if (s_mod == -INFINITY) continue;                                                  \
            const double p = exp(s_mod - lse_i);                                               \
            const Real* vrow = v + ((kb * Hkv + kh) * Lkv + j) * D;                            \
            double dp = 0.0;                                                                   \
            for (int64_t d = 0; d < D; ++d) dp += (double)dorow[d] * (double)vrow[d];          \
            const double ds_mod = p * (dp - di);                                               \
            st = fo_score_dapply(s, (double)s_scaled, b, h, iq, j, &dap);                      \
            if (st) break;                                                                     \
            const double coeff = ds_mod * dap * scale;                                         \
            for (int64_t d = 0; d < D; ++d) dq_acc[d] += coeff * (double)krow[d];              \
          }                                                                                    \
        }                                                                                      \
        for (int64_t d = 0; d < D; ++d) dqrow[d] = (Real)dq_acc[d];                            \
      }                                                                                        \
    }                                                                                          \
    /* pass 2: dk/dv over the transposed mask (:307-395) */                                    \
    double* dk_acc = (double*)malloc(sizeof(double) * (size_t)(bs_kv * D));                    \
    double* dv_acc = (double*)malloc(sizeof(double) * (size_t)(bs_kv * D));                    \
    for (int64_t task = 0; task < Bkv * Hkv * bm_t->rows && st == OK; ++task) {               \
      const int64_t c = task % bm_t->rows, kh = (task / bm_t->rows) % Hkv;                     \
      const int64_t ob = task / (bm_t->rows * Hkv);                                            \
      const int64_t j0 = c * bs_kv, j1 = j0 + bs_kv < Lkv ? j0 + bs_kv : Lkv, nj = j1 - j0;    \
      if (nj <= 0) continue;                                                                   \
      memset(dk_acc, 0, sizeof(double) * (size_t)(nj * D));                                    \
      memset(dv_acc, 0, sizeof(double) * (size_t)(nj * D));                                    \
      const int64_t b_begin = Bkv == 1 ? 0 : ob, b_end = Bkv == 1 ? B : ob + 1;                \
      for (int64_t b = b_begin; b < b_end && st == OK; ++b) {                                  \
        const int64_t kb = Bkv == 1 ? 0 : b;                                                   \
        for (int64_t gi = 0; gi < gqa_group && st == OK; ++gi) {                               \
          const int64_t h = kh * gqa_group + gi;                                               \
          const int64_t mb = bm->b_dims == 1 ? 0 : b, mh = bm->h_dims == 1 ? 0 : h;            \
          const int64_t nvisit = merged_visits(bm_t, mb, mh, c, vis);                          \
          for (int64_t vi = 0; vi < nvisit && st == OK; ++vi) {                                \
            const int64_t r = vis[vi].c;                                                       \
            const int full = vis[vi].full;                                                     \
            const int64_t i0 = r * bs_q, i1 = i0 + bs_q < Lq ? i0 + bs_q : Lq;                 \
            for (int64_t iq = i0; iq < i1 && st == OK; ++iq) {                                 \
              const int64_t slot = (b * Hq + h) * Lq + iq;                                     \
              const double lse_i = (double)lse[slot];                                          \
              if (lse_i == -INFINITY) continue;                                                \
              const Real* qrow = q + slot * D;                                                 \
              const Real* dorow = dout + slot * D;                                             \
              const double di = row_dot[slot];                                                 \
              for (int64_t j = j0; j < j1; ++j) {                                              \
                if (!full) {                                                                   \
                  int mv;                                                                      \
                  st = fo_mask_eval(mask, b, h, iq, j, &mv);                                   \
                  if (st) break;                                                               \
                  if (!mv) continue;                                                           \
                }                                                                              \
                const Real* krow = k + ((kb * Hkv + kh) * Lkv + j) * D;                        \
                Real dot = (Real)0;                                                            \
                for (int64_t d = 0; d < D; ++d) dot += qrow[d] * krow[d];                      \
                const Real s_scaled = dot * scale_r;                                           \
                double s_mod, dap;                                                             \
                st = fo_score_apply(s, (double)s_scaled, b, h, iq, j, &s_mod);                 \
                if (st) break;                                                                 \
                if (s_mod == -INFINITY) continue;                                              \
                const double p = exp(s_mod - lse_i);                                           \
                double* dvj = dv_acc + (j - j0) * D;                                           \
                const Real* vrow = v + ((kb * Hkv + kh) * Lkv + j) * D;                        \
                double dp = 0.0;                                                               \
                for (int64_t d = 0; d < D; ++d) {                                              \
                  dvj[d] += p * (double)dorow[d];                                              \
                  dp += (double)dorow[d] * (double)vrow[d];                                    \
                }                                                                              \
                const double ds_mod = p * (dp - di);                                           \
                st = fo_score_dapply(s, (double)s_scaled, b, h, iq, j, &dap);                  \
                if (st) break;                                                                 \
                const double coeff = ds_mod * dap * scale;                                     \
                double* dkj = dk_acc + (j - j0) * D;                                           \
                for (int64_t d = 0; d < D; ++d) dkj[d] += coeff * (double)qrow[d];             \
              }                                                                                \
            }                                                                                  \
          }                                                                                    \
        }                                                                                      \
      }                                                                                        \
      for (int64_t j = j0; j < j1; ++j) { /* :384-393 */                                       \
        Real* dkrow = dk + ((ob * Hkv + kh) * Lkv + j) * D;                                    \
        Real* dvrow = dv + ((ob * Hkv + kh) * Lkv + j) * D;                                    \
        for (int64_t d = 0; d < D; ++d) {                                                      \
          dkrow[d] = (Real)dk_acc[(j - j0) * D + d];                                           \
          dvrow[d] = (Real)dv_acc[(j - j0) * D + d];                                           \
        }                                                                                      \
      }                                                                                        \
    }                                                                                          \
    free(dk_acc);                                                                              \
    free(dv_acc);                                                                              \
    free(dq_acc);                                                                              \
    free(vis);                                                                                 \
    free(row_dot);                                                                             \
    return st;                                                                                 \
  }

FO_BACKWARD(fo_backward_f32, float)
FO_BACKWARD(fo_backward_f64, double)

/* ---- dense_forward (oracle.cpp:13-76), double ----------------------------- */
int fo_dense_forward_f64(const double* q, const double* k, const double* v, int64_t B,
                         int64_t Hq, int64_t Hkv, int64_t Bkv, int64_t Lq, int64_t Lkv, int64_t D,
                         double scale, int64_t gqa_group, const fo_score* s, const fo_mask* mask,
                         double* out, double* lse) {
  if (Hq != gqa_group * Hkv) return E_SHAPE;
  double* srow = (double*)malloc(sizeof(double) * (size_t)Lkv);
  int st = OK;
  for (int64_t b = 0; b < B && st == OK; ++b)
    for (int64_t h = 0; h < Hq && st == OK; ++h) {
      const int64_t kb = Bkv == 1 ? 0 : b, kh = h / gqa_group;
      for (int64_t iq = 0; iq < Lq && st == OK; ++iq) {
        const int64_t slot = (b * Hq + h) * Lq + iq;
        const double* qrow = q + slot * D;
        double row_max = -INFINITY;
        for (int64_t j = 0; j < Lkv; ++j) {
          int mv;
          st = fo_mask_eval(mask, b, h, iq, j, &mv);
          if (st) break;
          if (!mv) { srow[j] = -INFINITY; continue; }
          const double* krow = k + ((kb * Hkv + kh) * Lkv + j) * D;
          double dot = 0.0;
          for (int64_t d = 0; d < D; ++d) dot += qrow[d] * krow[d];
          double sm;
          st = fo_score_apply(s, dot * scale, b, h, iq, j, &sm);
          if (st) break;
          srow[j] = sm;
          if (sm > row_max) row_max = sm;
        }
        double* orow = out + slot * D;
        if (st || row_max == -INFINITY) {
          for (int64_t d = 0; d < D; ++d) orow[d] = 0.0;
          lse[slot] = -INFINITY;
          continue;
        }
        double denom = 0.0;
        for (int64_t j = 0; j < Lkv; ++j) {
          srow[j] = srow[j] == -INFINITY ? 0.0 : exp(srow[j] - row_max);
          denom += srow[j];
        }
        for (int64_t d = 0; d < D; ++d) {
          double a = 0.0;
          for (int64_t j = 0; j < Lkv; ++j) a += srow[j] * v[((kb * Hkv + kh) * Lkv + j) * D + d];
          orow[d] = a / denom;
        }
        lse[slot] = row_max + log(denom);
      }
    }
  free(srow);
  return st;
}

/* ---- convert_block_mask (paged_kv.cpp:154-228), kv side ------------------- */
int fo_convert_block_mask(int64_t b_dims, int64_t h_dims, int64_t rows, int64_t cols,
                          const int64_t* partial_num, const int64_t* partial_idx,
                          const int64_t* full_num, const int64_t* full_idx, int64_t batches,
                          int64_t max_logical_pages, int64_t num_physical_pages,
                          const int32_t* table, int64_t* o_partial_num, int64_t* o_partial_idx,
                          int64_t* o_full_num, int64_t* o_full_idx) {
  if (b_dims != 1 && b_dims != batches) return E_BM; /* :159-163 */
  const int64_t ocols = num_physical_pages;
  const int64_t nrows = batches * h_dims * rows;
  memset(o_partial_num, 0, sizeof(int64_t) * (size_t)nrows);
  memset(o_full_num, 0, sizeof(int64_t) * (size_t)nrows);
  memset(o_partial_idx, 0, sizeof(int64_t) * (size_t)(nrows * ocols));
  memset(o_full_idx, 0, sizeof(int64_t) * (size_t)(nrows * ocols));
  for (int64_t b = 0; b < batches; ++b) {
    const int64_t sb = b_dims == 1 ? 0 : b;
    for (int64_t h = 0; h < h_dims; ++h)
      for (int64_t r = 0; r < rows; ++r) {
        const int64_t src = (sb * h_dims + h) * rows + r, dst = (b * h_dims + h) * rows + r;
        o_partial_num[dst] = partial_num[src];
        o_full_num[dst] = full_num[src];
        for (int64_t i = 0; i < partial_num[src]; ++i) { /* map_block :186-193 */
          const int64_t c = partial_idx[src * cols + i];
          const int32_t page = c < max_logical_pages ? table[b * max_logical_pages + c] : -1;
          if (page < 0) return E_UNMAPPED_BLOCK;
          o_partial_idx[dst * ocols + i] = page;
        }
        for (int64_t i = 0; i < full_num[src]; ++i) {
          const int64_t c = full_idx[src * cols + i];
          const int32_t page = c < max_logical_pages ? table[b * max_logical_pages + c] : -1;
          if (page < 0) return E_UNMAPPED_BLOCK;
          o_full_idx[dst * ocols + i] = page;
        }
      }
  }
  return OK;
}
