// page_pool.cu — the PagedKVCache allocator on the device (paged_kv.hpp:50-89,
// paged_kv.cpp:13-152): free stack, page table, phys->logical map, owners and sequence
// lengths live in HBM and are updated by kernels, so a serving step never round-trips
// through the host.
//
// A batched update applies its requests in order with the reference's sequential semantics:
//   * append / erase requests of distinct sequences touch disjoint table rows, so their page
//     pops / pushes are placed by a prefix sum over the requests (request i pops the stack
//     slots count-1-S_i-j, S_i = pages popped before it) and run in parallel;
//   * assign = erase + pop on the same stack per request, whose pops can return pages the
//     same request just pushed, so the requests run one after another inside one CTA (the
//     threads of the CTA share each request's pushes and pops);
//   * the first failing request stops the batch (its predecessors stay applied), like the
//     exception of the reference's failing call.
// Token writes of the applied requests (write_tokens, paged_kv.cpp:54-70) follow in a
// second, grid-wide kernel: one warp per (token, head) row, 16-byte copies.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <string>

#include "internal.h"

namespace fa {
namespace {

constexpr int kThreads = 512;
enum { kStCode = 0, kStIndex = 1, kStNeeded = 2, kStAvail = 3, kStTokens = 4, kStOp = 5, kStBatch = 6, kStReason = 7 };
enum { kReasonTokens = 1, kReasonDuplicate = 2 };
enum { kMetaApplied = 0, kMetaTokens = 1 };

struct PoolView {
  int B, P, ps;
  int32_t *table, *p2l, *owner, *seq, *stack, *count, *status;
  int32_t *req_start, *req_off, *mark, *meta;  // scratch: B, B + 1, B, 4
};

PoolView view_of(const fa_page_pool& p) {
  PoolView v{};
  v.B = static_cast<int>(p.batches);
  v.P = static_cast<int>(p.num_pages);
  v.ps = static_cast<int>(p.page_size);
  v.table = p.table; v.p2l = p.phys_to_logical; v.owner = p.owner; v.seq = p.seq_len;
  v.stack = p.free_stack; v.count = p.free_count; v.status = p.status;
  v.req_start = p.scratch;
  v.req_off = p.scratch + v.B;
  v.mark = p.scratch + 2 * v.B + 1;
  v.meta = p.scratch + 3 * v.B + 1;
  return v;
}

__global__ void pool_init_kernel(PoolView v) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < (long long)v.B * v.P; i += stride) v.table[i] = -1;
  for (long long i = tid; i < v.P; i += stride) {
    v.p2l[i] = -1;
    v.owner[i] = -1;
    v.stack[i] = v.P - 1 - static_cast<int>(i);  // LIFO: page 0 on top (paged_kv.cpp:27-31)
  }
  for (long long i = tid; i < v.B; i += stride) {
    v.seq[i] = 0;
    v.mark[i] = INT_MAX;
  }
  if (tid == 0) {
    *v.count = v.P;
    for (int i = 0; i < 8; ++i) v.status[i] = 0;
    for (int i = 0; i < 4; ++i) v.meta[i] = 0;
  }
}

// deterministic_shuffle (random.hpp:49-56) of the free stack: a sequential Fisher-Yates walk
// over SplitMix64 draws, one thread (a one-time setup step).
__global__ void pool_shuffle_kernel(PoolView v, unsigned long long seed) {
  unsigned long long state = seed;
  const int n = *v.count;
  for (int i = n; i > 1; --i) {
    state += 0x9e3779b97f4a7c15ull;
    unsigned long long z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    const int j = static_cast<int>(z % static_cast<unsigned long long>(i));
    const int32_t t = v.stack[i - 1];
    v.stack[i - 1] = v.stack[j];
    v.stack[j] = t;
  }
}

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Exclusive block-wide prefix sum of x (every thread of the CTA calls it); *total = the sum.
__device__ int block_excl_scan(int x, int* total) {
  __shared__ int warp_sums[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_sums[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const int before = warp == 0 ? 0 : warp_sums[warp - 1];
  *total = warp_sums[(blockDim.x >> 5) - 1];
  __syncthreads();  // warp_sums is reused by the next call
  return before + incl - x;
}

__device__ int block_min(int x) {
  __shared__ int red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  x = __reduce_min_sync(0xffffffffu, x);
  if (lane == 0) red[warp] = x;
  __syncthreads();
  int r = lane < (int)(blockDim.x >> 5) ? red[lane] : INT_MAX;
  r = __reduce_min_sync(0xffffffffu, r);
  __syncthreads();
  return r;
}

// One CTA of kThreads threads applies the n requests; see the file comment.
__global__ void __launch_bounds__(kThreads) pool_update_kernel(PoolView v, int op, const int32_t* ids,
                                                               const int32_t* ntok, int n, int token_len) {
  __shared__ int s_fail, s_code, s_carry;
  const int tid = threadIdx.x;
  const bool with_tokens = op != FA_PAGE_ERASE;
  if (tid == 0) {
    s_fail = n;
    s_code = FA_OK;
    s_carry = 0;
    for (int i = 0; i < 8; ++i) v.status[i] = 0;
    v.status[kStOp] = op;
  }
  __syncthreads();
  // token offsets of the packed token tensor (all requests, applied or not)
  for (int base = 0; base < n; base += kThreads) {
    const int i = base + tid;
    const int x = (i < n && with_tokens) ? ntok[i] : 0;
    int tot;
    const int ex = block_excl_scan(x, &tot);
    if (i < n) v.req_off[i] = s_carry + ex;
    __syncthreads();
    if (tid == 0) s_carry += tot;
    __syncthreads();
  }
  if (tid == 0) {
    v.req_off[n] = s_carry;
    if (with_tokens && token_len >= 0 && s_carry != token_len) {  // nothing is applied
      s_fail = 0;
      s_code = FA_SHAPE_MISMATCH;
      v.status[kStReason] = kReasonTokens;
      v.status[kStTokens] = s_carry;
      v.status[kStAvail] = token_len;
    }
  }
  __syncthreads();
  // range and duplicate checks: the first bad request bounds the batch
  for (int i = tid; i < n; i += kThreads) {
    const int b = ids[i];
    if (b >= 0 && b < v.B) atomicMin(&v.mark[b], i);
  }
  __syncthreads();
  int bad = INT_MAX;
  for (int i = tid; i < n; i += kThreads) {
    const int b = ids[i];
    if (b < 0 || b >= v.B || v.mark[b] != i) bad = min(bad, i);
  }
  bad = block_min(bad);
  for (int i = tid; i < n; i += kThreads) {
    const int b = ids[i];
    if (b >= 0 && b < v.B) v.mark[b] = INT_MAX;
  }
  if (tid == 0 && bad < s_fail) {
    s_fail = bad;
    const int b = ids[bad];
    s_code = (b < 0 || b >= v.B) ? FA_INDEX_OUT_OF_RANGE : FA_SHAPE_MISMATCH;
    if (s_code == FA_SHAPE_MISMATCH) v.status[kStReason] = kReasonDuplicate;
    v.status[kStBatch] = b;
  }
  __syncthreads();
  const int limit0 = s_fail;
  int count = *v.count;
  const int ps = v.ps, P = v.P;

  if (op == FA_PAGE_ASSIGN) {
    // erase + pop per request, in order (assign, paged_kv.cpp:72-98)
    int i = 0;
    for (; i < limit0; ++i) {
      const int b = ids[i], nt = ntok[i];
      const int owned = ceil_div(v.seq[b], ps), needed = ceil_div(nt, ps);
      if (needed > count + owned) {  // capacity check before any mutation (:81-87)
        if (tid == 0) {
          s_fail = i;
          s_code = FA_OUT_OF_PAGES;
          v.status[kStNeeded] = needed;
          v.status[kStAvail] = count + owned;
          v.status[kStTokens] = nt;
        }
        break;
      }
      for (int lp = tid; lp < owned; lp += kThreads) {  // erase (:128-141): push in logical order
        const int page = v.table[b * P + lp];
        v.table[b * P + lp] = -1;
        v.p2l[page] = -1;
        v.owner[page] = -1;
        v.stack[count + lp] = page;
      }
      __syncthreads();
      count += owned;
      for (int lp = tid; lp < needed; lp += kThreads) {
        const int page = v.stack[count - 1 - lp];
        v.table[b * P + lp] = page;
        v.p2l[page] = lp;
        v.owner[page] = b;
      }
      count -= needed;
      if (tid == 0) {
        v.seq[b] = nt;
        v.req_start[i] = 0;
      }
      __syncthreads();
    }
  } else {
    // append (:100-126) / erase (:128-141): prefix sum of the pages each request pops / pushes
    s_carry = 0;
    __syncthreads();
    int fail = limit0;
    for (int base = 0; base < limit0; base += kThreads) {
      const int i = base + tid;
      int b = 0, old = 0, owned = 0, x = 0;
      if (i < limit0) {
        b = ids[i];
        old = v.seq[b];
        owned = ceil_div(old, ps);
        x = op == FA_PAGE_APPEND ? ceil_div(old + ntok[i], ps) - owned : owned;
      }
      int tot;
      const int ex = s_carry + block_excl_scan(x, &tot);
      // the first append whose pops exceed the free pages fails (S is monotone)
      int f = (op == FA_PAGE_APPEND && i < limit0 && ex + x > count) ? i : INT_MAX;
      f = block_min(f);
      if (f < fail) {
        fail = f;
        if (tid == 0) {
          s_code = FA_OUT_OF_PAGES;
          s_fail = f;
        }
        if (i == f) {
          v.status[kStNeeded] = x;
          v.status[kStAvail] = count - ex;
          v.status[kStTokens] = ntok[i];
        }
      }
      if (i < fail) {
        if (op == FA_PAGE_APPEND) {
          for (int j = 0; j < x; ++j) {
            const int page = v.stack[count - 1 - ex - j];
            v.table[b * P + owned + j] = page;
            v.p2l[page] = owned + j;
            v.owner[page] = b;
          }
          v.req_start[i] = old;
          v.seq[b] = old + ntok[i];
        } else {
          for (int lp = 0; lp < owned; ++lp) {
            const int page = v.table[b * P + lp];
            v.table[b * P + lp] = -1;
            v.p2l[page] = -1;
            v.owner[page] = -1;
            v.stack[count + ex + lp] = page;
          }
          v.seq[b] = 0;
        }
      }
      __syncthreads();
      if (tid == 0) s_carry += tot;
      __syncthreads();
      if (fail < limit0) break;
    }
    // pages moved by the applied requests
    int moved = 0;
    for (int i = tid; i < fail; i += kThreads) {
      const int b = ids[i];
      if (op == FA_PAGE_APPEND) moved += ceil_div(v.seq[b], ps) - ceil_div(v.req_start[i], ps);
    }
    if (op == FA_PAGE_APPEND) {
      int tot;
      block_excl_scan(moved, &tot);
      count -= tot;
    } else {
      count += s_carry;  // erase never fails past limit0; every owned page was pushed
    }
  }
  __syncthreads();
  if (tid == 0) {
    *v.count = count;
    v.status[kStCode] = s_code;
    v.status[kStIndex] = s_fail;
    v.meta[kMetaApplied] = s_fail;
    v.meta[kMetaTokens] = v.req_off[s_fail];
    if (s_code == FA_OUT_OF_PAGES || s_code == FA_INDEX_OUT_OF_RANGE) v.status[kStBatch] = ids[s_fail];
  }
}

// write_tokens (paged_kv.cpp:54-70) for the applied requests: one warp per (token, head) row
// of K and of V; rows are `cpr` 16-byte chunks.
__global__ void pool_write_kernel(PoolView v, const int32_t* ids, int n, const uint4* kt, const uint4* vt,
                                  uint4* kc, uint4* vc, int heads, int token_len, int cpr) {
  const int applied = v.meta[kMetaApplied];
  const int tokens = v.meta[kMetaTokens];  // tokens of the applied requests (a prefix)
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long cache_len = (long long)v.P * v.ps;
  for (long long w = warp; w < (long long)tokens * heads; w += nwarps) {
    const int g = static_cast<int>(w % tokens), h = static_cast<int>(w / tokens);
    int lo = 0, hi = applied - 1;  // last request with req_off <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (v.req_off[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const int b = ids[lo];
    const int pos = v.req_start[lo] + (g - v.req_off[lo]);
    const int page = v.table[b * v.P + pos / v.ps];
    const long long phys = (long long)page * v.ps + pos % v.ps;
    const long long src = ((long long)h * token_len + g) * cpr;
    const long long dst = ((long long)h * cache_len + phys) * cpr;
    for (int c = lane; c < cpr; c += 32) {
      kc[dst + c] = kt[src + c];
      vc[dst + c] = vt[src + c];
    }
  }
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace
}  // namespace fa

using namespace fa;

extern "C" {

size_t fa_page_pool_bytes(int64_t batches, int64_t num_pages) {
  if (batches < 1 || num_pages < 1) return 0;
  const size_t B = static_cast<size_t>(batches), P = static_cast<size_t>(num_pages);
  return al256(B * P * 4) + 3 * al256(P * 4) + al256(B * 4) + al256(64) + al256((4 * B + 8) * 4);
}

fa_status fa_page_pool_init(fa_page_pool* pool, void* mem, size_t bytes, int64_t batches, int64_t num_pages,
                            int64_t page_size, void* stream) {
  clear_error();
  FA_REQUIRE(pool != nullptr && mem != nullptr, FA_SHAPE_MISMATCH, "page_pool_init: NULL argument");
  FA_REQUIRE(batches >= 1 && num_pages >= 1 && page_size >= 1, FA_SHAPE_MISMATCH,
             "PagedKVCache: batches, num_pages and page_size must be >= 1");
  FA_REQUIRE(batches * num_pages < INT_MAX && num_pages * page_size < INT_MAX, FA_UNSUPPORTED,
             "page_pool_init: table or cache length exceeds int32 indexing");
  FA_REQUIRE(bytes >= fa_page_pool_bytes(batches, num_pages), FA_SHAPE_MISMATCH,
             "page_pool_init: device memory smaller than fa_page_pool_bytes");
  const size_t B = static_cast<size_t>(batches), P = static_cast<size_t>(num_pages);
  char* p = static_cast<char*>(mem);
  auto take = [&](size_t n) { int32_t* r = reinterpret_cast<int32_t*>(p); p += al256(n); return r; };
  pool->batches = batches;
  pool->num_pages = num_pages;
  pool->page_size = page_size;
  pool->table = take(B * P * 4);
  pool->phys_to_logical = take(P * 4);
  pool->owner = take(P * 4);
  pool->free_stack = take(P * 4);
  pool->seq_len = take(B * 4);
  pool->free_count = take(64);
  pool->status = pool->free_count + 8;
  pool->scratch = take((4 * B + 8) * 4);
  const PoolView v = view_of(*pool);
  const long long work = std::max<long long>(static_cast<long long>(B * P), static_cast<long long>(P));
  const int blocks = static_cast<int>(std::min<long long>((work + 255) / 256, 148LL * 8));
  pool_init_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(v);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

fa_status fa_page_pool_shuffle(const fa_page_pool* pool, uint64_t seed, void* stream) {
  clear_error();
  FA_REQUIRE(pool != nullptr && pool->free_stack != nullptr, FA_SHAPE_MISMATCH, "page_pool_shuffle: NULL pool");
  pool_shuffle_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(view_of(*pool), seed);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

fa_status fa_page_pool_status(const fa_page_pool* pool, int32_t* applied, void* stream) {
  clear_error();
  FA_REQUIRE(pool != nullptr && pool->status != nullptr, FA_SHAPE_MISMATCH, "page_pool_status: NULL pool");
  int32_t st[8];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FA_CHECK_CUDA(cudaMemcpyAsync(st, pool->status, sizeof(st), cudaMemcpyDeviceToHost, s));
  FA_CHECK_CUDA(cudaStreamSynchronize(s));
  if (applied != nullptr) *applied = st[kStIndex];
  const std::string who = "PagedKVCache: ";
  switch (st[kStCode]) {
    case FA_OK: return FA_OK;
    case FA_OUT_OF_PAGES:
      if (st[kStOp] == FA_PAGE_ASSIGN)  // paged_kv.cpp:83-86
        return set_error(FA_OUT_OF_PAGES, who + "assign of " + std::to_string(st[kStTokens]) + " tokens needs " +
                                              std::to_string(st[kStNeeded]) + " pages, only " +
                                              std::to_string(st[kStAvail]) + " available");
      return set_error(FA_OUT_OF_PAGES, who + "append of " + std::to_string(st[kStTokens]) +  // :111-115
                                            " tokens needs " + std::to_string(st[kStNeeded]) +
                                            " new pages, only " + std::to_string(st[kStAvail]) + " free");
    case FA_INDEX_OUT_OF_RANGE:  // check_batch, paged_kv.cpp:34-39
      return set_error(FA_INDEX_OUT_OF_RANGE, who + "batch " + std::to_string(st[kStBatch]) + " outside [0, " +
                                                  std::to_string(pool->batches) + ")");
    case FA_SHAPE_MISMATCH:
      if (st[kStReason] == kReasonTokens)
        return set_error(FA_SHAPE_MISMATCH, who + "token tensors hold " + std::to_string(st[kStAvail]) +
                                                " tokens but the requests need " + std::to_string(st[kStTokens]));
      return set_error(FA_SHAPE_MISMATCH, who + "batch " + std::to_string(st[kStBatch]) +
                                              " appears twice in one batched update (request " +
                                              std::to_string(st[kStIndex]) + ")");
    default:
      return set_error(st[kStCode], who + "update failed with status " + std::to_string(st[kStCode]));
  }
}

fa_status fa_page_pool_update(const fa_page_pool* pool, int32_t op, const int32_t* batch_ids,
                              const int32_t* n_tokens, int32_t n, const fa_tensor* kt, const fa_tensor* vt,
                              fa_tensor* kc, fa_tensor* vc, uint32_t flags, void* stream) {
  clear_error();
  FA_REQUIRE(pool != nullptr && pool->table != nullptr, FA_SHAPE_MISMATCH, "page_pool_update: NULL pool");
  FA_REQUIRE(op == FA_PAGE_ASSIGN || op == FA_PAGE_APPEND || op == FA_PAGE_ERASE, FA_SHAPE_MISMATCH,
             "page_pool_update: unknown op");
  FA_REQUIRE(n >= 0 && n <= pool->batches, FA_SHAPE_MISMATCH,
             "page_pool_update: n must be in [0, batches] (one request per sequence)");
  FA_REQUIRE(!(flags & ~uint32_t(FA_FLAG_NO_SYNC)), FA_SHAPE_MISMATCH, "page_pool_update: unknown flags");
  FA_REQUIRE(n == 0 || batch_ids != nullptr, FA_SHAPE_MISMATCH, "page_pool_update: NULL batch_ids");
  FA_REQUIRE(op == FA_PAGE_ERASE || n == 0 || n_tokens != nullptr, FA_SHAPE_MISMATCH,
             "page_pool_update: NULL n_tokens");
  const bool tokens = op != FA_PAGE_ERASE && kt != nullptr;
  int cpr = 0, heads = 0, token_len = -1;
  if (tokens) {
    FA_REQUIRE(vt != nullptr && kc != nullptr && vc != nullptr && kt->data && vt->data && kc->data && vc->data,
               FA_SHAPE_MISMATCH, "page_pool_update: token and cache tensors must all be given");
    FA_REQUIRE(kt->b == vt->b && kt->h == vt->h && kt->l == vt->l && kt->d == vt->d && kt->dtype == vt->dtype,
               FA_SHAPE_MISMATCH, "PagedKVCache: k tokens and v tokens must agree");
    FA_REQUIRE(kc->b == 1 && vc->b == 1 && kc->h == vc->h && kc->l == vc->l && kc->d == vc->d &&
                   kc->l == pool->num_pages * pool->page_size,
               FA_SHAPE_MISMATCH, "page_pool_update: cache must be (1, Hkv, num_pages * page_size, D)");
    FA_REQUIRE(kt->b == 1 && kt->h == kc->h && kt->d == kc->d && kt->dtype == kc->dtype && vc->dtype == kc->dtype,
               FA_SHAPE_MISMATCH,
               "PagedKVCache: token tensors must be (1," + std::to_string(kc->h) + ",n," + std::to_string(kc->d) + ")");
    const int esz = kt->dtype == FA_F32 ? 4 : 2;
    FA_REQUIRE((kt->d * esz) % 16 == 0, FA_UNSUPPORTED, "page_pool_update: row bytes must be a multiple of 16");
    FA_REQUIRE(kt->l * kt->h * kt->d < INT_MAX, FA_UNSUPPORTED, "page_pool_update: token tensor too large");
    cpr = static_cast<int>(kt->d * esz / 16);
    heads = static_cast<int>(kt->h);
    token_len = static_cast<int>(kt->l);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const PoolView v = view_of(*pool);
  pool_update_kernel<<<1, kThreads, 0, st>>>(v, op, batch_ids, n_tokens, n, token_len);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  if (tokens && token_len > 0) {
    const long long rows = static_cast<long long>(token_len) * heads;
    const int blocks = static_cast<int>(std::min<long long>((rows + 7) / 8, static_cast<long long>(num_sms()) * 8));
    pool_write_kernel<<<blocks, 256, 0, st>>>(v, batch_ids, n, static_cast<const uint4*>(kt->data),
                                               static_cast<const uint4*>(vt->data), static_cast<uint4*>(kc->data),
                                               static_cast<uint4*>(vc->data), heads, token_len, cpr);
    count_launch();
    FA_CHECK_CUDA(cudaGetLastError());
  }
  if (flags & FA_FLAG_NO_SYNC) return FA_OK;
  return fa_page_pool_status(pool, nullptr, stream);
}

fa_page_table fa_page_pool_table(const fa_page_pool* pool) {
  fa_page_table t{};
  if (pool == nullptr) return t;
  t.batches = pool->batches;
  t.max_logical_pages = pool->num_pages;
  t.num_physical_pages = pool->num_pages;
  t.page_size = pool->page_size;
  t.table = pool->table;
  t.phys_to_logical = pool->phys_to_logical;
  t.owner = pool->owner;
  t.seq_len = pool->seq_len;
  t.max_seq_len = 0;
  return t;
}

}  // extern "C"
