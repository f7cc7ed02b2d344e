// block_mask.cuh — BlockMask construction on sm_100a.
//
// Replaces create_block_mask (block_mask.cpp:79-115), transpose (:161-178) and
// convert_block_mask (paged_kv.cpp:154-228). Two kernels per build:
//   1. classify: one warp per (b, h, r, c) tile. The mask functor first tries a closed form
//      over the whole tile (MaskFn::tile_class: causal / sliding-window / prefix ranges,
//      document-id ranges of the tile's rows and columns, neighbourhood distances, composed
//      with AND = min / OR = max); only tiles it cannot decide are evaluated, lanes over query
//      rows and mask_mod 32 kv positions per word (MaskFn::bits32), leaving early as soon as
//      the tile is provably mixed (the reference's early exit, :96-105). Ragged tiles are
//      never FULL (:91-94). Output: one byte per tile.
//   2. compact: one warp per kv-side row and per q-side column (one launch) turns the byte
//      grid into ascending compacted index lists with ballot + popc prefix sums, counts and
//      zero-filled tails (:50-52): kv_num_blocks / kv_indices / full_kv_* and the q side.
// All integer work; HBM traffic is the grid plus the int32 outputs.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "host.cuh"
#include "mods.cuh"

namespace fa {
namespace bmk {
namespace {  // internal linkage: every including translation unit has its own copy

constexpr uint8_t kEmpty = 0, kPartial = 1, kFull = 2;

template <class MaskT>
__global__ void __launch_bounds__(256) classify_kernel(MaskT mask, int b_dims, int h_dims,
                                                       int rows, int cols, int q_len, int kv_len,
                                                       int bs_q, int bs_kv, uint8_t* __restrict__ grid) {
  const int lane = threadIdx.x & 31;
  const long long warp_global = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const long long ntiles = static_cast<long long>(b_dims) * h_dims * rows * cols;
  for (long long tile = warp_global; tile < ntiles; tile += nwarps) {
    const int c = static_cast<int>(tile % cols);
    const int r = static_cast<int>((tile / cols) % rows);
    const int h = static_cast<int>((tile / (static_cast<long long>(cols) * rows)) % h_dims);
    const int b = static_cast<int>(tile / (static_cast<long long>(cols) * rows * h_dims));
    const int q0 = r * bs_q, q1 = min(q0 + bs_q, q_len);
    const int k0 = c * bs_kv, k1 = min(k0 + bs_kv, kv_len);
    const bool ragged = (q1 - q0 != bs_q) || (k1 - k0 != bs_kv);
    // closed form first (causal / sliding / prefix ranges, document id ranges, ...)
    const int cls = mask.tile_class(b, h, q0, q1, k0, k1, lane);
    bool any = cls == kTileAll, all = cls == kTileAll;
    if (cls == kTileMixed) {
      // evaluate: lanes take query rows, mask_mod 32 kv positions per word (bits32); stop as
      // soon as the tile is provably mixed (the reference's early exit, block_mask.cpp:96-105)
      any = false;
      all = true;
      for (int qb = q0; qb < q1; qb += 32) {
        const int q = qb + lane;
        bool my_any = false, my_all = true;
        if (q < q1) {
          for (int kw = k0; kw < k1; kw += 32) {
            const uint32_t valid = range_bits32(kw, kw, k1 - 1);
            const uint32_t bits = mask.bits32(b, h, q, kw, k1) & valid;
            my_any |= bits != 0u;
            my_all &= bits == valid;
          }
        }
        any = __any_sync(0xffffffffu, my_any) || any;
        all = __all_sync(0xffffffffu, my_all) && all;
        if (any && !all) break;
      }
    }
    // ragged tiles are never FULL (block_mask.cpp:91-94)
    if (lane == 0) grid[tile] = !any ? kEmpty : ((all && !ragged) ? kFull : kPartial);
  }
}

// Compacts `nlines` lines of `len` tiles each. Line i's tile j lives at
// grid[base(i) + j*stride]; outputs are (nlines) counts and (nlines, len) indices.
__global__ void __launch_bounds__(256) compact_kernel(const uint8_t* __restrict__ grid, int nlines,
                                                      int len, int lines_per_bh, int bh_stride,
                                                      int line_stride, int elem_stride,
                                                      int32_t* __restrict__ part_num,
                                                      int32_t* __restrict__ part_idx,
                                                      int32_t* __restrict__ full_num,
                                                      int32_t* __restrict__ full_idx) {
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int line = warp_global; line < nlines; line += nwarps) {
    const int bh = line / lines_per_bh, li = line % lines_per_bh;
    const long long base = static_cast<long long>(bh) * bh_stride + static_cast<long long>(li) * line_stride;
    int np = 0, nf = 0;
    int32_t* pi = part_idx + static_cast<long long>(line) * len;
    int32_t* fi = full_idx + static_cast<long long>(line) * len;
    for (int j0 = 0; j0 < len; j0 += 32) {
      const int j = j0 + lane;
      const uint8_t kind = j < len ? grid[base + static_cast<long long>(j) * elem_stride] : kEmpty;
      const unsigned pm = __ballot_sync(0xffffffffu, kind == kPartial);
      const unsigned fm = __ballot_sync(0xffffffffu, kind == kFull);
      const unsigned lower = (1u << lane) - 1u;
      if (kind == kPartial) pi[np + __popc(pm & lower)] = j;   // push_block :65-66
      if (kind == kFull) fi[nf + __popc(fm & lower)] = j;      // push_block :62-64
      np += __popc(pm);
      nf += __popc(fm);
    }
    for (int j = np + lane; j < len; j += 32) pi[j] = 0;        // zero tails, make_empty :50-52
    for (int j = nf + lane; j < len; j += 32) fi[j] = 0;
    if (lane == 0) {
      part_num[line] = np;
      full_num[line] = nf;
    }
  }
}

// Both sides in one launch: warps [0, nrows) compact kv-side rows, the rest q-side columns.
__global__ void __launch_bounds__(256) compact_both_kernel(const uint8_t* __restrict__ grid, int bh, int rows,
                                                           int cols, int32_t* __restrict__ kpn,
                                                           int32_t* __restrict__ kpi, int32_t* __restrict__ kfn,
                                                           int32_t* __restrict__ kfi, int32_t* __restrict__ qpn,
                                                           int32_t* __restrict__ qpi, int32_t* __restrict__ qfn,
                                                           int32_t* __restrict__ qfi) {
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nrows = bh * rows, nlines = nrows + (qpn != nullptr ? bh * cols : 0);
  for (int line = warp_global; line < nlines; line += nwarps) {
    const bool kv_side = line < nrows;
    const int li = kv_side ? line : line - nrows;
    const int per = kv_side ? rows : cols;            // lines per (b, h)
    const int len = kv_side ? cols : rows;            // elements per line
    const int bhi = li / per, l = li % per;
    const long long base = static_cast<long long>(bhi) * rows * cols + (kv_side ? static_cast<long long>(l) * cols : l);
    const int estride = kv_side ? 1 : cols;
    int32_t* pi = (kv_side ? kpi : qpi) + static_cast<long long>(li) * len;
    int32_t* fi = (kv_side ? kfi : qfi) + static_cast<long long>(li) * len;
    int np = 0, nf = 0;
    for (int j0 = 0; j0 < len; j0 += 32) {
      const int j = j0 + lane;
      const uint8_t kind = j < len ? grid[base + static_cast<long long>(j) * estride] : kEmpty;
      const unsigned pm = __ballot_sync(0xffffffffu, kind == kPartial);
      const unsigned fm = __ballot_sync(0xffffffffu, kind == kFull);
      const unsigned lower = (1u << lane) - 1u;
      if (kind == kPartial) pi[np + __popc(pm & lower)] = j;   // push_block :65-66
      if (kind == kFull) fi[nf + __popc(fm & lower)] = j;      // push_block :62-64
      np += __popc(pm);
      nf += __popc(fm);
    }
    for (int j = np + lane; j < len; j += 32) pi[j] = 0;        // zero tails, make_empty :50-52
    for (int j = nf + lane; j < len; j += 32) fi[j] = 0;
    if (lane == 0) {
      (kv_side ? kpn : qpn)[li] = np;
      (kv_side ? kfn : qfn)[li] = nf;
    }
  }
}

// Rebuild the kind grid from kv-side lists (to_dense, block_mask.cpp:117-138).
__global__ void scatter_kinds_kernel(int nrows, int cols, const int32_t* __restrict__ pn,
                                     const int32_t* __restrict__ pi, const int32_t* __restrict__ fn,
                                     const int32_t* __restrict__ fi, uint8_t* __restrict__ grid) {
  const int row = blockIdx.x;
  if (row >= nrows) return;
  uint8_t* g = grid + static_cast<long long>(row) * cols;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) g[c] = kEmpty;
  __syncthreads();
  const int np = pn[row], nf = fn[row];
  for (int i = threadIdx.x; i < np; i += blockDim.x) g[pi[static_cast<long long>(row) * cols + i]] = kPartial;
  for (int i = threadIdx.x; i < nf; i += blockDim.x) g[fi[static_cast<long long>(row) * cols + i]] = kFull;
}

// convert_block_mask (paged_kv.cpp:154-228): logical column -> physical page.
__global__ void convert_kernel(int batches, int h_dims, int rows, int cols, int src_b_dims,
                               const int32_t* __restrict__ pn, const int32_t* __restrict__ pi,
                               const int32_t* __restrict__ fn, const int32_t* __restrict__ fi,
                               const int32_t* __restrict__ table, int max_logical_pages,
                               int out_cols, int32_t* __restrict__ opn, int32_t* __restrict__ opi,
                               int32_t* __restrict__ ofn, int32_t* __restrict__ ofi,
                               int* __restrict__ err) {
  const int line = blockIdx.x;  // (b, h, r) of the output
  const int nlines = batches * h_dims * rows;
  if (line >= nlines) return;
  const int r = line % rows, h = (line / rows) % h_dims, b = line / (rows * h_dims);
  const int sb = src_b_dims == 1 ? 0 : b;
  const long long src = (static_cast<long long>(sb) * h_dims + h) * rows + r;
  const int np = pn[src], nf = fn[src];
  int32_t* o_pi = opi + static_cast<long long>(line) * out_cols;
  int32_t* o_fi = ofi + static_cast<long long>(line) * out_cols;
  for (int i = threadIdx.x; i < out_cols; i += blockDim.x) {
    int32_t vp = 0, vf = 0;
    if (i < np) {
      const int c = pi[src * cols + i];
      vp = c < max_logical_pages ? table[static_cast<long long>(b) * max_logical_pages + c] : -1;
      if (vp < 0) { atomicExch(err, 1); vp = 0; }
    }
    if (i < nf) {
      const int c = fi[src * cols + i];
      vf = c < max_logical_pages ? table[static_cast<long long>(b) * max_logical_pages + c] : -1;
      if (vf < 0) { atomicExch(err, 1); vf = 0; }
    }
    o_pi[i] = vp;
    o_fi[i] = vf;
  }
  if (threadIdx.x == 0) {
    opn[line] = np;
    ofn[line] = nf;
  }
}

inline int grid_for(long long warps_needed) {
  const long long blocks = (warps_needed * 32 + 255) / 256;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(blocks, 148LL * 16)));
}


template <class MaskT>
void launch_classify(MaskT m, int bd, int hd, int rows, int cols, int ql, int kl, int bsq,
                            int bskv, uint8_t* grid, cudaStream_t st) {
  const long long tiles = static_cast<long long>(bd) * hd * rows * cols;
  classify_kernel<MaskT><<<grid_for(tiles), 256, 0, st>>>(m, bd, hd, rows, cols, ql, kl, bsq, bskv, grid);
  count_launch();
}

inline fa_status compact_both(int bd, int hd, int rows, int cols, const uint8_t* grid,
                              fa_block_mask* bm, cudaStream_t st) {
  const long long lines = static_cast<long long>(bd) * hd * (rows + (bm->q_num_blocks != nullptr ? cols : 0));
  compact_both_kernel<<<grid_for(lines), 256, 0, st>>>(grid, bd * hd, rows, cols, bm->kv_num_blocks,
                                                       bm->kv_indices, bm->full_kv_num_blocks,
                                                       bm->full_kv_indices, bm->q_num_blocks, bm->q_indices,
                                                       bm->full_q_num_blocks, bm->full_q_indices);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}


// fa_block_mask_geometry (make_empty's checks, block_mask.cpp:29-55)
inline fa_status geometry(int64_t b_dims, int64_t h_dims, int64_t q_len, int64_t kv_len, int64_t bs_q,
                          int64_t bs_kv, int64_t* rows, int64_t* cols, size_t* ws) {
  FA_REQUIRE(b_dims >= 1 && h_dims >= 1, FA_SHAPE_MISMATCH, "create_block_mask: mask dims must be >= 1");
  FA_REQUIRE(q_len >= 1 && kv_len >= 1 && bs_q >= 1 && bs_kv >= 1, FA_SHAPE_MISMATCH,
             "create_block_mask: lengths and block sizes must be >= 1");
  const int64_t r = (q_len + bs_q - 1) / bs_q, c = (kv_len + bs_kv - 1) / bs_kv;
  FA_REQUIRE(b_dims * h_dims * r * c < (int64_t(1) << 31), FA_SHAPE_MISMATCH,
             "create_block_mask: block grid too large");
  if (rows) *rows = r;
  if (cols) *cols = c;
  if (ws) *ws = static_cast<size_t>(b_dims * h_dims * r * c);
  return FA_OK;
}

// create_block_mask + transpose (block_mask.cpp:79-115, :161-178) for any mask functor: the
// geometry fields of `bm` are written, its caller-allocated arrays filled (q side when non-NULL).
template <class MaskT>
fa_status build(MaskT mask, int64_t b_dims, int64_t h_dims, int64_t q_len, int64_t kv_len, int64_t bs_q,
                int64_t bs_kv, fa_block_mask* bm, void* workspace, size_t workspace_bytes, cudaStream_t st) {
  int64_t rows = 0, cols = 0;
  size_t need = 0;
  fa_status s = geometry(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, &rows, &cols, &need);
  if (s != FA_OK) return s;
  FA_REQUIRE(bm != nullptr, FA_SHAPE_MISMATCH, "create_block_mask: NULL argument");
  FA_REQUIRE(workspace != nullptr && workspace_bytes >= need, FA_SHAPE_MISMATCH,
             "create_block_mask: workspace too small");
  FA_REQUIRE(bm->kv_num_blocks && bm->kv_indices && bm->full_kv_num_blocks && bm->full_kv_indices,
             FA_SHAPE_MISMATCH, "create_block_mask: kv-side arrays must be allocated");
  bm->b_dims = b_dims;
  bm->h_dims = h_dims;
  bm->rows = rows;
  bm->cols = cols;
  bm->bs_q = bs_q;
  bm->bs_kv = bs_kv;
  bm->q_len = q_len;
  bm->kv_len = kv_len;
  uint8_t* grid = static_cast<uint8_t*>(workspace);
  const int bd = (int)b_dims, hd = (int)h_dims, R = (int)rows, Cc = (int)cols;
  launch_classify(mask, bd, hd, R, Cc, (int)q_len, (int)kv_len, (int)bs_q, (int)bs_kv, grid, st);
  FA_CHECK_CUDA(cudaGetLastError());
  return compact_both(bd, hd, R, Cc, grid, bm, st);
}

}  // namespace
}  // namespace bmk
}  // namespace fa
