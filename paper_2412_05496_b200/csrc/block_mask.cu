// block_mask.cu — the C ABI of the BlockMask builder (create_block_mask / transpose,
// block_mask.cpp:79-115, :161-178) and of convert_block_mask (paged_kv.cpp:154-228) over the
// kernels in include/flexattn_b200/block_mask.cuh, for the built-in mask functors.
#include <string>

#include "internal.h"
#include "flexattn_b200/block_mask.cuh"

using namespace fa;

extern "C" fa_status fa_block_mask_geometry(int64_t b_dims, int64_t h_dims, int64_t q_len,
                                            int64_t kv_len, int64_t bs_q, int64_t bs_kv,
                                            int64_t* rows, int64_t* cols, size_t* ws) {
  clear_error();
  return bmk::geometry(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, rows, cols, ws);
}

extern "C" fa_status fa_create_block_mask(const fa_mask_desc* mask, int64_t b_dims, int64_t h_dims,
                                          int64_t q_len, int64_t kv_len, int64_t bs_q,
                                          int64_t bs_kv, fa_block_mask* bm, void* workspace,
                                          size_t workspace_bytes, void* stream) {
  clear_error();
  fa_status s = bmk::geometry(b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, nullptr, nullptr, nullptr);
  if (s != FA_OK) return s;
  FA_REQUIRE(mask != nullptr && bm != nullptr, FA_SHAPE_MISMATCH, "create_block_mask: NULL argument");
  if ((s = check_mask_desc(*mask, q_len, kv_len)) != FA_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const MaskParams mp = to_mask_params(*mask);
  switch (mask_kind_of(*mask)) {
    case kMaskNoop: return bmk::build(MaskFn<kMaskNoop>{mp}, b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, bm, workspace, workspace_bytes, st);
    case kMaskCausalOnly: return bmk::build(MaskFn<kMaskCausalOnly>{mp}, b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, bm, workspace, workspace_bytes, st);
    case kMaskSlidingOnly: return bmk::build(MaskFn<kMaskSlidingOnly>{mp}, b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, bm, workspace, workspace_bytes, st);
    case kMaskDocCausal: return bmk::build(MaskFn<kMaskDocCausal>{mp}, b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, bm, workspace, workspace_bytes, st);
    default: return bmk::build(MaskFn<kMaskDynamic>{mp}, b_dims, h_dims, q_len, kv_len, bs_q, bs_kv, bm, workspace, workspace_bytes, st);
  }
}

extern "C" fa_status fa_transpose_block_mask(fa_block_mask* bm, void* workspace,
                                             size_t workspace_bytes, void* stream) {
  clear_error();
  FA_REQUIRE(bm != nullptr && bm->q_num_blocks && bm->q_indices && bm->full_q_num_blocks &&
                 bm->full_q_indices,
             FA_SHAPE_MISMATCH, "transpose: q-side arrays must be allocated");
  const size_t need = static_cast<size_t>(bm->b_dims * bm->h_dims * bm->rows * bm->cols);
  FA_REQUIRE(workspace != nullptr && workspace_bytes >= need, FA_SHAPE_MISMATCH,
             "transpose: workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* grid = static_cast<uint8_t*>(workspace);
  const int nrows = (int)(bm->b_dims * bm->h_dims * bm->rows);
  bmk::scatter_kinds_kernel<<<nrows, 128, 0, st>>>(nrows, (int)bm->cols, bm->kv_num_blocks,
                                              bm->kv_indices, bm->full_kv_num_blocks,
                                              bm->full_kv_indices, grid);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  const int bd = (int)bm->b_dims, hd = (int)bm->h_dims, R = (int)bm->rows, Cc = (int)bm->cols;
  const int ncols = bd * hd * Cc;
  bmk::compact_kernel<<<bmk::grid_for(ncols), 256, 0, st>>>(grid, ncols, R, Cc, R * Cc, 1, Cc,
                                                  bm->q_num_blocks, bm->q_indices,
                                                  bm->full_q_num_blocks, bm->full_q_indices);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

namespace {

// convert_block_mask's geometry checks and kernel; unmapped blocks set *d_err (stream-ordered)
fa_status convert_launch(const fa_block_mask* lg, const fa_page_table* pt, fa_block_mask* out, int* d_err,
                         cudaStream_t st) {
  FA_REQUIRE(lg && pt && out, FA_SHAPE_MISMATCH, "convert_block_mask: NULL argument");
  FA_REQUIRE(lg->bs_kv == pt->page_size, FA_BLOCK_MASK_MISMATCH,
             "convert_block_mask: kv block size " + std::to_string(lg->bs_kv) +
                 " must equal page size " + std::to_string(pt->page_size));
  FA_REQUIRE(lg->b_dims == 1 || lg->b_dims == pt->batches, FA_BLOCK_MASK_MISMATCH,
             "convert_block_mask: mask batch dim must be 1 or " + std::to_string(pt->batches));
  FA_REQUIRE(d_err != nullptr, FA_CUDA_ERROR, "convert_block_mask: no status word");
  out->b_dims = pt->batches;
  out->h_dims = lg->h_dims;
  out->rows = lg->rows;
  out->cols = pt->num_physical_pages;
  out->bs_q = lg->bs_q;
  out->bs_kv = lg->bs_kv;
  out->q_len = lg->q_len;
  out->kv_len = pt->num_physical_pages * pt->page_size;
  FA_CHECK_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), st));
  const int nlines = (int)(out->b_dims * out->h_dims * out->rows);
  bmk::convert_kernel<<<nlines, 128, 0, st>>>((int)pt->batches, (int)lg->h_dims, (int)lg->rows,
                                         (int)lg->cols, (int)lg->b_dims, lg->kv_num_blocks,
                                         lg->kv_indices, lg->full_kv_num_blocks, lg->full_kv_indices,
                                         pt->table, (int)pt->max_logical_pages, (int)out->cols,
                                         out->kv_num_blocks, out->kv_indices,
                                         out->full_kv_num_blocks, out->full_kv_indices, d_err);
  count_launch();
  FA_CHECK_CUDA(cudaGetLastError());
  return FA_OK;
}

}  // namespace

extern "C" fa_status fa_convert_block_mask(const fa_block_mask* lg, const fa_page_table* pt,
                                           fa_block_mask* out, void* stream) {
  clear_error();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* d_err = scheduler_counter(kSlotConvertErr, st);  // this (device, stream)'s status word
  fa_status s = convert_launch(lg, pt, out, d_err, st);
  if (s != FA_OK) return s;
  int h_err = 0;
  FA_CHECK_CUDA(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FA_CHECK_CUDA(cudaStreamSynchronize(st));
  FA_REQUIRE(h_err == 0, FA_UNMAPPED_BLOCK,
             "convert_block_mask: a logical block referenced by the mask has no physical page");
  return FA_OK;
}

extern "C" fa_status fa_convert_block_mask_async(const fa_block_mask* lg, const fa_page_table* pt,
                                                 fa_block_mask* out, int32_t* status, void* stream) {
  clear_error();
  FA_REQUIRE(status != nullptr, FA_SHAPE_MISMATCH, "convert_block_mask_async: NULL status word");
  return convert_launch(lg, pt, out, status, static_cast<cudaStream_t>(stream));
}
