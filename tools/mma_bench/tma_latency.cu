// Microbenchmark: latency and per-SM throughput of 32 KB TMA tile loads (two 64 x 128 bf16
// boxes, 128-byte swizzle: the Q / K / V / dO tiles of the attention kernels).
//   mode 0: one CTA, the same tile every time (L2 hit)        -> latency
//   mode 1: one CTA, a new tile every time (cold, from HBM)    -> latency
//   mode 2: 148 CTAs, new tiles, `depth` loads in flight each -> per-SM throughput
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_latency.cu -o tma_latency -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_2412_05496_b200/csrc/sm100_ptx.cuh"
using namespace fa;

constexpr int kBH = 64, kL = 8192, kD = 128, kTileBytes = 128 * kD * 2;

__global__ void bench(const __grid_constant__ CUtensorMap tm, int mode, int iters, int depth,
                      long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
  fence_barrier_init();
  const int ntiles = kBH * (kL / 128);
  long long total = 0;
  uint32_t phase[4] = {0, 0, 0, 0};
  auto issue = [&](int slot, int tile) {
    const int bh = tile / (kL / 128), rb = tile % (kL / 128);
    mbar_expect_tx(&bar[slot], kTileBytes);
    for (int ch = 0; ch < 2; ++ch)
      tma_load_3d(buf + slot * kTileBytes + ch * 16384, &tm, &bar[slot], ch * 64, rb * 128, bh);
  };
  int next = (blockIdx.x * 977) % ntiles;
  const long long t0 = clock64();
  if (mode < 2) {
    for (int it = 0; it < iters; ++it) {
      const int tile = mode == 0 ? 5 : (next = (next + 131) % ntiles);
      const long long a = clock64();
      issue(0, tile);
      mbar_wait(&bar[0], phase[0]);
      phase[0] ^= 1;
      total += clock64() - a;
    }
    out[blockIdx.x] = total / iters;
  } else {
    for (int s = 0; s < depth; ++s) issue(s, next = (next + 131) % ntiles);
    for (int it = 0; it < iters; ++it) {
      const int s = it % depth;
      mbar_wait(&bar[s], phase[s]);
      phase[s] ^= 1;
      if (it + depth < iters) issue(s, next = (next + 131) % ntiles);
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* x;
  cudaMalloc(&x, (size_t)kBH * kL * kD * 2);
  cudaMemset(x, 0, (size_t)kBH * kL * kD * 2);
  void* fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[3] = {kD, kL, kBH};
  cuuint64_t str[2] = {kD * 2, (cuuint64_t)kL * kD * 2};
  cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
  ((EncodeFn)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  long long* out;
  cudaMalloc(&out, 148 * sizeof(long long));
  const int smem = 4 * kTileBytes + 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<long long> h(148);
  for (int mode = 0; mode < 2; ++mode) {
    bench<<<1, 32, smem>>>(tm, mode, 64, 1, out);
    cudaMemcpy(h.data(), out, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %lld cycles per 32 KB load\n", mode, mode == 0 ? "L2 hit" : "cold", h[0]);
  }
  for (int depth = 1; depth <= 4; depth *= 2) {
    for (int grid : {1, 148}) {
      const int iters = 256;
      bench<<<grid, 32, smem>>>(tm, 2, iters, depth, out);
      cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("streaming grid %3d depth %d: %.1f B/clk per SM (%.0f cycles per load)\n", grid, depth,
             (double)iters * kTileBytes / mx, (double)mx / iters);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
