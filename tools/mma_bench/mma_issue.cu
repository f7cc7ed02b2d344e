// Microbenchmark: tcgen05.mma issue cost. N=64 MMAs (32 cycles of tensor work each) issued
//   mode 0: by lane 0 inside `if (lane == 0)` (per-MMA waterfall: ELECT/R2UR.BROADCAST/BRA)
//   mode 1: by the whole warp, stage index from a warp-uniform loop, elect.sync inside the asm
// with descriptors recomputed per GEMM from a stage index (as the attention kernels do).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_issue.cu -o mma_issue
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2412_05496_b200/csrc/sm100_ptx.cuh"
using namespace fa;

__device__ __forceinline__ void umma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  constexpr uint32_t idesc = make_idesc_bf16(128, 64, 0, 0);
  if (MODE == 0 && threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int st = it & 1;
      const uint64_t a0 = make_sdesc_sw128(opaque_u32(smem_u32(smem)), 16, 1024);
      const uint64_t b0 = make_sdesc_sw128(opaque_u32(smem_u32(smem + 32768 + st * 32768)), 16, 1024);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
        umma_ss(tm + (st * 64), a0 + off, b0 + off, idesc, kk > 0);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  } else if (MODE == 1 && warp == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int st = it & 1;
      const uint64_t a0 = make_sdesc_sw128(smem_u32(smem), 16, 1024);
      const uint64_t b0 = make_sdesc_sw128(smem_u32(smem + 32768 + st * 32768), 16, 1024);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
        umma_ss_elect(tm + (st * 64), a0 + off, b0 + off, idesc, kk > 0);
      }
    }
    umma_commit_elect(&bar);
    mbar_wait(&bar, 0);
    if (lane == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

template <int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = bench<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int iters = 2000;
  k<<<148, 128, 131072>>>(10, d);
  k<<<148, 128, 131072>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-44s %.1f cycles / MMA (128x64x16, 32 cycles of work)  [%s]\n", name, s / 148 / iters / 8,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("lane-0 branch (waterfall per MMA)");
  run<1>("whole warp + elect.sync in the asm");
  return 0;
}
