// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128 N=128 K=16) for the operand
// layouts the backward kernel uses, one issuing thread per CTA, one CTA per SM:
//   0 SS  A K-major,  B K-major     (S^T = K Q^T, dP^T = V dO^T)
//   1 TS  A TMEM,     B MN-major    (dV += P^T dO, dK += dS^T Q)
//   2 SS  A MN-major, B MN-major    (dQ^T = K^T dS^T)
//   3 SS  A K-major,  B MN-major
//   4 the backward's per-block sequence S, dP, dK, dQ, dV (40 instructions)
// optionally with 8 warps streaming st.shared (128-bit) concurrently (smem write pressure).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_modes.cu -o mma_modes
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2412_05496_b200/csrc/sm100_ptx.cuh"
using namespace fa;

template <int MODE, int STS>
__global__ void __launch_bounds__(320, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) {
    uint32_t x = i * 2654435761u + blockIdx.x * 97u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    reinterpret_cast<uint32_t*>(smem)[i] = (x & 0x807f807fu) | 0x3e003e00u;
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
  if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t kk_idesc = make_idesc_bf16(128, 128, 0, 0);
    const uint32_t kn_idesc = make_idesc_bf16(128, 128, 0, 1);
    const uint32_t nn_idesc = make_idesc_bf16(128, 128, 1, 1);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768), c = smem_u32(smem + 65536);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE == 0 || MODE == 4) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tm + 0, make_sdesc_sw128(a + off, 16, 1024), make_sdesc_sw128(b + off, 16, 1024), kk_idesc, kk > 0);
        }
      }
      if (MODE == 4) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tm + 128, make_sdesc_sw128(c + off, 16, 1024), make_sdesc_sw128(b + off, 16, 1024), kk_idesc, kk > 0);
        }
      }
      if (MODE == 1 || MODE == 4) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tm + 256, tm + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8), make_sdesc_sw128(b + kk * 2048, 16384, 1024),
                  kn_idesc, 1u);
      }
      if (MODE == 4) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tm + 384, tm + 128 + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8), make_sdesc_sw128(c + kk * 2048, 16384, 1024),
                  kn_idesc, 1u);
      }
      if (MODE == 2 || MODE == 4) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tm + 128, make_sdesc_sw128(a + kk * 2048, 16384, 1024), make_sdesc_sw128(c + kk * 2048, 16384, 1024),
                  nn_idesc, kk > 0);
      }
      if (MODE == 3) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tm + 128, make_sdesc_sw128(a + off, 16, 1024), make_sdesc_sw128(c + kk * 2048, 16384, 1024),
                  kn_idesc, kk > 0);
        }
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (STS == 1 && warp >= 2) {
    uint4* dst = reinterpret_cast<uint4*>(smem + 131072) + (warp - 2) * 32 * 16 + lane;
    uint32_t x = lane;
    while (!done) {
#pragma unroll
      for (int v = 0; v < 16; ++v) dst[v * 32] = make_uint4(x, x + 1, x + 2, x + 3);
      ++x;
    }
  } else if (STS == 2 && warp >= 2) {  // tcgen05.ld streams of 32 columns (S-like reads)
    const uint32_t tq = tm + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    long long n = 0, t0 = clock64();
    while (!done) {
      uint32_t r[32];
      tmem_ld32(tq + ((warp >> 2) & 1) * 64, r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i];
      ++n;
    }
    if (lane == 0 && warp == 2) out[148 + blockIdx.x] = (clock64() - t0) / (n > 0 ? n : 1);
    if (acc == 12345) out[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

template <int MODE, int STS>
void run(const char* name, int per_iter) {
  long long* d;
  cudaMalloc(&d, 296 * sizeof(long long));
  auto k = bench<MODE, STS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
  const int iters = 2000;
  k<<<148, 320, 196608>>>(10, d);
  k<<<148, 320, 196608>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (STS == 2) printf("   (tcgen05.ld 32x32b.x32 per warp: %lld cycles each, 8 warps)\n", h[148]);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-44s mode=%d  %.1f cycles / MMA (K=16)   [%s]\n", name, STS, s / 148 / iters / per_iter,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 0>("SS K/K (S, dP)", 8);
  run<1, 0>("TS B MN-major (dV, dK)", 8);
  run<2, 0>("SS MN/MN (dQ^T)", 8);
  run<3, 0>("SS K/MN", 8);
  run<4, 0>("bwd block sequence S dP dV dK dQ", 40);
  run<0, 2>("SS K/K (S, dP) + tmem ld", 8);
  run<1, 2>("TS B MN-major (dV, dK) + tmem ld", 8);
  run<2, 2>("SS MN/MN (dQ^T) + tmem ld", 8);
  run<4, 2>("bwd block sequence + tmem ld", 40);
  return 0;
}
