// Microbenchmark: tcgen05.mma kind::f16 (M=128, N=128, K=16 per instruction) issued by one
// thread, SS (A,B in smem) vs TS (A in TMEM), alone and with concurrent traffic from other
// warps: red.global.add.v4.f32 streams, tcgen05.ld streams, st.shared streams.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2412_05496_b200/csrc/sm100_ptx.cuh"
using namespace fa;

template <bool TS, int MODE, bool RND = false>
__global__ void __launch_bounds__(256, 1) bench(int iters, long long* out, float* gbuf) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) {
    uint32_t x = RND ? (i * 2654435761u + blockIdx.x * 97u) : 0x3f803f80u;
    if (RND) { x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15; x = (x & 0x807f807fu) | 0x3e003e00u; }
    reinterpret_cast<uint32_t*>(smem)[i] = x;
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
  if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(128, 128, 0, 0);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = make_sdesc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
        if (TS) {
          umma_ts(tm + 256, tm + kk * 8, bd, idesc, 1u);
        } else {
          const uint64_t ad = make_sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          umma_ss(tm + 256, ad, bd, idesc, 1u);
        }
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp >= 4 && MODE != 0) {
    // interference warps (TMEM lanes of warp%4)
    const uint32_t tq = tm + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    float* dst = gbuf + (blockIdx.x * 4 + (warp - 4)) * 32 * 128 + lane * 128;
    uint4* sdst = reinterpret_cast<uint4*>(smem + 65536) + (warp - 4) * 32 * 16 + lane * 16;
    while (!done) {
      if (MODE == 1) {
#pragma unroll
        for (int v = 0; v < 32; ++v) red_add_v4(dst + v * 4, 1.f, 1.f, 1.f, 1.f);
      } else if (MODE == 2) {
        uint32_t r[32];
        tmem_ld32(tq + 128, r);
        tmem_wait_ld();
        if (r[0] == 12345u) dst[0] = 1.f;
      } else if (MODE == 3) {
#pragma unroll
        for (int v = 0; v < 16; ++v) sdst[v] = make_uint4(v, v, v, v);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

// The backward's per-block MMA sequence back to back (no waits): MMA1 SS S^T=K Q^T ->[0,128),
// MMA2 SS dP^T=V dO^T ->[128,256), MMA3 TS dV+=P^T dO (MN B) ->[256,384), MMA4 TS dK+=dS^T Q
// ->[384,512), MMA5 SS dQ=dS K (MN A, MN B) ->[128,256). Nominal 5 x 512 = 2560 cycles.
template <int VARIANT>
__global__ void __launch_bounds__(128, 1) bwd_seq(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) {
    uint32_t x = i * 2654435761u; x ^= x >> 13; x = (x & 0x807f807fu) | 0x3e003e00u;
    reinterpret_cast<uint32_t*>(smem)[i] = x;
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t ss = make_idesc_bf16(128, 128, 0, 0), ts = make_idesc_bf16(128, 128, 0, 1),
                   mm = make_idesc_bf16(128, 128, 1, 1);
    const uint32_t K = smem_u32(smem), V = K + 32768, Q = K + 65536, dO = K + 98304, dS = K + 131072;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (VARIANT & 1) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        umma_ss(tm + 0, make_sdesc_sw128(K + off, 16, 1024), make_sdesc_sw128(Q + off, 16, 1024), ss, kk > 0);
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        umma_ss(tm + 128, make_sdesc_sw128(V + off, 16, 1024), make_sdesc_sw128(dO + off, 16, 1024), ss, kk > 0);
      }
      }
      if (VARIANT & 2) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_ts(tm + 256, tm + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8), make_sdesc_sw128(dO + kk * 2048, 16384, 1024), ts, 1);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_ts(tm + 384, tm + 128 + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8), make_sdesc_sw128(Q + kk * 2048, 16384, 1024), ts, 1);
      }
      if (VARIANT & 4) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_ss(tm + 128, make_sdesc_sw128(dS + kk * 2048, 16384, 1024), make_sdesc_sw128(K + kk * 2048, 16384, 1024), mm, kk > 0);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

template <int VARIANT>
void run_seq(const char* name, int iters, int gemms) {
  long long* d; cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(bwd_seq<VARIANT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 1024);
  bwd_seq<VARIANT><<<148, 128, 196608 + 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-34s: %7.1f cycles per iteration (nominal %d) (%s)\n", name, avg / iters, gemms * 512, cudaGetErrorString(e));
  cudaFree(d);
}

template <bool TS, int MODE, bool RND = false>
void run(const char* name, int iters, float* gbuf) {
  long long* d; cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(bench<TS, MODE, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  bench<TS, MODE, RND><<<148, 256, 98304 + 1024>>>(iters, d, gbuf);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-28s: %7.1f cycles per K=16 MMA (64 = full rate) (%s)\n", name, avg / (8.0 * iters), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  float* gbuf; cudaMalloc(&gbuf, 148 * 4 * 32 * 128 * sizeof(float));
  run_seq<7>("bwd MMA1..5 sequence", 500, 5);
  run_seq<1>("bwd MMA1+MMA2 (SS K-major)", 500, 2);
  run_seq<2>("bwd MMA3+MMA4 (TS, MN-major B)", 500, 2);
  run_seq<4>("bwd MMA5 (SS, MN-major A and B)", 500, 1);
  run<false, 0>("SS alone", 4000, gbuf);
  run<false, 0, true>("SS alone random data", 4000, gbuf);
  run<true, 0, true>("TS alone random data", 4000, gbuf);
  run<true, 0>("TS alone", 4000, gbuf);
  run<false, 1>("SS + red.global stream", 4000, gbuf);
  run<true, 1>("TS + red.global stream", 4000, gbuf);
  run<false, 2>("SS + tcgen05.ld stream", 4000, gbuf);
  run<true, 2>("TS + tcgen05.ld stream", 4000, gbuf);
  run<false, 3>("SS + st.shared stream", 4000, gbuf);
  run<true, 3>("TS + st.shared stream", 4000, gbuf);
  return 0;
}
