// Microbenchmark: mbarrier wake-up latency (cycles from arrive to the waiter passing its wait)
// for three wait styles: try_wait with a suspend-time hint, try_wait without a hint, and a
// test_wait spin. Warp 0 lane 0 arrives; warp 1 lane 0 waits. 64 rounds, averaged.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mbar_latency.cu -o mbar_latency
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2412_05496_b200/csrc/sm100_ptx.cuh"
using namespace fa;

__device__ __forceinline__ bool try_wait_nohint(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

template <int STYLE>
__global__ void bench(long long* out) {
  __shared__ uint64_t bar[2];
  __shared__ volatile long long t_arrive[64];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
  __syncthreads();
  long long acc = 0;
  for (int r = 0; r < 64; ++r) {
    if (warp == 0 && lane == 0) {
      // wait for the waiter to be parked (ack barrier), then spin a while and arrive
      if (r > 0) while (!test_wait(&bar[1], (r - 1) & 1)) {}
      const long long t0 = clock64();
      while (clock64() - t0 < 4000) {}
      t_arrive[r] = clock64();
      mbar_arrive(&bar[0]);
    } else if (warp == 1 && lane == 0) {
      if (STYLE == 0) mbar_wait(&bar[0], r & 1);
      else if (STYLE == 1) { while (!try_wait_nohint(&bar[0], r & 1)) {} }
      else { while (!test_wait(&bar[0], r & 1)) {} }
      const long long t1 = clock64();
      acc += t1 - t_arrive[r];
      mbar_arrive(&bar[1]);
    }
  }
  if (warp == 1 && lane == 0) out[blockIdx.x] = acc / 64;
}

template <int STYLE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  bench<STYLE><<<148, 64>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-36s %.0f cycles arrive->wake  [%s]\n", name, s / 148, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("try_wait + suspend hint (mbar_wait)");
  run<1>("try_wait, no hint");
  run<2>("test_wait spin");
  return 0;
}
