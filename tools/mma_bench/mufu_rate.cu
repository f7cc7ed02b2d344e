// Microbenchmark: per-SMSP issue cost of ex2.approx (MUFU.EX2), the bf16 pack
// (F2FP.BF16.F32.PACK_AB) and FFMA2 in a softmax-like inner loop. 1 warp per SMSP (4 warps)
// or 2 warps per SMSP (8 warps); each warp runs 32 independent chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mufu_rate.cu -o mufu_rate
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned pack(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<unsigned*>(&v);
}

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = -0.001f * (threadIdx.x + i);
  unsigned acc = 0;
  float2 s = make_float2(0.f, 0.f);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      if (MODE == 0) {  // ex2 only
        v[i] = ex2(v[i]);
        v[i + 1] = ex2(v[i + 1]);
      } else if (MODE == 1) {  // pack only
        acc ^= pack(v[i], v[i + 1]);
        v[i] += 1e-7f;
      } else {  // softmax body: ffma2, 2 ex2, fadd2, pack
        const float2 x = __ffma2_rn(make_float2(v[i], v[i + 1]), make_float2(1.f, 1.f), make_float2(-0.5f, -0.5f));
        const float2 p = make_float2(ex2(x.x), ex2(x.y));
        s = __fadd2_rn(s, p);
        acc ^= pack(p.x, p.y);
        v[i] = p.x * 0.5f;
        v[i + 1] = p.y * 0.5f;
      }
    }
  }
  const long long t1 = clock64();
  float r = s.x + s.y + (float)acc;
#pragma unroll
  for (int i = 0; i < 32; ++i) r += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1024);
  const int iters = 1000;
  const char* names[3] = {"ex2", "pack", "softmax body (ffma2 + 2 ex2 + fadd2 + pack)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {4, 8, 16}) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<1, warps * 32>>>(out, cyc, iters);
        if (mode == 1) k<1><<<1, warps * 32>>>(out, cyc, iters);
        if (mode == 2) k<2><<<1, warps * 32>>>(out, cyc, iters);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      }
      // per SMSP: warps/4 warps, each 16 pair-iterations x iters
      const double per_pair = (double)h / (iters * 16.0 * (warps / 4));
      printf("%-45s warps %2d: %.2f cycles per pair-iteration per SMSP (= %.2f per warp-instr of ex2 pair/2)\n",
             names[mode], warps, per_pair, per_pair / 2);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
