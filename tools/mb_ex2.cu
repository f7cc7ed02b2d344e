#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
__device__ __forceinline__ unsigned ex2bf2(unsigned x){unsigned y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y;}
__device__ __forceinline__ unsigned ex2h2(unsigned x){unsigned y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y;}
__device__ __forceinline__ float ex2f(float x){float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;}
template<int MODE>
__global__ void k(unsigned* out, int iters, unsigned seed){
  unsigned r[8]; for(int i=0;i<8;++i) r[i]=seed*(threadIdx.x+i);
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<8;++i){
      if(MODE==0) r[i]=__float_as_uint(ex2f(__uint_as_float(r[i])));
      else if(MODE==1) r[i]=ex2bf2(r[i]);
      else r[i]=ex2h2(r[i]);
    }
  }
  unsigned s=0; for(int i=0;i<8;++i) s^=r[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  unsigned* d; cudaMalloc(&d, 148*8*1024*4);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters=4096;
  for(int mode=0;mode<3;++mode){
    for(int rep=0;rep<2;++rep){
    cudaEventRecord(a);
    if(mode==0) k<0><<<148*4,512>>>(d,iters,1); else if(mode==1) k<1><<<148*4,512>>>(d,iters,1); else k<2><<<148*4,512>>>(d,iters,1);
    cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b);
    double ops=148.0*4*512*iters*8; // instructions (lanes)
    if(rep) printf("mode %d: %.3f ms, %.1f Ginstr-lanes/s, per SM per clk(1.9GHz) %.2f lane-instr\n", mode, ms, ops/ms/1e6, ops/(ms*1e-3)/148/1.9e9);
    }
  }
  return 0;
}
