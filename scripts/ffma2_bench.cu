// Micro-benchmark: FFMA vs FFMA2 (fma.rn.f32x2) throughput on one B200. 148x8 CTAs of 256 threads,
// 8 independent chains per thread. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_bench ffma2_bench.cu
// Measured (round 1): FFMA 72.1 TFLOP/s, FFMA2 74.1 TFLOP/s -- same FP32 pipe rate, half the issue slots.
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;}
__global__ void k1(float* out, int iters){
  float a[8]; for(int i=0;i<8;++i) a[i]=threadIdx.x*0.001f+i;
  const float b=0.999f, c=0.001f;
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<8;++i) a[i]=__fmaf_rn(a[i],b,c);
  }
  float s=0; for(int i=0;i<8;++i) s+=a[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k2(float* out, int iters){
  u64 a[8]; for(int i=0;i<8;++i) { float x=threadIdx.x*0.001f+i; asm("mov.b64 %0, {%1,%1};" : "=l"(a[i]) : "f"(x)); }
  u64 b, c; { float x=0.999f, y=0.001f; asm("mov.b64 %0, {%1,%1};" : "=l"(b) : "f"(x)); asm("mov.b64 %0, {%1,%1};" : "=l"(c) : "f"(y)); }
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<8;++i) a[i]=fma2(a[i],b,c);
  }
  float s=0; for(int i=0;i<8;++i){ float lo,hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i])); s+=lo+hi; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  float* d; cudaMalloc(&d, 148*8*256*4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=20000;
  for(int rep=0;rep<2;++rep){
  k1<<<148*8,256>>>(d,iters); cudaEventRecord(e0); k1<<<148*8,256>>>(d,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms1; cudaEventElapsedTime(&ms1,e0,e1);
  k2<<<148*8,256>>>(d,iters); cudaEventRecord(e0); k2<<<148*8,256>>>(d,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms2; cudaEventElapsedTime(&ms2,e0,e1);
  double fl1 = 148.0*8*256*iters*8*2, fl2 = fl1*2;
  printf("FFMA : %.3f ms  %.1f TFLOP/s\nFFMA2: %.3f ms  %.1f TFLOP/s\n", ms1, fl1/ms1/1e9, ms2, fl2/ms2/1e9);
  }
  return 0;
}
