// Throughput probe: packed FADD2/FMUL2 (add/mul.rn.f32x2, sm_100a) vs scalar
// FADD/FMUL, 8 independent chains per thread, full occupancy.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b){ u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b){ u64 d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float add1(float a, float b){ float d; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ float mul1(float a, float b){ float d; asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__global__ void kx2(u64* out, u64 s, int n){ u64 r[8]; for(int i=0;i<8;i++) r[i]=s+i+threadIdx.x;
  for(int it=0; it<n; ++it){
#pragma unroll
    for(int i=0;i<8;i++){ r[i]=add2(r[i],s); r[i]=mul2(r[i],s);} }
  u64 t=0; for(int i=0;i<8;i++) t^=r[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=t; }
__global__ void kx1(float* out, float s, int n){ float r[8]; for(int i=0;i<8;i++) r[i]=s+i+threadIdx.x;
  for(int it=0; it<n; ++it){
#pragma unroll
    for(int i=0;i<8;i++){ r[i]=add1(r[i],s); r[i]=mul1(r[i],s);} }
  float t=0; for(int i=0;i<8;i++) t+=r[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=t; }
int main(){ int blocks=148*8, th=256, n=4096; void* o; cudaMalloc(&o, (size_t)blocks*th*8);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for(int rep=0;rep<2;rep++){
  cudaEventRecord(a); kx1<<<blocks,th>>>((float*)o,1.0f,n); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  double ins=(double)blocks*th/32*n*16; printf("scalar: %.3f ms, %.1f warp-instr/clk/SM @1.965GHz, %.2f Tflop-ops/s\n", ms, ins/(ms*1e-3)/148/1.965e9, (double)blocks*th*n*16/(ms*1e-3)/1e12);
  cudaEventRecord(a); kx2<<<blocks,th>>>((u64*)o,0x3f8000003f800000ull,n); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("x2:     %.3f ms, %.1f warp-instr/clk/SM @1.965GHz, %.2f Tflop-ops/s\n", ms, ins/(ms*1e-3)/148/1.965e9, (double)blocks*th*n*32/(ms*1e-3)/1e12);}
  return 0; }
