// Microbenchmark: FP32 pipe throughput on sm_100a — scalar FFMA vs packed FFMA2 (f32x2),
// plus an ALU-pipe mix (FMNMX3), to decide whether packed FP32 doubles the FMA-pipe rate
// or only saves issue slots (SURVEY.md §8.d.3 "FFMA vs FFMA2 microbenchmark").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_pipes fp32_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;":"=l"(r):"l"(a),"l"(b),"l"(c)); return r;}
__device__ __forceinline__ u64 pk(float a, float b){u64 r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ float lo(u64 v){float a,b; asm("mov.b64 {%0,%1}, %2;":"=f"(a),"=f"(b):"l"(v)); return a+b;}
__device__ __forceinline__ float fmin3(float a, float b, float c){float r; asm volatile("min.f32 %0, %1, %2, %3;":"=f"(r):"f"(a),"f"(b),"f"(c)); return r;}

#define ITERS 4096
// 16 independent scalar FFMA chains per thread: 16*ITERS FFMA
__global__ void k_ffma(float* out, float b, float c){
  float a[16];
  #pragma unroll
  for(int i=0;i<16;i++) a[i]=threadIdx.x*1e-3f+i;
  for(int it=0;it<ITERS;it++){
    #pragma unroll
    for(int i=0;i<16;i++) a[i]=__fmaf_rn(a[i],b,c);
  }
  float s=0;
  #pragma unroll
  for(int i=0;i<16;i++) s+=a[i];
  if(s==1234.5f) out[0]=s;
}
// 8 independent packed FFMA2 chains: 16*ITERS lane-FMAs, 8*ITERS instructions
__global__ void k_ffma2(float* out, float b, float c){
  u64 a[8]; u64 bb=pk(b,b), cc=pk(c,c);
  #pragma unroll
  for(int i=0;i<8;i++) a[i]=pk(threadIdx.x*1e-3f+i, i+0.5f);
  for(int it=0;it<ITERS;it++){
    #pragma unroll
    for(int i=0;i<8;i++) a[i]=fma2(a[i],bb,cc);
  }
  float s=0;
  #pragma unroll
  for(int i=0;i<8;i++) s+=lo(a[i]);
  if(s==1234.5f) out[0]=s;
}
// 8 packed FFMA2 chains + 4 FMNMX3 per iteration (ALU pipe co-issue test)
__global__ void k_ffma2_alu(float* out, float b, float c){
  u64 a[8]; u64 bb=pk(b,b), cc=pk(c,c);
  float m[4];
  #pragma unroll
  for(int i=0;i<8;i++) a[i]=pk(threadIdx.x*1e-3f+i, i+0.5f);
  #pragma unroll
  for(int i=0;i<4;i++) m[i]=1e30f+i;
  for(int it=0;it<ITERS;it++){
    #pragma unroll
    for(int i=0;i<8;i++) a[i]=fma2(a[i],bb,cc);
    #pragma unroll
    for(int i=0;i<4;i++) { float x0,x1; asm("mov.b64 {%0,%1}, %2;":"=f"(x0),"=f"(x1):"l"(a[2*i])); m[i]=fmin3(m[i],x0,x1); }
  }
  float s=0;
  #pragma unroll
  for(int i=0;i<8;i++) s+=lo(a[i]);
  #pragma unroll
  for(int i=0;i<4;i++) s+=m[i];
  if(s==1234.5f) out[0]=s;
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads=256, blocks=sms*8;
  double lanes=(double)threads*blocks;
  for(int rep=0;rep<2;rep++){
    float ms;
    cudaEventRecord(e0); k_ffma<<<blocks,threads>>>(out,0.999f,1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    double ffma=lanes*16.0*ITERS/(ms*1e-3);
    printf("scalar FFMA : %.3f ms  %.2f T lane-FMA/s  (%.1f lane-FMA/clk/SM at %d MHz max)\n", ms, ffma/1e12, ffma/(sms*(clk*1e3)), clk/1000);
    cudaEventRecord(e0); k_ffma2<<<blocks,threads>>>(out,0.999f,1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    double f2=lanes*16.0*ITERS/(ms*1e-3);
    printf("packed FFMA2: %.3f ms  %.2f T lane-FMA/s  (%.1f lane-FMA/clk/SM)\n", ms, f2/1e12, f2/(sms*(clk*1e3)));
    cudaEventRecord(e0); k_ffma2_alu<<<blocks,threads>>>(out,0.999f,1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    double f3=lanes*16.0*ITERS/(ms*1e-3);
    printf("FFMA2+FMNMX3: %.3f ms  %.2f T lane-FMA/s  (%.1f lane-FMA/clk/SM)\n", ms, f3/1e12, f3/(sms*(clk*1e3)));
  }
  printf("sms=%d err=%s\n", sms, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
