// Which pipe do the min/compare/select ops occupy next to packed FFMA2?  Each kernel runs 8
// independent FFMA2 chains per iteration plus an extra op mix; the slowdown vs the pure FFMA2 loop
// tells whether the extra ops steal FMA-pipe cycles (design data for DESIGN.md §4.2).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix pipe_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;":"=l"(r):"l"(a),"l"(b),"l"(c)); return r;}
__device__ __forceinline__ u64 pk(float a, float b){u64 r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ void upk(u64 v, float& a, float& b){asm("mov.b64 {%0,%1}, %2;":"=f"(a),"=f"(b):"l"(v));}
__device__ __forceinline__ float fmin3(float a, float b, float c){float r; asm volatile("min.f32 %0, %1, %2, %3;":"=f"(r):"f"(a),"f"(b),"f"(c)); return r;}
__device__ __forceinline__ float fmin2(float a, float b){float r; asm volatile("min.f32 %0, %1, %2;":"=f"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ int imin2(int a, int b){int r; asm volatile("min.s32 %0, %1, %2;":"=r"(r):"r"(a),"r"(b)); return r;}
__device__ __forceinline__ int iadd3(int a, int b, int c){int r; asm volatile("add.s32 %0, %1, %2; add.s32 %0, %0, %3;":"=r"(r):"r"(a),"r"(b),"r"(c)); return r;}

#define ITERS 2048
template<int MODE, int NX>
__global__ void k(float* out, float b, float c){
  u64 a[8]; u64 bb=pk(b,b), cc=pk(c,c);
  float m[8]; int im[8]; unsigned um[8];
  #pragma unroll
  for(int i=0;i<8;i++){ a[i]=pk(threadIdx.x*1e-3f+i, i+0.5f); m[i]=1e30f+i; im[i]=0x7f000000+i; um[i]=0x7f000000u+i; }
  for(int it=0;it<ITERS;it++){
    #pragma unroll
    for(int i=0;i<8;i++) a[i]=fma2(a[i],bb,cc);
    #pragma unroll
    for(int i=0;i<NX;i++){
      float x0,x1; upk(a[i],x0,x1);
      if(MODE==1) m[i]=fmin3(m[i],x0,x1);
      if(MODE==2) m[i]=fmin2(m[i],x0);
      if(MODE==3) im[i]=imin2(im[i],__float_as_int(x0));
      if(MODE==4) im[i]=imin2(imin2(im[i],__float_as_int(x0)),__float_as_int(x1));
      if(MODE==5) { bool p=x0<m[i]; m[i]=p?x0:m[i]; im[i]=p?it:im[i]; }
      if(MODE==6) im[i]=iadd3(im[i],__float_as_int(x0),__float_as_int(x1));
    }
  }
  float s=0;
  #pragma unroll
  for(int i=0;i<8;i++){ float x0,x1; upk(a[i],x0,x1); s+=x0+x1+m[i]+im[i]+um[i]; }
  if(s==1234.5f) out[0]=s;
}
template<int MODE,int NX> void run(const char* name, int sms, int clk, float* out){
  int threads=256, blocks=sms*8;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE,NX><<<blocks,threads>>>(out,0.999f,1e-3f);
  cudaEventRecord(e0); k<MODE,NX><<<blocks,threads>>>(out,0.999f,1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  double lane=(double)threads*blocks*16.0*ITERS;
  double cyc_per_iter_per_warp = (ms*1e-3*clk*1e3) / ((double)threads*blocks/32/ (sms*4)) / ITERS;
  printf("%-34s x%d : %.3f ms  %.1f lane-FMA/clk/SM  %.2f clk/iter/SMSP-warp-slot (16 = pure FFMA2)\n", name, NX, ms, lane/(ms*1e-3)/(sms*clk*1e3), cyc_per_iter_per_warp);
}
int main(){
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out,4);
  for(int p=0;p<2;p++){
  run<0,0>("pure FFMA2", sms, clk, out);
  run<1,2>("FMNMX3 (3-input fp min)", sms, clk, out);
  run<1,4>("FMNMX3 (3-input fp min)", sms, clk, out);
  run<1,8>("FMNMX3 (3-input fp min)", sms, clk, out);
  run<2,4>("FMNMX (2-input fp min)", sms, clk, out);
  run<2,8>("FMNMX (2-input fp min)", sms, clk, out);
  run<3,4>("IMNMX (int min on float bits)", sms, clk, out);
  run<3,8>("IMNMX (int min on float bits)", sms, clk, out);
  run<4,4>("2x IMNMX", sms, clk, out);
  run<4,8>("2x IMNMX", sms, clk, out);
  run<5,4>("FSETP+FSEL+SEL", sms, clk, out);
  run<6,4>("IADD (x2)", sms, clk, out);
  run<6,8>("IADD (x2)", sms, clk, out);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
