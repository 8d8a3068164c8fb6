// Microbenchmark of candidate NN inner loops on sm_100a (design data for DESIGN.md §4.2).
// Each variant: every thread holds R queries in registers, sweeps T targets staged in smem
// (float4 x,y,z,pad; broadcast reads), computes d = (x-y)^2 with the fixed op order and keeps a
// running min (+ argmin bookkeeping per variant).  Reports directed pairs/s and the FMA-pipe
// fraction (6 lane-ops per pair / (SMs*128*clk)).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nn_loops nn_loops.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b){u64 r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ void upk(u64 v, float& a, float& b){asm("mov.b64 {%0,%1}, %2;":"=f"(a),"=f"(b):"l"(v));}
__device__ __forceinline__ u64 sub2(u64 a, u64 b){u64 r; asm("sub.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 mul2(u64 a, u64 b){u64 r; asm("mul.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;":"=l"(r):"l"(a),"l"(b),"l"(c)); return r;}
__device__ __forceinline__ float min3(float a, float b, float c){float r; asm("min.f32 %0, %1, %2, %3;":"=f"(r):"f"(a),"f"(b),"f"(c)); return r;}

#define T 4096   // targets in smem (64 KB)

// VARIANT 0: scalar ops, per-pair argmin (FSETP/FSEL/SEL per pair)
template<int R>
__global__ void __launch_bounds__(128) v_scalar_pair(const float4* __restrict__ tg, const float4* __restrict__ q, int reps, float* od, int* oi){
  extern __shared__ float4 sm[];
  for(int i=threadIdx.x;i<T;i+=blockDim.x) sm[i]=tg[i];
  __syncthreads();
  float qx[R],qy[R],qz[R],best[R]; int bi[R];
  int base=(blockIdx.x*blockDim.x+threadIdx.x)*R;
  #pragma unroll
  for(int r=0;r<R;r++){float4 p=q[base+r]; qx[r]=p.x;qy[r]=p.y;qz[r]=p.z;best[r]=INFINITY;bi[r]=-1;}
  for(int rep=0;rep<reps;rep++)
  for(int j=0;j<T;j++){ float4 t=sm[j];
    #pragma unroll
    for(int r=0;r<R;r++){ float dx=__fsub_rn(qx[r],t.x),dy=__fsub_rn(qy[r],t.y),dz=__fsub_rn(qz[r],t.z);
      float s=__fmul_rn(dx,dx); s=__fmaf_rn(dy,dy,s); s=__fmaf_rn(dz,dz,s);
      bool p=s<best[r]; best[r]=p?s:best[r]; bi[r]=p?j:bi[r]; } }
  #pragma unroll
  for(int r=0;r<R;r++){od[base+r]=best[r]; oi[base+r]=bi[r];}
}

// VARIANT 1: packed f32x2, chunk-of-C argmin: m = min(chunk ∪ best) via FMNMX3, FSETP + SEL per chunk
template<int R, int C>
__global__ void __launch_bounds__(128) v_packed_chunk(const float4* __restrict__ tg, const float4* __restrict__ q, int reps, float* od, int* oi){
  extern __shared__ float4 sm[];
  for(int i=threadIdx.x;i<T;i+=blockDim.x) sm[i]=tg[i];
  __syncthreads();
  u64 qx[R/2],qy[R/2],qz[R/2]; float best[R]; int bi[R];
  int base=(blockIdx.x*blockDim.x+threadIdx.x)*R;
  #pragma unroll
  for(int r=0;r<R/2;r++){float4 a=q[base+2*r],b=q[base+2*r+1]; qx[r]=pk(a.x,b.x);qy[r]=pk(a.y,b.y);qz[r]=pk(a.z,b.z);}
  #pragma unroll
  for(int r=0;r<R;r++){best[r]=INFINITY;bi[r]=-1;}
  for(int rep=0;rep<reps;rep++)
  for(int j=0;j<T;j+=C){
    float4 t[C];
    #pragma unroll
    for(int k=0;k<C;k++) t[k]=sm[j+k];
    #pragma unroll
    for(int r=0;r<R/2;r++){
      float dl[C],dh[C];
      #pragma unroll
      for(int k=0;k<C;k++){ u64 dx=sub2(qx[r],pk(t[k].x,t[k].x)),dy=sub2(qy[r],pk(t[k].y,t[k].y)),dz=sub2(qz[r],pk(t[k].z,t[k].z));
        u64 s=mul2(dx,dx); s=fma2(dy,dy,s); s=fma2(dz,dz,s); upk(s,dl[k],dh[k]); }
      float ml,mh;
      if(C==4){ ml=min3(min3(dl[0],dl[1],dl[2]),dl[3],best[2*r]); mh=min3(min3(dh[0],dh[1],dh[2]),dh[3],best[2*r+1]); }
      else { ml=min3(min3(min3(dl[0],dl[1],dl[2]),dl[3],dl[4]),min3(dl[5],dl[6],dl[7]),best[2*r]);
             mh=min3(min3(min3(dh[0],dh[1],dh[2]),dh[3],dh[4]),min3(dh[5],dh[6],dh[7]),best[2*r+1]); }
      bool pl=ml<best[2*r], ph=mh<best[2*r+1];
      bi[2*r]=pl?j:bi[2*r]; bi[2*r+1]=ph?j:bi[2*r+1];
      best[2*r]=ml; best[2*r+1]=mh;
    }
  }
  #pragma unroll
  for(int r=0;r<R;r++){od[base+r]=best[r]; oi[base+r]=bi[r];}
}

// VARIANT 2: packed f32x2, value-only running min via FMNMX3 folding; block-level change detect
// every K targets (FSETP+SEL per K), index recovered later by re-scanning the winning block.
template<int R, int K>
__global__ void __launch_bounds__(128) v_packed_block(const float4* __restrict__ tg, const float4* __restrict__ q, int reps, float* od, int* oi){
  extern __shared__ float4 sm[];
  for(int i=threadIdx.x;i<T;i+=blockDim.x) sm[i]=tg[i];
  __syncthreads();
  u64 qx[R/2],qy[R/2],qz[R/2]; float best[R]; int bi[R];
  int base=(blockIdx.x*blockDim.x+threadIdx.x)*R;
  #pragma unroll
  for(int r=0;r<R/2;r++){float4 a=q[base+2*r],b=q[base+2*r+1]; qx[r]=pk(a.x,b.x);qy[r]=pk(a.y,b.y);qz[r]=pk(a.z,b.z);}
  #pragma unroll
  for(int r=0;r<R;r++){best[r]=INFINITY;bi[r]=-1;}
  for(int rep=0;rep<reps;rep++)
  for(int j0=0;j0<T;j0+=K){
    float old[R];
    #pragma unroll
    for(int r=0;r<R;r++) old[r]=best[r];
    #pragma unroll 2
    for(int j=j0;j<j0+K;j+=2){
      float4 t0=sm[j], t1=sm[j+1];
      #pragma unroll
      for(int r=0;r<R/2;r++){
        u64 dx=sub2(qx[r],pk(t0.x,t0.x)),dy=sub2(qy[r],pk(t0.y,t0.y)),dz=sub2(qz[r],pk(t0.z,t0.z));
        u64 s=mul2(dx,dx); s=fma2(dy,dy,s); s=fma2(dz,dz,s);
        u64 ex=sub2(qx[r],pk(t1.x,t1.x)),ey=sub2(qy[r],pk(t1.y,t1.y)),ez=sub2(qz[r],pk(t1.z,t1.z));
        u64 u=mul2(ex,ex); u=fma2(ey,ey,u); u=fma2(ez,ez,u);
        float sl,sh,ul,uh; upk(s,sl,sh); upk(u,ul,uh);
        best[2*r]=min3(best[2*r],sl,ul); best[2*r+1]=min3(best[2*r+1],sh,uh);
      }
    }
    #pragma unroll
    for(int r=0;r<R;r++) bi[r]=(best[r]<old[r])?j0:bi[r];
  }
  #pragma unroll
  for(int r=0;r<R;r++){od[base+r]=best[r]; oi[base+r]=bi[r];}
}

// VARIANT 3: scalar ops, value-only FMNMX3 folding (no packed), block change detect
template<int R, int K>
__global__ void __launch_bounds__(128) v_scalar_block(const float4* __restrict__ tg, const float4* __restrict__ q, int reps, float* od, int* oi){
  extern __shared__ float4 sm[];
  for(int i=threadIdx.x;i<T;i+=blockDim.x) sm[i]=tg[i];
  __syncthreads();
  float qx[R],qy[R],qz[R],best[R]; int bi[R];
  int base=(blockIdx.x*blockDim.x+threadIdx.x)*R;
  #pragma unroll
  for(int r=0;r<R;r++){float4 p=q[base+r]; qx[r]=p.x;qy[r]=p.y;qz[r]=p.z;best[r]=INFINITY;bi[r]=-1;}
  for(int rep=0;rep<reps;rep++)
  for(int j0=0;j0<T;j0+=K){
    float old[R];
    #pragma unroll
    for(int r=0;r<R;r++) old[r]=best[r];
    #pragma unroll 2
    for(int j=j0;j<j0+K;j+=2){ float4 t0=sm[j], t1=sm[j+1];
      #pragma unroll
      for(int r=0;r<R;r++){
        float dx=__fsub_rn(qx[r],t0.x),dy=__fsub_rn(qy[r],t0.y),dz=__fsub_rn(qz[r],t0.z);
        float s=__fmul_rn(dx,dx); s=__fmaf_rn(dy,dy,s); s=__fmaf_rn(dz,dz,s);
        float ex=__fsub_rn(qx[r],t1.x),ey=__fsub_rn(qy[r],t1.y),ez=__fsub_rn(qz[r],t1.z);
        float u=__fmul_rn(ex,ex); u=__fmaf_rn(ey,ey,u); u=__fmaf_rn(ez,ez,u);
        best[r]=min3(best[r],s,u);
      } }
    #pragma unroll
    for(int r=0;r<R;r++) bi[r]=(best[r]<old[r])?j0:bi[r];
  }
  #pragma unroll
  for(int r=0;r<R;r++){od[base+r]=best[r]; oi[base+r]=bi[r];}
}

// VARIANT 4: packed, distances only (no min at all) — FMA-only ceiling (sum to keep live)
template<int R>
__global__ void __launch_bounds__(128) v_packed_nomin(const float4* __restrict__ tg, const float4* __restrict__ q, int reps, float* od, int* oi){
  extern __shared__ float4 sm[];
  for(int i=threadIdx.x;i<T;i+=blockDim.x) sm[i]=tg[i];
  __syncthreads();
  u64 qx[R/2],qy[R/2],qz[R/2]; u64 acc[R/2];
  int base=(blockIdx.x*blockDim.x+threadIdx.x)*R;
  #pragma unroll
  for(int r=0;r<R/2;r++){float4 a=q[base+2*r],b=q[base+2*r+1]; qx[r]=pk(a.x,b.x);qy[r]=pk(a.y,b.y);qz[r]=pk(a.z,b.z); acc[r]=0;}
  for(int rep=0;rep<reps;rep++)
  for(int j=0;j<T;j++){ float4 t=sm[j];
    #pragma unroll
    for(int r=0;r<R/2;r++){ u64 dx=sub2(qx[r],pk(t.x,t.x)),dy=sub2(qy[r],pk(t.y,t.y)),dz=sub2(qz[r],pk(t.z,t.z));
      u64 s=fma2(dx,dx,acc[r]); s=fma2(dy,dy,s); acc[r]=fma2(dz,dz,s);} }
  #pragma unroll
  for(int r=0;r<R/2;r++){float a,b; upk(acc[r],a,b); od[base+2*r]=a; od[base+2*r+1]=b; oi[base+2*r]=0; oi[base+2*r+1]=0;}
}

typedef void(*KFn)(const float4*,const float4*,int,float*,int*);
int sms, clk;
float4 *dT,*dQ; float* od; int* oi;
void run(const char* name, KFn f, int R, int blocksPerSM){
  int threads=128; int blocks=sms*blocksPerSM; int reps=4;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, T*16);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f<<<blocks,threads,T*16>>>(dT,dQ,1,od,oi);
  cudaEventRecord(e0); f<<<blocks,threads,T*16>>>(dT,dQ,reps,od,oi); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  double pairs=(double)blocks*threads*R*T*reps;
  double pps=pairs/(ms*1e-3);
  cudaFuncAttributes a; cudaFuncGetAttributes(&a,f);
  printf("%-28s R=%2d occ=%d regs=%3d  %.3f ms  %.3f Tpairs/s  FMA-pipe %.1f%% of peak@%dMHz  err=%s\n", name, R, blocksPerSM, a.numRegs, ms, pps/1e12,
         100.0*pps*6/(sms*128.0*clk*1e3), clk/1000, cudaGetErrorString(cudaGetLastError()));
}
int main(){
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  size_t nq=(size_t)sms*16*128*32;
  cudaMalloc(&dT,T*16); cudaMalloc(&dQ,nq*16); cudaMalloc(&od,nq*4); cudaMalloc(&oi,nq*4);
  float4* h=(float4*)malloc(nq*16); for(size_t i=0;i<nq;i++){h[i]=make_float4((i*37%1000)*1e-3f,(i*91%1000)*1e-3f,(i*13%1000)*1e-3f,0);}
  cudaMemcpy(dQ,h,nq*16,cudaMemcpyHostToDevice); cudaMemcpy(dT,h+7,T*16,cudaMemcpyHostToDevice);
  for(int pass=0;pass<2;pass++){
  for(int occ: {2,4}){
  run("scalar per-pair argmin", v_scalar_pair<8>, 8, occ);
  run("packed chunk4", v_packed_chunk<8,4>, 8, occ);
  run("packed chunk8", v_packed_chunk<8,8>, 8, occ);
  run("packed chunk4", v_packed_chunk<16,4>, 16, occ);
  run("packed block K=64", v_packed_block<8,64>, 8, occ);
  run("packed block K=64", v_packed_block<16,64>, 16, occ);
  run("scalar block K=64", v_scalar_block<8,64>, 8, occ);
  run("scalar block K=64", v_scalar_block<16,64>, 16, occ);
  run("packed no-min (ceiling)", v_packed_nomin<8>, 8, occ);
  run("packed no-min (ceiling)", v_packed_nomin<16>, 16, occ);
  }}
  return 0;
}
