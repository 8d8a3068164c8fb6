// redux_tp.cu — throughput of redux.sync.min (u32 and f32) vs FMNMX3, and whether they co-issue.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float fmin3(float a, float b, float c) { float r; asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ unsigned rmin(unsigned v) { unsigned r; asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v)); return r; }
__device__ __forceinline__ float rminf(float v) { float r; asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v)); return r; }

template <int MODE>
__global__ void k(float* out, int iters, float seed) {
    float a[8];
    unsigned u[8];
    for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i); u[i] = __float_as_uint(a[i]); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) a[i] = fmin3(a[i], a[(i + 1) & 7] + 1.f, seed);
            if (MODE == 1) u[i] = rmin(u[i] ^ it) + i;
            if (MODE == 2) a[i] = rminf(a[i] + seed) * 0.5f;
            if (MODE == 3) { a[i] = fmin3(a[i], a[(i + 1) & 7], seed); u[i] = rmin(u[i] ^ it); }
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + u[i];
    if (s == 1.2345f) out[0] = s;
}

int main() {
    float* d;
    cudaMalloc(&d, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[4] = {"FMNMX3 x8 (+FADD)", "REDUX.MIN.U32 x8 (+IADD/LOP)", "REDUX.MIN.F32 x8 (+FADD,FMUL)", "FMNMX3 x8 + REDUX.U32 x8"};
    for (int m = 0; m < 4; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            const int iters = 4096;
            cudaEventRecord(e0);
            if (m == 0) k<0><<<148 * 4, 256>>>(d, iters, 1.0f);
            if (m == 1) k<1><<<148 * 4, 256>>>(d, iters, 1.0f);
            if (m == 2) k<2><<<148 * 4, 256>>>(d, iters, 1.0f);
            if (m == 3) k<3><<<148 * 4, 256>>>(d, iters, 1.0f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            // warp-instr of the named op per SMSP: 148*4 CTAs * 8 warps * iters * 8 / (148*4 SMSPs)
            const double per_smsp = 4.0 * 8 * iters * 8 / 4;
            if (rep) printf("%-34s %.3f ms  -> %.2f cycles per op-instr per SMSP (at 1.9 GHz)\n", names[m], ms, ms * 1e-3 * 1.9e9 / per_smsp);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
