// fma_mix.cu — can scalar FFMA (fmalite) run alongside packed FFMA2 (fmaheavy) to exceed 128
// lane-FMA/clk/SM?  Independent chains, 8 warps x 4 CTAs per SM.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
template <int NP, int NS>
__global__ void k(float* out, int iters, float s) {
    unsigned long long p[NP > 0 ? NP : 1];
    float f[NS > 0 ? NS : 1];
    const unsigned long long m = 0x3f8000003f800000ull;
    for (int i = 0; i < NP; ++i) p[i] = 0x3f0000003f000000ull + i + threadIdx.x;
    for (int i = 0; i < NS; ++i) f[i] = s * (i + threadIdx.x);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NP; ++i) p[i] = fma2(p[i], m, m);
#pragma unroll
        for (int i = 0; i < NS; ++i) f[i] = fmaf(f[i], 0.999f, s);
    }
    float t = 0;
    for (int i = 0; i < NP; ++i) t += __uint_as_float((unsigned)p[i]);
    for (int i = 0; i < NS; ++i) t += f[i];
    if (t == 1.2345f) out[0] = t;
}
template <int NP, int NS> void run(const char* name, float* d) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 8192, ctas = 148 * 4, thr = 256;
    k<NP, NS><<<ctas, thr>>>(d, 16, 1.f);
    cudaEventRecord(a); k<NP, NS><<<ctas, thr>>>(d, iters, 1.f); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double lane_ops = (double)ctas * thr * iters * (2.0 * NP + NS);
    printf("%-28s %.3f ms  %.1f lane-FMA/clk/SM at 1.965 GHz\n", name, ms, lane_ops / (ms * 1e-3) / 148 / 1.965e9);
}
int main() {
    float* d; cudaMalloc(&d, 4);
    run<8, 0>("FFMA2 x8", d);
    run<0, 16>("FFMA x16", d);
    run<8, 8>("FFMA2 x8 + FFMA x8", d);
    run<8, 4>("FFMA2 x8 + FFMA x4", d);
    run<8, 16>("FFMA2 x8 + FFMA x16", d);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
