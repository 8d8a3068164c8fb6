// umma_accum.cu — measures the fp32 accumulation error of tcgen05.mma kind::f16 (K = 16, fp16
// operands, fp32 accumulator, no input accumulator): D = sum_k A_k B_k with mixed-magnitude exact
// products, compared with the exact (fp64) sum.  Reports the max error in units of 2^-24 * 2^E where
// 2^E bounds the largest |product| (the truncation-after-alignment model predicts < 16 units).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ inline int cm_off(int r, int k) { return (r / 8) * 256 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2; }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}

__global__ void mm(const __half* A, const __half* B, float* D) {
    __shared__ __align__(1024) unsigned char sa[128 * 32];
    __shared__ __align__(1024) unsigned char sb[128 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x;
    const __half* Ab = A + (size_t)blockIdx.x * 128 * 16;
    const __half* Bb = B + (size_t)blockIdx.x * 128 * 16;
    for (int e = t; e < 128 * 16; e += blockDim.x) {
        *(__half*)(sa + cm_off(e / 16, e % 16)) = Ab[e];
        *(__half*)(sb + cm_off(e / 16, e % 16)) = Bb[e];
    }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tmem_base;
    if (t == 0) {
        const uint32_t idesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                     "l"(make_desc(smem_u32(sa))), "l"(make_desc(smem_u32(sb))), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int w = t / 32, lane = t % 32, row = w * 32 + lane;
    for (int c0 = 0; c0 < 128; c0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tm + ((uint32_t)(w * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int q = 0; q < 8; ++q) D[(size_t)blockIdx.x * 128 * 128 + row * 128 + c0 + q] = __uint_as_float(v[q]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

static double rnd() { return rand() / (RAND_MAX + 1.0); }

int main() {
    const int NB = 64;  // blocks of 128x128 outputs
    const size_t nA = (size_t)NB * 128 * 16;
    __half* hA = (__half*)malloc(nA * 2);
    __half* hB = (__half*)malloc(nA * 2);
    float* D = (float*)malloc((size_t)NB * 128 * 128 * 4);
    srand(7);
    for (size_t i = 0; i < nA; ++i) {
        // mixed magnitudes: value = sign * m * 2^-e, e in [0, 20], fp16-exact
        const int mode = rand() % 4;
        double v;
        if (mode == 0) v = (rnd() - 0.5);                       // ~0.5 scale
        else if (mode == 1) v = (rnd() - 0.5) * ldexp(1.0, -(rand() % 12));
        else if (mode == 2) v = (rnd() - 0.5) * ldexp(1.0, -11 - rand() % 8);   // tiny (lo parts)
        else v = (rand() % 2 ? 1 : -1) * 0.75;
        hA[i] = __float2half((float)v);
        v = (rnd() - 0.5) * ((rand() % 3 == 0) ? ldexp(1.0, -(rand() % 14)) : 2.0);
        hB[i] = __float2half((float)v);
    }
    __half *dA, *dB;
    float* dD;
    cudaMalloc(&dA, nA * 2);
    cudaMalloc(&dB, nA * 2);
    cudaMalloc(&dD, (size_t)NB * 128 * 128 * 4);
    cudaMemcpy(dA, hA, nA * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, nA * 2, cudaMemcpyHostToDevice);
    mm<<<NB, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    printf("err=%s\n", cudaGetErrorString(e));
    cudaMemcpy(D, dD, (size_t)NB * 128 * 128 * 4, cudaMemcpyDeviceToHost);
    double worst_units = 0, worst_rn_units = 0;
    long n_exact = 0, n = 0;
    for (int blk = 0; blk < NB; ++blk)
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; ++j) {
                double s = 0, maxp = 0, sabs = 0;
                for (int k = 0; k < 16; ++k) {
                    const double p = (double)__half2float(hA[((size_t)blk * 128 + i) * 16 + k]) *
                                     (double)__half2float(hB[((size_t)blk * 128 + j) * 16 + k]);
                    s += p;
                    maxp = fmax(maxp, fabs(p));
                    sabs += fabs(p);
                }
                const double got = D[(size_t)blk * 128 * 128 + i * 128 + j];
                const double err = fabs(got - s);
                if (maxp > 0) {
                    const double unit = ldexp(1.0, ilogb(maxp) - 23);   // ulp of the largest product
                    worst_units = fmax(worst_units, err / unit);
                }
                const double rn = (double)(float)s;
                if (got == rn) ++n_exact;
                if (fabs(s) > 0) worst_rn_units = fmax(worst_rn_units, err / ldexp(1.0, ilogb(fabs(s)) - 23));
                ++n;
            }
    printf("pairs=%ld  max err / ulp(max |product|) = %.3f   fraction equal to RN(exact sum) = %.4f   max err / ulp(result) = %.3f\n",
           n, worst_units, (double)n_exact / n, worst_rn_units);
    return 0;
}
