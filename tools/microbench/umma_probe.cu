// umma_probe.cu — first tcgen05 probe: D[128x128] = A[128x16] . B[128x16]^T (fp16 in, fp32 accum in
// TMEM), SWIZZLE_NONE K-major operands in shared memory.  Checks the descriptor conventions.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (r, k) in the no-swizzle K-major core-matrix layout
__host__ __device__ inline int cm_off(int r, int k, int lbo, int sbo) {
    return (r / 8) * sbo + (k / 8) * lbo + (r % 8) * 16 + (k % 8) * 2;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, int lbo, int sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;   // version = 1 (sm100)
    return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__global__ void probe(const __half* A, const __half* B, float* D, int lbo, int sbo, int swapdesc) {
    __shared__ __align__(1024) unsigned char sa[128 * 32];
    __shared__ __align__(1024) unsigned char sb[128 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x;
    for (int e = t; e < 128 * 16; e += blockDim.x) {
        const int r = e / 16, k = e % 16;
        *(__half*)(sa + cm_off(r, k, lbo, sbo)) = A[e];
        *(__half*)(sb + cm_off(r, k, lbo, sbo)) = B[e];
    }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");   // generic smem writes -> async proxy (MMA reads)
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tmem_base;
    if (t == 0) {
        const int l = swapdesc ? sbo : lbo, s = swapdesc ? lbo : sbo;
        const uint64_t da = make_desc(smem_u32(sa), l, s), db = make_desc(smem_u32(sb), l, s);
        // kind::f16: c F32 (bit 4), a/b F16 (0), K-major both, N=128 (>>3 at bit 17), M=128 (>>4 at bit 24)
        const uint32_t idesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
            "l"(da), "l"(db), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    // wait for the MMA
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
            smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int w = t / 32, lane = t % 32;
    const int row = w * 32 + lane;
    for (int c0 = 0; c0 < 128; c0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tm + ((uint32_t)(w * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int q = 0; q < 8; ++q) D[row * 128 + c0 + q] = __uint_as_float(v[q]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

int main() {
    __half hA[128 * 16], hB[128 * 16];
    float fA[128 * 16], fB[128 * 16];
    srand(1);
    for (int i = 0; i < 128 * 16; ++i) {
        fA[i] = (float)(rand() % 17 - 8) / 8.f;
        fB[i] = (float)(rand() % 17 - 8) / 8.f;
        hA[i] = __float2half(fA[i]);
        hB[i] = __float2half(fB[i]);
    }
    __half *dA, *dB;
    float* dD;
    cudaMalloc(&dA, sizeof(hA));
    cudaMalloc(&dB, sizeof(hB));
    cudaMalloc(&dD, 128 * 128 * 4);
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    static float D[128 * 128];
    const int cfg[4][3] = {{128, 256, 0}, {256, 128, 0}, {128, 256, 1}, {2048, 128, 0}};
    for (int c = 0; c < 4; ++c) {
        cudaMemset(dD, 0, 128 * 128 * 4);
        probe<<<1, 128>>>(dA, dB, dD, cfg[c][0], cfg[c][1], cfg[c][2]);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; ++j) {
                double r = 0;
                for (int k = 0; k < 16; ++k) r += (double)fA[i * 16 + k] * fB[j * 16 + k];
                maxerr = fmax(maxerr, fabs(r - D[i * 128 + j]));
            }
        printf("cfg lbo=%d sbo=%d swap=%d: err=%s maxerr=%g D[0]=%g D[1]=%g\n", cfg[c][0], cfg[c][1], cfg[c][2],
               cudaGetErrorString(e), maxerr, D[0], D[1]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
