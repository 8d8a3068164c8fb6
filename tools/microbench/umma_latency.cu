// umma_latency.cu — round-trip latency of (tcgen05.mma M=128 N=128 K=16 x2 -> tcgen05.commit ->
// mbarrier observed) and of tcgen05.ld 32x32b.x32 (+ wait::ld), measured with clock64 in one CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void wait_par(uint64_t* bar, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(bar)), "r"(par));
}

__global__ void lat(long long* out, int nmma) {
    __shared__ __align__(1024) unsigned char sa[128 * 32];
    __shared__ __align__(1024) unsigned char sb[128 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x;
    for (int e = t; e < 128 * 32; e += blockDim.x) { sa[e] = 0; sb[e] = 0; }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
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
    const uint32_t idesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    if (t == 0) {
        const uint64_t da = make_desc(smem_u32(sa)), db = make_desc(smem_u32(sb));
        long long t0 = clock64();
        for (int it = 0; it < 200; ++it) {
            for (int m = 0; m < nmma; ++m)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + (m & 3) * 128),
                             "l"(da), "l"(db), "r"(idesc), "r"(0));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
            wait_par(&bar, it & 1);
        }
        out[0] = (clock64() - t0) / 200;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t < 32) {
        uint32_t v[32];
        long long t0 = clock64();
        for (int it = 0; it < 200; ++it) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                  "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
                  "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
                  "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(tm + (it & 3) * 32));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            if ((v[0] ^ v[31]) == 12345u) out[5] = 1;
        }
        if (t == 0) out[1] = (clock64() - t0) / 200;
        // 4 loads then one wait
        t0 = clock64();
        for (int it = 0; it < 200; ++it) {
            uint32_t w[4];
            for (int h = 0; h < 4; ++h) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                      "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
                      "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
                      "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(tm + h * 32));
                w[h] = v[h] ^ v[31 - h];
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            if ((w[0] ^ w[1] ^ w[2] ^ w[3]) == 12345u) out[5] = 1;
        }
        if (t == 0) out[2] = (clock64() - t0) / 200;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    long long h[8];
    for (int nmma : {1, 2, 4, 8, 16}) {
        lat<<<1, 128>>>(d, nmma);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
        printf("nmma=%2d: mma+commit+wait %lld cyc | ld.x32+wait %lld cyc | 4x ld.x32 + wait %lld cyc (%s)\n", nmma, h[0], h[1], h[2],
               cudaGetErrorString(e));
    }
    return 0;
}
