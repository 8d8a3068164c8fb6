// tmem_ld_bw.cu — tcgen05.ld throughput: W warps (W/4 per SMSP lane quarter) each loading 128 columns
// per iteration with shapes 32x32b.x32 (4 loads) / .x64 (2) / .x128 (1), one wait::ld per iteration.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define R8(b) "=r"(v[b]), "=r"(v[b + 1]), "=r"(v[b + 2]), "=r"(v[b + 3]), "=r"(v[b + 4]), "=r"(v[b + 5]), "=r"(v[b + 6]), "=r"(v[b + 7])
template <int SHAPE>
__device__ __forceinline__ void ld128(uint32_t addr, uint32_t* v) {
    if constexpr (SHAPE == 32) {
        for (int h = 0; h < 4; ++h) {
            uint32_t* w = v + 32 * h;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]), "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]), "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
                         : "r"(addr + 32 * h));
        }
    } else if constexpr (SHAPE == 16) {   // 16 columns per load, 8 loads
        for (int h = 0; h < 8; ++h) {
            uint32_t* w = v + 16 * h;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
                         : "r"(addr + 16 * h));
        }
    }
}

template <int SHAPE>
__global__ void bw(long long* out, int iters) {
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t v[128];
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        ld128<SHAPE>(tm + (it & 3) * 128, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        acc ^= v[0] ^ v[37] ^ v[127];
    }
    long long dt = clock64() - t0;
    if (acc == 0x12345) out[7] = 1;
    __syncthreads();
    if (t == 0) out[0] = dt / iters;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    long long h;
    for (int W : {1, 4, 8, 16}) {
        bw<32><<<1, 32 * W>>>(d, 400);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("warps=%2d x32: %lld cyc per 128-col iteration per warp -> %.1f B/clk/SM\n", W, h, 32.0 * 128 * 4 * W / h);
        bw<16><<<1, 32 * W>>>(d, 400);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("warps=%2d x16: %lld cyc per 128-col iteration per warp -> %.1f B/clk/SM (%s)\n", W, h, 32.0 * 128 * 4 * W / h, cudaGetErrorString(e));
    }
    return 0;
}
