// cd_device.cuh — device-side helpers for libcd (sm_100a only).
// Packed-FP32 (f32x2) arithmetic, mbarrier + 1-D TMA bulk copies, and the fixed distance formula.
#pragma once
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libcd is written for sm_100a only (compile with -gencode arch=compute_100a,code=sm_100a)"
#endif

namespace cdk {

// Programmatic dependent launch (CD_PDL): kernels of the step are launched with programmatic stream
// serialisation so that a kernel's launch and CTA rasterisation overlap its predecessor's tail; every
// such kernel calls pdl_wait() before touching memory its predecessors wrote or read (it returns once
// the predecessor grid has completed and its writes are visible; a no-op without a programmatic edge).
#ifndef CD_PDL
#define CD_PDL 0
#endif
__device__ __forceinline__ void pdl_wait() {
#if CD_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// Device bounds checks for debug builds (-DCD_DEBUG_CHECKS=1, tools/build_variant.py): a failed check
// traps the kernel (cudaErrorLaunchFailure / assert) instead of corrupting memory.
#if CD_DEBUG_CHECKS
#define CD_CHECK(cond)                                                                          \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("CD_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                          \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define CD_CHECK(cond) \
    do {               \
    } while (0)
#endif


typedef unsigned long long u64;

// ---------------------------------------------------------------- tiling constants
constexpr int kFwdThreads = 128;                 // 4 warps per CTA
constexpr int kR = 16;                           // queries per thread (8 packed f32x2 pairs)
constexpr int kRSmall = 8;                       // fused kernel on small clouds: 1024-row query tiles
constexpr int kQTile = kFwdThreads * kR;         // 2048 queries per CTA
constexpr int kTile = 512;                       // targets per shared-memory stage (8 KB)
constexpr int kStages = 3;                       // TMA ring depth
constexpr int kBlockK = 32;                      // argmin block: the winning block is re-scanned
constexpr int kPad = kQTile;                     // packed clouds are padded to a multiple of this
constexpr int kMergeThreads = 256;               // queries per merge/epilogue CTA

// ---------------------------------------------------------------- packed FP32 (FADD2/FMUL2/FFMA2)
__device__ __forceinline__ u64 pk2(float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(u64 v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// 3-input min (FMNMX3): returns the non-NaN operand when one is NaN.
__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// The fixed fp32 distance formula: dx = RN(x - y); s = RN(dx*dx);
// s = fma(dy, dy, s); s = fma(dz, dz, s).  Per lane, the packed f32x2 ops round exactly like
// these scalar .rn ops, so this scalar form reproduces the packed loop bit for bit.
__device__ __forceinline__ float dist_rn(float qx, float qy, float qz, float tx, float ty, float tz) {
    float dx = __fsub_rn(qx, tx);
    float dy = __fsub_rn(qy, ty);
    float dz = __fsub_rn(qz, tz);
    float s = __fmul_rn(dx, dx);
    s = __fmaf_rn(dy, dy, s);
    s = __fmaf_rn(dz, dz, s);
    return s;
}

// Row key merged over target splits with a 64-bit atomicMin: the distance bits (d >= 0, so unsigned
// order is float order) then the block start (lowest block among equal minima); blk = -1 (no finite
// distance) becomes 0xffffffff.  Keys are >= 0 as signed 64-bit integers.
__device__ __forceinline__ long long row_key(float best, int blk) {
    return (long long)(((unsigned long long)__float_as_uint(best) << 32) | (unsigned long long)(unsigned)blk);
}

// 3-D Hilbert index of the cell (x[0], x[1], x[2]) of a 2^k grid (3k bits; Skilling's transpose
// algorithm, then bit interleave).  Space-filling order for the pruned paths: consecutive runs are
// more compact than Morton (Z-order) runs, so tile and block boxes are tighter.
__device__ __forceinline__ uint32_t hilbert3(uint32_t x0, uint32_t x1, uint32_t x2, int k) {
    uint32_t X[3] = {x0, x1, x2};
    const uint32_t M = 1u << (k - 1);
    for (uint32_t Q = M; Q > 1; Q >>= 1) {
        const uint32_t P = Q - 1;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (X[i] & Q) {
                X[0] ^= P;
            } else {
                const uint32_t t = (X[0] ^ X[i]) & P;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
    X[1] ^= X[0];
    X[2] ^= X[1];
    uint32_t t = 0;
    for (uint32_t Q = M; Q > 1; Q >>= 1)
        if (X[2] & Q) t ^= Q - 1;
    X[0] ^= t;
    X[1] ^= t;
    X[2] ^= t;
    // bit interleave (k <= 10): bit i of X[0] / X[1] / X[2] -> code bit 3i + 2 / 3i + 1 / 3i
    auto spread3 = [](uint32_t x) {
        x &= 0x3ffu;
        x = (x | (x << 16)) & 0x030000FFu;
        x = (x | (x << 8)) & 0x0300F00Fu;
        x = (x | (x << 4)) & 0x030C30C3u;
        x = (x | (x << 2)) & 0x09249249u;
        return x;
    };
    return (spread3(X[0]) << 2) | (spread3(X[1]) << 1) | spread3(X[2]);
}

// ---------------------------------------------------------------- mbarrier + TMA bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(u64* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(u64* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "CD_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra CD_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared (cp.async.bulk, SASS UBLKCP), completion counted on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, u64* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace cdk
