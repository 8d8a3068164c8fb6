// nn_tc.cu — tensor-core forward of the exact bidirectional nearest-neighbour search (DESIGN.md §4.7,
// reading R27).  The 5th-generation tensor cores (tcgen05.mma, accumulators in TMEM) evaluate an
// APPROXIMATION of every squared distance; the exact fp32 results of the fixed formula (§4.2) are then
// recovered by re-evaluating only the targets that the approximation cannot rule out:
//
//   tc_bbox_kernel    per batch element: exact bounding box of the finite points of both clouds.
//   tc_pack_kernel    centre c and power-of-two scale s per batch element (|u| <= 1/2 for
//                     u = (p - c) s); packed float4 clouds (+inf padding) for the exact re-scans; the
//                     MMA operands: per point 16 fp16 values in the tcgen05 no-swizzle K-major
//                     core-matrix layout (128-row tiles of 4 KB), u split as h + l (fp16 hi/lo):
//                       query  row  [h, l, h, n_h, n_l, 1, 1, 0,0,0]        (n = |u|^2 split hi/lo)
//                       target row  [-2H, -2H, -2L, 1, 1, N_h, N_l, 0,0,0]
//                     so that one K=16 MMA gives  D~ = |u|^2 + |w|^2 - 2 u.w  (the l.L term dropped);
//                     resets the top-3 key arrays.
//   nn_tc_kernel      CTA = 1024 queries (8 sub-blocks of 128) x a split of the targets (128-target
//                     tiles through a TMA ring); warp 0 = TMA producer, warp 1 = MMA issuer (TMEM
//                     owner), warps 2-5 = rows (D1 = Q T^T: TMEM lane = query), warps 6-9 = columns
//                     (D2 = T Q^T: TMEM lane = target).  Per (tile, sub-block) two M=128 N=128 K=16
//                     MMAs into a double-buffered 2 x 256-column TMEM accumulator.  Epilogue threads
//                     read their lane's 128 values (tcgen05.ld), fold 32-value chunks with FMNMX3 and
//                     keep the three smallest chunk minima with the first two chunks' block starts.
//                     At the end they merge into global top-3 keys (first = min, second = min of the
//                     rest, third value) with 64-bit atomicMin; every key that loses a comparison is
//                     pushed one level down, so the final arrays are exactly the 3 smallest keys.
//   tc_resolve_kernel exact re-scan (dist_rn) of block 1, and of block 2 when its approximate minimum
//                     lies inside the band m1 + T; if the third value is inside the band too the row is
//                     queued for tc_fallback_kernel (exact brute force over all targets).
//   tc_chunks_kernel  per-chunk fp64 sums and hit counts from the final distances -> partials.
//
// Exactness (R27): |D~ - s^2 |p - q|^2| <= E (E = kTcErel U^2: fp16 split residuals + the measured tensor-
// core fp32 accumulation, truncation after alignment, <= 16 ulp of the largest product; profiles/
// r01_umma_accum.txt) and the fp32 formula is within 2^-20 relative of |p - q|^2.  Any target whose
// exact fp32 distance equals the row minimum then has D~ <= m1 + T with T = 2E + 2^-18 (|m1| + E), so
// it lies in a block whose chunk minimum is inside the band: re-scanning every such block gives the
// exact minimum and the lowest index, i.e. the brute force's result bit for bit.
#include "cd_device.cuh"
#include "cd_internal.h"

#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>

namespace cdk {

constexpr int kTcRows = 128;                     // MMA M = N = 128
constexpr int kTcSub = 8;                        // query sub-blocks per CTA
constexpr int kTcQB = kTcRows * kTcSub;          // 1024 queries per CTA
constexpr int kTcStages = 3;                     // target tile ring
#ifndef CD_TC_HALVES
#define CD_TC_HALVES 1
#endif
constexpr int kTcHalves = CD_TC_HALVES;          // column halves per lane quarter (1: a warp reads all 128 columns)
constexpr int kTcEpiWarps = 8 * kTcHalves;       // 2 groups (rows, columns) x 4 lane quarters x halves
constexpr int kTcThreads = 32 * (3 + kTcEpiWarps);   // + TMA warp + 2 MMA warps (one per group)
constexpr int kTcTileBytes = kTcRows * 32;       // 128 rows x 16 fp16
constexpr int kTcChunk = 64;                     // targets / queries per tracked chunk (block)
constexpr float kTcErel = 1.6e-5f;               // R27: E = kTcErel * U^2 (4e-6 at U = 1/2: 2x the derived bound)
constexpr float kTcPadNorm = 30000.0f;           // padded operand rows: D~ >= 30000

// ------------------------------------------------------------------------------------------ helpers
// order-preserving map float -> u32 (unsigned order = float order, NaN excluded)
__device__ __forceinline__ uint32_t ford(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float funord(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
// byte offset of element (row r, k) inside a 128 x 16 fp16 no-swizzle K-major tile (LBO 128, SBO 256)
__device__ __forceinline__ int tc_cm_off(int r, int k) {
    return (r >> 3) * 256 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46);
}

// ------------------------------------------------------------------------------------------ bbox
struct TcBoxArgs {
    const float* src[2];
    int npts[2];
    int B;
    unsigned* box;   // [B][6]: ford(lo xyz), ford(-hi xyz), both reduced with atomicMin (identity ~0)
};

__global__ void __launch_bounds__(256) tc_bbox_kernel(TcBoxArgs a) {
    const int b = blockIdx.y;
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    const int64_t n0 = a.npts[0], n = n0 + a.npts[1];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const float* p = e < n0 ? a.src[0] + ((int64_t)b * n0 + e) * 3 : a.src[1] + ((int64_t)b * a.npts[1] + (e - n0)) * 3;
        const float x = __ldg(p), y = __ldg(p + 1), z = __ldg(p + 2);
        if (isfinite(x) && isfinite(y) && isfinite(z)) {
            lo[0] = fminf(lo[0], x); hi[0] = fmaxf(hi[0], x);
            lo[1] = fminf(lo[1], y); hi[1] = fmaxf(hi[1], y);
            lo[2] = fminf(lo[2], z); hi[2] = fmaxf(hi[2], z);
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
    if ((threadIdx.x & 31) == 0 && lo[0] <= hi[0])
        for (int k = 0; k < 3; ++k) {
            atomicMin(&a.box[b * 6 + k], ford(lo[k]));
            atomicMin(&a.box[b * 6 + 3 + k], ford(-hi[k]));
        }
}

// ------------------------------------------------------------------------------------------ pack
struct TcPackArgs {
    const float* src[2];
    int npts[2], ppad[2];
    int B;
    const unsigned* box;
    float4* pack[2];          // [B][ppad] float4, +inf padding
    unsigned char* op[2];     // [B][ppad/128][4096 B] fp16 operand tiles (0: query form, 1: target form)
    unsigned* fb_count;       // fallback queue length
};

// centre c, power-of-two scale s and U >= max |u| (U <= 1/2) of a batch element
__device__ __forceinline__ void tc_scale(const unsigned* box, float c[3], float& s, float& U) {
    float R = 0.f;
    bool any = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float lo = funord(box[k]), hi = -funord(box[3 + k]);   // ~0 (empty) -> NaN
        if (!(lo <= hi)) any = false;
        c[k] = 0.5f * lo + 0.5f * hi;
        R = fmaxf(R, fmaxf(hi - c[k], c[k] - lo));
    }
    if (!any) {
        c[0] = c[1] = c[2] = 0.f;
        s = 1.f;
        U = 0.5f;
        return;
    }
    R *= 1.0f + 1.0f / 1048576.0f;
    int e = 0;
    frexpf(R, &e);                   // R = m 2^e, m in [0.5, 1): 2^e >= R
    s = R > 0.f ? ldexpf(1.0f, -(e + 1)) : 1.0f;   // |u| <= R s <= 1/2
    U = R > 0.f ? fminf(0.5f, R * s * (1.0f + 1.0f / 1048576.0f)) : 0.5f;
}

__global__ void __launch_bounds__(256) tc_pack_kernel(TcPackArgs a) {
    const int64_t P0 = (int64_t)a.B * a.ppad[0];
    const int64_t total = P0 + (int64_t)a.B * a.ppad[1];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = e < P0 ? 0 : 1;
        const int64_t f = c == 0 ? e : e - P0;
        const int b = (int)(f / a.ppad[c]);
        const int i = (int)(f - (int64_t)b * a.ppad[c]);
        __half row[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) row[k] = __float2half(0.f);
        if (i < a.npts[c]) {
            const float* p = a.src[c] + ((int64_t)b * a.npts[c] + i) * 3;
            const float x = p[0], y = p[1], z = p[2];
            a.pack[c][f] = make_float4(x, y, z, 0.f);
            float cc[3], s, U;
            tc_scale(a.box + b * 6, cc, s, U);
            const float u[3] = {__fmul_rn(__fsub_rn(x, cc[0]), s), __fmul_rn(__fsub_rn(y, cc[1]), s),
                                __fmul_rn(__fsub_rn(z, cc[2]), s)};
            __half h[3], l[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                h[k] = __float2half_rn(u[k]);
                l[k] = __float2half_rn(__fsub_rn(u[k], __half2float(h[k])));
            }
            const float n = __fmaf_rn(u[2], u[2], __fmaf_rn(u[1], u[1], __fmul_rn(u[0], u[0])));
            const __half nh = __float2half_rn(n);
            const __half nl = __float2half_rn(__fsub_rn(n, __half2float(nh)));
            const __half one = __float2half(1.f);
            if (c == 0) {   // query form
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    row[k] = h[k];
                    row[3 + k] = l[k];
                    row[6 + k] = h[k];
                }
                row[9] = nh;
                row[10] = nl;
                row[11] = one;
                row[12] = one;
            } else {        // target form
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const __half m2h = __float2half_rn(-2.f * __half2float(h[k]));   // exact
                    row[k] = m2h;
                    row[3 + k] = m2h;
                    row[6 + k] = __float2half_rn(-2.f * __half2float(l[k]));         // exact
                }
                row[9] = one;
                row[10] = one;
                row[11] = nh;
                row[12] = nl;
            }
        } else {
            a.pack[c][f] = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
            row[c == 0 ? 9 : 11] = __float2half(kTcPadNorm);
        }
        unsigned char* tile = a.op[c] + (f >> 7) * kTcTileBytes;
        const int r = (int)(f & 127);
        // two 16-byte core-matrix rows (k 0-7 and 8-15)
        uint4 lo4, hi4;
        __half* lo = reinterpret_cast<__half*>(&lo4);
        __half* hi = reinterpret_cast<__half*>(&hi4);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            lo[k] = row[k];
            hi[k] = row[8 + k];
        }
        *reinterpret_cast<uint4*>(tile + tc_cm_off(r, 0)) = lo4;
        *reinterpret_cast<uint4*>(tile + tc_cm_off(r, 8)) = hi4;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.fb_count = 0u;
}

// ------------------------------------------------------------------------------------------ main kernel
struct TcArgs {
    const unsigned char* op[2];
    int npts[2], ppad[2];
    int qblocks, splits, ttiles;   // per batch element: query blocks, target splits, target tiles
    float4* rowsum;   // [splits][B*N]: (m1, m2, m3, b1 | b2 << 16) per (split, query row)
    float4* colsum;   // [qblocks][B*M]: the same per (query block, target)
};

// insert a chunk minimum into a thread's local top-3 (two with blocks): branch-free sorting network
// (the epilogue runs it for every chunk; a data-dependent branch diverges across the warp)
__device__ __forceinline__ void top3_insert(float cm, int blk, float& m1, int& b1, float& m2, int& b2, float& m3) {
    const bool p1 = cm < m1, p2 = cm < m2;
    m3 = fminf(m3, fmaxf(m2, cm));
    m2 = fminf(m2, fmaxf(m1, cm));
    b2 = p2 ? (p1 ? b1 : blk) : b2;
    b1 = p1 ? blk : b1;
    m1 = fminf(m1, cm);
}

__device__ __forceinline__ float4 top3_pack(float m1, int b1, float m2, int b2, float m3) {
    return make_float4(m1, m2, m3, __int_as_float((b1 & 0xffff) | (b2 << 16)));
}

__device__ __forceinline__ float chunk_min32(const uint32_t* v) {
    float a0 = fmin3(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]));
    float a1 = fmin3(__uint_as_float(v[8]), __uint_as_float(v[9]), __uint_as_float(v[10]));
    float a2 = fmin3(__uint_as_float(v[16]), __uint_as_float(v[17]), __uint_as_float(v[18]));
    float a3 = fmin3(__uint_as_float(v[24]), __uint_as_float(v[25]), __uint_as_float(v[26]));
#pragma unroll
    for (int j = 3; j < 7; j += 2) {
        a0 = fmin3(a0, __uint_as_float(v[j]), __uint_as_float(v[j + 1]));
        a1 = fmin3(a1, __uint_as_float(v[8 + j]), __uint_as_float(v[9 + j]));
        a2 = fmin3(a2, __uint_as_float(v[16 + j]), __uint_as_float(v[17 + j]));
        a3 = fmin3(a3, __uint_as_float(v[24 + j]), __uint_as_float(v[25 + j]));
    }
    a0 = fmin3(a0, __uint_as_float(v[7]), a1);
    a2 = fmin3(a2, __uint_as_float(v[15]), __uint_as_float(v[23]));
    return fmin3(a0, a2, fmin3(a3, __uint_as_float(v[31]), INFINITY));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(u64* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_commit(u64* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
        "l"(da), "l"(db), "r"(idesc), "r"(0)
        : "memory");
}

// One (tile, sub-block) step of an epilogue warp: wait for the accumulator, read the lane's 64
// values of its column half (two 32-column loads), release the TMEM buffer, return the chunk minimum.
__device__ __forceinline__ void tc_step_min(uint32_t tl, int step, u64* tfull, u64* tempty, int lane,
                                            float c[2 / kTcHalves]) {
    const int buf = step & 1;
    const int use = step >> 1;
    mbar_wait(&tfull[buf], use & 1);
    __syncwarp();
    tc_fence_after();
    uint32_t v[64];
#pragma unroll
    for (int h = 0; h < 2 / kTcHalves; ++h) {
#ifdef CD_TC_NOLD
        v[0] = tl + h; v[63] = step;
#else
        tmem_ld32(tl + buf * 128 + 64 * h, v);
        tmem_ld32(tl + buf * 128 + 64 * h + 32, v + 32);
        tmem_wait_ld();
#endif
#ifdef CD_TC_NOCOMPUTE
        c[h] = __uint_as_float(v[0] ^ v[63]);
#else
        c[h] = fminf(chunk_min32(v), chunk_min32(v + 32));
#endif
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[buf]);
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__global__ void __launch_bounds__(kTcThreads, 1) nn_tc_kernel(TcArgs a) {
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    unsigned char* sq = tc_smem;                                  // 8 query sub-block tiles (32 KB)
    unsigned char* st = tc_smem + kTcSub * kTcTileBytes;          // target tile ring
    u64* full_bar = reinterpret_cast<u64*>(st + kTcStages * kTcTileBytes);
    u64* empty_bar = full_bar + kTcStages;
    u64* tfull = empty_bar + kTcStages;    // [2 groups][2 buffers]
    u64* tempty = tfull + 4;               // [2 groups][2 buffers]
    u64* qbar = tempty + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qbar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    const int qblk = blockIdx.x / a.splits, split = blockIdx.x - (blockIdx.x / a.splits) * a.splits;
    const int t0 = (int)((int64_t)split * a.ttiles / a.splits), t1 = (int)((int64_t)(split + 1) * a.ttiles / a.splits);
    const int nt = t1 - t0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 2);   // released by both groups' MMA commits
        }
        for (int s = 0; s < 4; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], kTcEpiWarps / 2);
        }
        mbar_init(qbar, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {   // TMA producer
            const unsigned char* Q = a.op[0] + ((int64_t)b * (a.ppad[0] / kTcRows) + (int64_t)qblk * kTcSub) * kTcTileBytes;
            const unsigned char* T = a.op[1] + ((int64_t)b * (a.ppad[1] / kTcRows) + t0) * kTcTileBytes;
            mbar_arrive_expect_tx(qbar, kTcSub * kTcTileBytes);
            tma_load_1d(sq, Q, kTcSub * kTcTileBytes, qbar);
            for (int k = 0; k < nt; ++k) {
                const int s = k % kTcStages;
                if (k >= kTcStages) mbar_wait(&empty_bar[s], ((k / kTcStages) - 1) & 1);
                mbar_arrive_expect_tx(&full_bar[s], kTcTileBytes);
                tma_load_1d(st + s * kTcTileBytes, T + (int64_t)k * kTcTileBytes, kTcTileBytes, &full_bar[s]);
            }
        }
    } else if (warp == 1 || warp == 2) {
        if (lane == 0) {   // MMA issuer of group g: g = 0 -> D1 = Q_q T^T (lane = query), 1 -> D2 = T Q_q^T
            const int g = warp - 1;
            const uint32_t idesc = (1u << 4) | ((uint32_t)(kTcRows >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
            mbar_wait(qbar, 0);
            tc_fence_after();
            for (int k = 0; k < nt; ++k) {
                const int s = k % kTcStages;
                mbar_wait(&full_bar[s], (k / kTcStages) & 1);
                tc_fence_after();
                const uint64_t dt = tc_desc(smem_u32(st + s * kTcTileBytes));
#pragma unroll
                for (int q = 0; q < kTcSub; ++q) {
                    const int buf = q & 1;
                    const int use = k * (kTcSub / 2) + (q >> 1);   // n-th use of this buffer
                    if (use > 0) mbar_wait(&tempty[2 * g + buf], (use - 1) & 1);
                    tc_fence_after();
                    const uint64_t dq = tc_desc(smem_u32(sq + q * kTcTileBytes));
#ifndef CD_TC_NOMMA
                    if (g == 0) tc_mma(tmem + buf * 128, dq, dt, idesc);
                    else tc_mma(tmem + 256 + buf * 128, dt, dq, idesc);
#endif
                    tc_commit(&tfull[2 * g + buf]);
                }
                tc_commit(&empty_bar[s]);
            }
        }
    } else {
        // epilogue: warps 2-9 = rows (D1), 10-17 = columns (D2); a warp reads the TMEM lane quarter
        // warp % 4 (hardware rule) and the column half (warp - 2) / 4 % 2 of its group's accumulator:
        // one 64-column chunk per step.  The two halves of a lane quarter merge through shared memory.
        const int w = warp - 3;
        const int group = w / (4 * kTcHalves);
        const int half = kTcHalves == 1 ? 0 : (w >> 2) & 1;
        const int lbase = 32 * (warp & 3);
        const int r = lbase + lane;
        const uint32_t tl = tmem + ((uint32_t)lbase << 16) + (group ? 256u : 0u) + 64u * half;
        constexpr int CPS = 2 / kTcHalves;   // 64-column chunks per warp and step
        const int N = a.npts[0], M = a.npts[1];
        const int64_t BN = (int64_t)gridDim.y * N, BM = (int64_t)gridDim.y * M;
        const int pair_bar = 1 + group * 4 + (warp & 3);   // named barrier of the two halves (64 threads)
        // shared state: rows [5][kTcSub][2 halves][128]; column-half exchange [5][128] per group
        float* rs = reinterpret_cast<float*>(tmem_slot + 4);
        float* xs = rs + 5 * kTcSub * 2 * kTcRows;
        auto RS = [&](int f, int q) -> float& { return rs[((f * kTcSub + q) * 2 + half) * kTcRows + r]; };
        if (group == 0)
            for (int q = 0; q < kTcSub; ++q) {
                RS(0, q) = INFINITY;
                RS(1, q) = INFINITY;
                RS(2, q) = INFINITY;
                RS(3, q) = __int_as_float(0);
                RS(4, q) = __int_as_float(0);
            }
        float cm1 = INFINITY, cm2 = INFINITY, cm3 = INFINITY;
        int cb1 = 0, cb2 = 0;
#pragma unroll 1
        for (int step = 0; step < nt * kTcSub; ++step) {
            const int k = step / kTcSub, q = step - k * kTcSub;
            float c[CPS];
            tc_step_min(tl, step, tfull + 2 * group, tempty + 2 * group, lane, c);
            if (group == 0) {
                float m1 = RS(0, q), m2 = RS(1, q), m3 = RS(2, q);
                int b1 = __float_as_int(RS(3, q)), b2 = __float_as_int(RS(4, q));
#pragma unroll
                for (int h = 0; h < CPS; ++h) top3_insert(c[h], 2 * k + half + h, m1, b1, m2, b2, m3);   // local chunk
                RS(0, q) = m1;
                RS(1, q) = m2;
                RS(2, q) = m3;
                RS(3, q) = __int_as_float(b1);
                RS(4, q) = __int_as_float(b2);
            } else {
#pragma unroll
                for (int h = 0; h < CPS; ++h) top3_insert(c[h], 2 * q + half + h, cm1, cb1, cm2, cb2, cm3);   // local chunk
                if (q == kTcSub - 1) {
                    float* x = xs + r;   // [5][128]
                    if (kTcHalves == 2 && half == 1) {
                        x[0] = cm1;
                        x[kTcRows] = cm2;
                        x[2 * kTcRows] = cm3;
                        x[3 * kTcRows] = __int_as_float(cb1);
                        x[4 * kTcRows] = __int_as_float(cb2);
                    }
                    if (kTcHalves == 2) named_bar(pair_bar, 64);
                    if (half == 0) {
                        if (kTcHalves == 2) {
                            top3_insert(x[0], __float_as_int(x[3 * kTcRows]), cm1, cb1, cm2, cb2, cm3);
                            top3_insert(x[kTcRows], __float_as_int(x[4 * kTcRows]), cm1, cb1, cm2, cb2, cm3);
                            top3_insert(x[2 * kTcRows], -1, cm1, cb1, cm2, cb2, cm3);
                        }
                        const int j = (t0 + k) * kTcRows + r;
                        if (j < M) a.colsum[(int64_t)qblk * BM + (int64_t)b * M + j] = top3_pack(cm1, cb1, cm2, cb2, cm3);
                    }
                    if (kTcHalves == 2) named_bar(pair_bar, 64);   // exchange slot free again
                    cm1 = cm2 = cm3 = INFINITY;
                    cb1 = cb2 = 0;
                }
            }
        }
        if (group == 0) {
            if (kTcHalves == 2) named_bar(pair_bar, 64);
            if (half == 0)
                for (int q = 0; q < kTcSub; ++q) {
                    const int i = qblk * kTcQB + q * kTcRows + r;
                    float m1 = RS(0, q), m2 = RS(1, q), m3 = RS(2, q);
                    int b1 = __float_as_int(RS(3, q)), b2 = __float_as_int(RS(4, q));
                    if (kTcHalves == 2) {
                        const int o = kTcRows;   // the other half's slots
                        top3_insert((&RS(0, q))[o], __float_as_int((&RS(3, q))[o]), m1, b1, m2, b2, m3);
                        top3_insert((&RS(1, q))[o], __float_as_int((&RS(4, q))[o]), m1, b1, m2, b2, m3);
                        top3_insert((&RS(2, q))[o], -1, m1, b1, m2, b2, m3);
                    }
                    if (i < N) a.rowsum[(int64_t)split * BN + (int64_t)b * N + i] = top3_pack(m1, b1, m2, b2, m3);
                }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------------------------------------------ resolve
struct TcResolveArgs {
    const unsigned* box;
    const float4* pack[2];
    int npts[2], ppad[2];
    int B, splits, ttiles, qblocks;
    const float4* sums[2];   // 0: rowsum [splits][B*N], 1: colsum [qblocks][B*M]
    float* d_out[2];
    int32_t* idx_out[2];
    unsigned* fb_count;
    unsigned* fb_list;       // (dir << 31) | flat row
};

__device__ __forceinline__ void rescan_block(float4 q, const float4* T, int start, int nT, float& bd, int& bi) {
    const int end = min(start + kTcChunk, nT);
    for (int j = start; j < end; ++j) {
        const float4 t = T[j];
        const float d = dist_rn(q.x, q.y, q.z, t.x, t.y, t.z);
        if (d < bd || (d == bd && j < bi)) {
            bd = d;
            bi = j;
        }
    }
}

// Merge the per-CTA summaries of a row: global top-2 chunk minima with their first target index
// (-1: a value whose chunk is unknown, i.e. some CTA's third) and the third value; then re-scan the
// chunks inside the band warp-cooperatively (lanes over the chunk's targets: coalesced loads).
__global__ void __launch_bounds__(256) tc_resolve_kernel(TcResolveArgs a) {
    const int64_t L0 = (int64_t)a.B * a.npts[0];
    const int64_t L = L0 + (int64_t)a.B * a.npts[1];
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32; base < L; base += nwarps * 32) {
        const int64_t e = base + lane;
        const bool valid = e < L;
        const int dir = (valid && e >= L0) ? 1 : 0;
        const int64_t g = dir == 0 ? e : e - L0;
        const int n = a.npts[dir];
        const int b = valid ? (int)(g / n) : 0;
        const int i = valid ? (int)(g - (int64_t)b * n) : 0;
        float g1 = INFINITY, g2 = INFINITY, g3 = INFINITY;
        int gb1 = -1, gb2 = -1;
        if (valid) {
            const int64_t stride = (int64_t)a.B * n;
            const int nsum = dir == 0 ? a.splits : a.qblocks;
            for (int k = 0; k < nsum; ++k) {
                const float4 v = a.sums[dir][(int64_t)k * stride + g];
                const int cb = dir == 0 ? (int)((int64_t)k * a.ttiles / a.splits) * kTcRows : k * kTcQB;
                const unsigned bb = __float_as_uint(v.w);
                top3_insert(v.x, cb + kTcChunk * (int)(bb & 0xffffu), g1, gb1, g2, gb2, g3);
                top3_insert(v.y, cb + kTcChunk * (int)(bb >> 16), g1, gb1, g2, gb2, g3);
                top3_insert(v.z, -1, g1, gb1, g2, gb2, g3);
            }
        }
        int nblk = 0;
        bool fb = false;
        if (valid && g1 < INFINITY) {
            float cc[3], sc, U;
            tc_scale(a.box + b * 6, cc, sc, U);
            const float E = kTcErel * U * U;
            const float thr = g1 + (2.f * E + (fabsf(g1) + E) * (1.0f / 262144.0f));
            fb = gb1 < 0 || g3 <= thr || (g2 <= thr && gb2 < 0);
            nblk = fb ? 0 : (g2 <= thr ? 2 : 1);
        }
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (nblk) q = a.pack[dir][(int64_t)b * a.ppad[dir] + i];
        float my_d = INFINITY;
        int my_i = 0x7fffffff;
        unsigned todo = __ballot_sync(0xffffffffu, nblk > 0);
        // four rows per step: lane group grp (8 lanes) re-scans the grp-th pending row; its 8 lanes
        // take interleaved targets of each 64-target chunk (every load instruction covers one
        // contiguous 128-byte line per row), then an 8-lane (distance, index) reduction
        const int grp = lane >> 3, gl = lane & 7;
        while (todo) {
            int src = -1;
            {
                unsigned t = todo;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int f = t ? __ffs(t) - 1 : -1;
                    if (t) t &= t - 1;
                    if (k == grp) src = f;
                }
                todo = t;
            }
            const int srcc = src < 0 ? 0 : src;
            const int sdir = __shfl_sync(0xffffffffu, dir, srcc);
            const int sb = __shfl_sync(0xffffffffu, b, srcc);
            const int snb = __shfl_sync(0xffffffffu, nblk, srcc);
            const int s1 = __shfl_sync(0xffffffffu, gb1, srcc), s2 = __shfl_sync(0xffffffffu, gb2, srcc);
            const float qx = __shfl_sync(0xffffffffu, q.x, srcc), qy = __shfl_sync(0xffffffffu, q.y, srcc),
                        qz = __shfl_sync(0xffffffffu, q.z, srcc);
            float bd = INFINITY;
            int bi = 0x7fffffff;
            if (src >= 0) {
                const int snT = a.npts[1 - sdir];
                const float4* T = a.pack[1 - sdir] + (int64_t)sb * a.ppad[1 - sdir];
                for (int h = 0; h < snb; ++h) {
                    const int start = h == 0 ? s1 : s2;
                    float4 t[kTcChunk / 8];
#pragma unroll
                    for (int u = 0; u < kTcChunk / 8; ++u) t[u] = T[min(start + 8 * u + gl, snT - 1)];
#pragma unroll
                    for (int u = 0; u < kTcChunk / 8; ++u) {   // j ascending per lane
                        const int j = start + 8 * u + gl;
                        const float d = dist_rn(qx, qy, qz, t[u].x, t[u].y, t[u].z);
                        if (j < snT && (d < bd || (d == bd && j < bi))) {
                            bd = d;
                            bi = j;
                        }
                    }
                }
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                const float od = __shfl_xor_sync(0xffffffffu, bd, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (od < bd || (od == bd && oi < bi)) {
                    bd = od;
                    bi = oi;
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {   // hand each group's result to the row's own lane
                const int ks = __shfl_sync(0xffffffffu, src, 8 * k);
                const float kd = __shfl_sync(0xffffffffu, bd, 8 * k);
                const int ki = __shfl_sync(0xffffffffu, bi, 8 * k);
                if (lane == ks) {
                    my_d = kd;
                    my_i = ki;
                }
            }
        }
        if (valid) {
            a.d_out[dir][g] = my_d;
            a.idx_out[dir][g] = my_i == 0x7fffffff ? -1 : my_i;
        }
        // warp-aggregated enqueue of the rows the band cannot settle (one atomic per warp)
        const unsigned fbm = __ballot_sync(0xffffffffu, fb);
        if (fbm) {
            const int leader = __ffs(fbm) - 1;
            unsigned qbase = 0;
            if (lane == leader) qbase = atomicAdd(a.fb_count, (unsigned)__popc(fbm));
            qbase = __shfl_sync(0xffffffffu, qbase, leader);
            if (fb) a.fb_list[qbase + __popc(fbm & ((1u << lane) - 1u))] = ((unsigned)dir << 31) | (unsigned)g;
        }
    }
}

// Exact re-scan of the queued rows (the band could not be settled from the merged summaries): one CTA
// (256 threads) per row.  It re-reads the row's per-CTA summaries and scans only what can hold a
// target inside the band: the identified chunks whose minimum is inside it, and the WHOLE target
// range of every CTA whose third chunk minimum is inside it (that CTA's untracked chunks may be
// too); with thousands of such ranges (never seen) the whole cloud.  Targets are compared
// lexicographically on (distance, index), so the range order does not matter.
constexpr int kTcFbRanges = 2048;
__global__ void __launch_bounds__(256) tc_fallback_kernel(TcResolveArgs a) {
    const unsigned count = *a.fb_count;
    __shared__ float sd[8];
    __shared__ int si[8];
    __shared__ float s_g1[8];
    __shared__ int2 s_rng[kTcFbRanges];
    __shared__ unsigned s_nr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (unsigned w = blockIdx.x; w < count; w += gridDim.x) {
        const unsigned item = a.fb_list[w];
        const int dir = item >> 31;
        const int64_t g = item & 0x7fffffffu;
        const int n = a.npts[dir], nT = a.npts[1 - dir];
        const int b = (int)(g / n);
        const int i = (int)(g - (int64_t)b * n);
        CD_CHECK(b < a.B && i < n);
        const float4 q = a.pack[dir][(int64_t)b * a.ppad[dir] + i];
        const float4* T = a.pack[1 - dir] + (int64_t)b * a.ppad[1 - dir];
        const int64_t stride = (int64_t)a.B * n;
        const int nsum = dir == 0 ? a.splits : a.qblocks;
        // the band threshold from the smallest approximate minimum (as tc_resolve_kernel)
        float m = INFINITY;
        for (int k = threadIdx.x; k < nsum; k += 256) m = fminf(m, a.sums[dir][(int64_t)k * stride + g].x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) s_g1[warp] = m;
        if (threadIdx.x == 0) s_nr = 0u;
        __syncthreads();
        float g1 = s_g1[0];
        for (int k = 1; k < 8; ++k) g1 = fminf(g1, s_g1[k]);
        float cc[3], sc, U;
        tc_scale(a.box + b * 6, cc, sc, U);
        const float E = kTcErel * U * U;
        const float thr = g1 + (2.f * E + (fabsf(g1) + E) * (1.0f / 262144.0f));
        // ranges to scan
        for (int k = threadIdx.x; k < nsum; k += 256) {
            const float4 v = a.sums[dir][(int64_t)k * stride + g];
            const int cb = dir == 0 ? (int)((int64_t)k * a.ttiles / a.splits) * kTcRows : k * kTcQB;
            const int ce = dir == 0 ? (int)((int64_t)(k + 1) * a.ttiles / a.splits) * kTcRows : (k + 1) * kTcQB;
            const unsigned bb = __float_as_uint(v.w);
            if (v.z <= thr) {
                const unsigned r = atomicAdd(&s_nr, 1u);
                if (r < kTcFbRanges) s_rng[r] = make_int2(cb, min(ce, nT));
            } else {
                if (v.x <= thr) {
                    const unsigned r = atomicAdd(&s_nr, 1u);
                    const int c0 = cb + kTcChunk * (int)(bb & 0xffffu);
                    if (r < kTcFbRanges) s_rng[r] = make_int2(c0, min(c0 + kTcChunk, nT));
                }
                if (v.y <= thr) {
                    const unsigned r = atomicAdd(&s_nr, 1u);
                    const int c0 = cb + kTcChunk * (int)(bb >> 16);
                    if (r < kTcFbRanges) s_rng[r] = make_int2(c0, min(c0 + kTcChunk, nT));
                }
            }
        }
        __syncthreads();
        const unsigned nr = s_nr;
        const bool whole = nr > (unsigned)kTcFbRanges;
        float bd = INFINITY;
        int bi = 0x7fffffff;
        const unsigned nscan = whole ? 1u : nr;
        for (unsigned r = 0; r < nscan; ++r) {
            const int2 rg = whole ? make_int2(0, nT) : s_rng[r];
            CD_CHECK(rg.x >= 0 && rg.y <= nT);
            for (int j0 = rg.x; j0 < rg.y; j0 += 256 * 4) {
                float4 t[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) t[u] = T[min(j0 + 256 * u + (int)threadIdx.x, rg.y - 1)];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + 256 * u + (int)threadIdx.x;
                    const float d = dist_rn(q.x, q.y, q.z, t[u].x, t[u].y, t[u].z);
                    if (j < rg.y && (d < bd || (d == bd && j < bi))) {
                        bd = d;
                        bi = j;
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float od = __shfl_xor_sync(0xffffffffu, bd, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (od < bd || (od == bd && oi < bi)) {
                bd = od;
                bi = oi;
            }
        }
        if (lane == 0) {
            sd[warp] = bd;
            si[warp] = bi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < 8; ++k)
                if (sd[k] < bd || (sd[k] == bd && si[k] < bi)) {
                    bd = sd[k];
                    bi = si[k];
                }
            a.d_out[dir][g] = bd;
            a.idx_out[dir][g] = bi == 0x7fffffff ? -1 : bi;
        }
        __syncthreads();
    }
}

// per-chunk fp64 sums + hit counts of the final distances (fixed order)
struct TcChunkArgs {
    const float* d[2];
    int n[2], nchunks[2];
    int64_t chunk_off[2];
    int B;
    double* chunk_sum;
    int* chunk_hits;
    double tau2;
};

__global__ void __launch_bounds__(kMergeThreads) tc_chunks_kernel(TcChunkArgs a) {
    int u = blockIdx.x;
    int dir = 0;
    if (u >= a.B * a.nchunks[0]) {
        dir = 1;
        u -= a.B * a.nchunks[0];
    }
    const int b = u / a.nchunks[dir];
    const int chunk = u - b * a.nchunks[dir];
    const int i = chunk * kMergeThreads + threadIdx.x;
    double v = 0.0;
    int h = 0;
    if (i < a.n[dir]) {
        const float d = a.d[dir][(int64_t)b * a.n[dir] + i];
        v = (double)d;
        h = (a.tau2 >= 0.0 && (double)d <= a.tau2) ? 1 : 0;
    }
    __shared__ double ss[kMergeThreads / 32];
    __shared__ int sh[kMergeThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_down_sync(0xffffffffu, v, o);
        h += __shfl_down_sync(0xffffffffu, h, o);
    }
    if ((threadIdx.x & 31) == 0) {
        ss[threadIdx.x >> 5] = v;
        sh[threadIdx.x >> 5] = h;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        int t = 0;
        for (int w = 0; w < kMergeThreads / 32; ++w) {
            s += ss[w];
            t += sh[w];
        }
        const int64_t c = a.chunk_off[dir] + (int64_t)b * a.nchunks[dir] + chunk;
        a.chunk_sum[c] = s;
        a.chunk_hits[c] = t;
    }
}

// ------------------------------------------------------------------------------------------ host
static int tc_cdiv(int64_t x, int64_t y) { return (int)((x + y - 1) / y); }

static int tc_sms() { return current_sm_count(); }

void plan_tc(TcPlan& p, int B, int N, int M, int forced_splits) {
    p.B = B;
    p.npts[0] = N;
    p.npts[1] = M;
    p.ppad[0] = tc_cdiv(N, kTcQB) * kTcQB;
    p.ppad[1] = tc_cdiv(M, kTcRows) * kTcRows;
    p.qblocks = p.ppad[0] / kTcQB;
    p.ttiles = p.ppad[1] / kTcRows;
    // one CTA per SM (512 TMEM columns): split the targets so the units fill the SMs in near-whole waves
    const int64_t units = (int64_t)B * p.qblocks, slots = tc_sms();
    int best = 1;
    double bt = 1e300;
    for (int s = 1; s <= std::min(16, p.ttiles); ++s) {
        const double t = (double)tc_cdiv(units * s, slots) * ((double)tc_cdiv(p.ttiles, s) + 1.0);
        if (t < bt * 0.999) {
            bt = t;
            best = s;
        }
    }
    p.splits = forced_splits > 0 ? std::min(forced_splits, p.ttiles) : best;
    p.nchunks[0] = tc_cdiv(N, kMergeThreads);
    p.nchunks[1] = tc_cdiv(M, kMergeThreads);
    p.chunk_off[0] = 0;
    p.chunk_off[1] = (int64_t)B * p.nchunks[0];
    const int64_t chunks = p.chunk_off[1] + (int64_t)B * p.nchunks[1];
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    p.off_box = take((size_t)B * 6 * 4);
    for (int c = 0; c < 2; ++c) {
        p.off_pack[c] = take((size_t)B * p.ppad[c] * 16);
        p.off_op[c] = take((size_t)B * p.ppad[c] * 32);
    }
    p.off_rowsum = take((size_t)p.splits * B * N * 16);
    p.off_colsum = take((size_t)p.qblocks * B * M * 16);
    p.off_fb = take(256 + (size_t)B * ((int64_t)N + M) * 4);
    p.off_chunk_sum = take((size_t)chunks * 8);
    p.off_chunk_hits = take((size_t)chunks * 4);
    p.bytes = off;
}

int tc_launches(const TcPlan& p) { (void)p; return 7; }   // bbox, pack, main, resolve, fallback, chunks, partials

cudaError_t launch_tc(const TcPlan& p, const float* x, const float* y, const FwdOutputs& o, void* ws, cudaStream_t st) {
    char* w = static_cast<char*>(ws);
    const int sms = tc_sms();
    unsigned* box = reinterpret_cast<unsigned*>(w + p.off_box);
    cudaMemsetAsync(box, 0xff, (size_t)p.B * 6 * 4, st);   // identity of the atomicMin reductions
    float4* pack[2] = {reinterpret_cast<float4*>(w + p.off_pack[0]), reinterpret_cast<float4*>(w + p.off_pack[1])};
    unsigned char* op[2] = {reinterpret_cast<unsigned char*>(w + p.off_op[0]),
                            reinterpret_cast<unsigned char*>(w + p.off_op[1])};
    float4* rowsum = reinterpret_cast<float4*>(w + p.off_rowsum);
    float4* colsum = reinterpret_cast<float4*>(w + p.off_colsum);
    unsigned* fb_count = reinterpret_cast<unsigned*>(w + p.off_fb);
    unsigned* fb_list = fb_count + 64;
    {
        TcBoxArgs a{{x, y}, {p.npts[0], p.npts[1]}, p.B, box};
        tc_bbox_kernel<<<dim3(std::max(1, std::min(64, tc_cdiv((int64_t)p.npts[0] + p.npts[1], 4096))), p.B), 256, 0, st>>>(a);
    }
    {
        TcPackArgs a;
        a.src[0] = x;
        a.src[1] = y;
        for (int c = 0; c < 2; ++c) {
            a.npts[c] = p.npts[c];
            a.ppad[c] = p.ppad[c];
            a.pack[c] = pack[c];
            a.op[c] = op[c];
        }
        a.B = p.B;
        a.box = box;
        a.fb_count = fb_count;
        const int64_t total = (int64_t)p.B * (p.ppad[0] + p.ppad[1]);
        tc_pack_kernel<<<(int)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 16), 256, 0, st>>>(a);
    }
    {
        TcArgs a;
        a.op[0] = op[0];
        a.op[1] = op[1];
        for (int c = 0; c < 2; ++c) {
            a.npts[c] = p.npts[c];
            a.ppad[c] = p.ppad[c];
        }
        a.qblocks = p.qblocks;
        a.splits = p.splits;
        a.ttiles = p.ttiles;
        a.rowsum = rowsum;
        a.colsum = colsum;
        const size_t smem = (size_t)(kTcSub + kTcStages) * kTcTileBytes + 256 + (5 * kTcSub * 2 * kTcRows + 5 * kTcRows) * 4;
        ensure_smem_attr((const void*)nn_tc_kernel, (int)smem);
        if (g_prof_start) record_profile_event(g_prof_start, st);
        nn_tc_kernel<<<dim3(p.qblocks * p.splits, p.B), kTcThreads, smem, st>>>(a);
        if (g_prof_stop) record_profile_event(g_prof_stop, st);
    }
    TcResolveArgs ra;
    for (int c = 0; c < 2; ++c) {
        ra.pack[c] = pack[c];
        ra.npts[c] = p.npts[c];
        ra.ppad[c] = p.ppad[c];
        ra.d_out[c] = o.d[c];
        ra.idx_out[c] = o.idx[c];
    }
    ra.B = p.B;
    ra.box = box;
    ra.splits = p.splits;
    ra.ttiles = p.ttiles;
    ra.qblocks = p.qblocks;
    ra.sums[0] = rowsum;
    ra.sums[1] = colsum;
    ra.fb_count = fb_count;
    ra.fb_list = fb_list;
    {
        const int64_t L = (int64_t)p.B * ((int64_t)p.npts[0] + p.npts[1]);
        tc_resolve_kernel<<<(int)std::min<int64_t>((L + 255) / 256, (int64_t)sms * 16), 256, 0, st>>>(ra);
        tc_fallback_kernel<<<sms * 16, 256, 0, st>>>(ra);
#ifdef CD_TC_STATS
        unsigned h = 0;
        cudaStreamSynchronize(st);
        cudaMemcpy(&h, fb_count, 4, cudaMemcpyDeviceToHost);
        printf("tc fallback rows: %u of %lld\n", h, (long long)p.B * ((long long)p.npts[0] + p.npts[1]));
#endif
    }
    double* chunk_sum = reinterpret_cast<double*>(w + p.off_chunk_sum);
    int* chunk_hits = reinterpret_cast<int*>(w + p.off_chunk_hits);
    {
        TcChunkArgs a;
        for (int c = 0; c < 2; ++c) {
            a.d[c] = o.d[c];
            a.n[c] = p.npts[c];
            a.nchunks[c] = p.nchunks[c];
            a.chunk_off[c] = p.chunk_off[c];
        }
        a.B = p.B;
        a.chunk_sum = chunk_sum;
        a.chunk_hits = chunk_hits;
        a.tau2 = o.tau >= 0.f ? (double)o.tau * (double)o.tau : -1.0;
        tc_chunks_kernel<<<(unsigned)(p.B * (p.nchunks[0] + p.nchunks[1])), kMergeThreads, 0, st>>>(a);
    }
    if (o.partials) return launch_partials(chunk_sum, chunk_hits, p.nchunks, p.chunk_off, p.B, o.partials, 3, st);
    return cudaGetLastError();
}

}  // namespace cdk
