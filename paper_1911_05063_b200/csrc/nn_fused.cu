// nn_fused.cu — fused bidirectional forward (built into the hot path):
// every distance d(x_i, y_j) is evaluated ONCE and feeds both nearest-neighbour directions.
//
//   nn_fused_kernel   CTA = 2048 X rows (kR = 16 per thread, packed f32x2; 1024 rows / kRSmall = 8
//                     when the clouds are too small to fill the GPU with 2048-row tiles) x one split of Y
//                     (3-stage TMA bulk ring).  Row direction (x -> nearest y): value-only running
//                     min folded two targets per FMNMX3, argmin block tracked per kBlockK targets
//                     (as nn_fwd_kernel).  Column direction (y -> nearest x): per target, min over
//                     the thread's 16 rows (FMNMX3 tree), the warp minimum by one REDUX.MIN on the
//                     float bits (d >= 0: unsigned order is float order), and the lowest lane
//                     holding it by ballot; lane t keeps target t of each 32-target block.
//                     Per smem tile the 4 warps' results are combined in shared memory and one
//                     packed key (float bits << 32 | first row of the winning thread) per target
//                     goes to global memory with atomicMin (u64): the minimum key is the minimum
//                     distance with the lowest row group, independent of CTA order (deterministic).
//   nn_col_resolve_kernel  per Y row: unpack the key, re-evaluate the winning thread's 16 rows
//                     with the same .rn ops, keep the lowest row index with d == min (exact).
//
// (y - x)^2 == (x - y)^2 bit for bit in IEEE arithmetic (negation is exact), so the column
// distances equal a direct y -> x evaluation with the fixed op order of DESIGN.md §4.2.
#include "cd_device.cuh"
#include "cd_internal.h"

#include <algorithm>

namespace cdk {

#ifndef CD_FUSED_UNROLL
#define CD_FUSED_UNROLL 2
#endif
constexpr int kFusedUnroll = CD_FUSED_UNROLL;   // target pairs per inner-loop body

struct FusedArgs {
    const float4* xp;   // packed X (rows)
    const float4* yp;   // packed Y (targets / columns)
    int N, M, xpad, ypad;
    int q0, q1;         // X row slice
    int qtiles, splits, ttiles;
    int split_unit;       // targets per split unit: kTile or kBlockK
    int64_t slice_total;  // B * (q1 - q0)
    long long* rowkey;  // [B*(q1-q0)]: min over splits of (best bits << 32 | block start)
    long long* colkey;  // [B][M], non-negative keys; kColKeyEmpty = none
};

#ifndef CD_FUSED_MINB
#define CD_FUSED_MINB 3
#endif
template <bool kPartial, int R>   // kPartial: block-granular splits (partial tiles); R: rows per thread
__global__ void __launch_bounds__(kFwdThreads, CD_FUSED_MINB) nn_fused_kernel(FusedArgs a) {
    __shared__ __align__(128) float4 sm[kStages][kTile];
    __shared__ float colv[2][kFwdThreads / 32][kTile];
    __shared__ unsigned char coll[2][kFwdThreads / 32][kTile];
    __shared__ __align__(8) u64 full_bar[kStages];

    pdl_wait();
    const int b = blockIdx.y;
    const int tile = blockIdx.x / a.splits;
    const int split = blockIdx.x - tile * a.splits;
    const float4* __restrict__ Q = a.xp + (int64_t)b * a.xpad;
    const float4* __restrict__ T = a.yp + (int64_t)b * a.ypad;
    // split s covers the split units [s*nu/S, (s+1)*nu/S): 512-target tiles normally, 32-target
    // blocks when there are too few tiles to fill the GPU (small M; plan_forward)
    const int ulen = a.split_unit;                      // targets per split unit (512 or 32)
    const int nu = (a.M + ulen - 1) / ulen;
    const int j0 = (int)((int64_t)split * nu / a.splits) * ulen;
    const int j1b = (int)((int64_t)(split + 1) * nu / a.splits) * ulen;   // unit-aligned end (<= ppad)
    const int j1 = min(j1b, a.M);
    const int ntiles = (j1b - j0 + kTile - 1) / kTile;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int pre = min(kStages, ntiles);
        for (int k = 0; k < pre; ++k) {
            const uint32_t bytes = (uint32_t)min(kTile, j1b - (j0 + k * kTile)) * 16;
            mbar_arrive_expect_tx(&full_bar[k], bytes);
            tma_load_1d(sm[k], T + j0 + (int64_t)k * kTile, bytes, &full_bar[k]);
        }
    }

    const int qbase = a.q0 + tile * (kFwdThreads * R) + threadIdx.x * R;  // first row of this thread's group
    u64 qx[R / 2], qy[R / 2], qz[R / 2];
#pragma unroll
    for (int r = 0; r < R / 2; ++r) {
        // rows past the slice end duplicate the last row of the slice: same values, higher index,
        // so they never win a column and their row results are never stored
        const float4 p0 = Q[min(qbase + 2 * r, a.q1 - 1)];
        const float4 p1 = Q[min(qbase + 2 * r + 1, a.q1 - 1)];
        qx[r] = pk2(p0.x, p1.x);
        qy[r] = pk2(p0.y, p1.y);
        qz[r] = pk2(p0.z, p1.z);
    }
    float best[R];
    int blk[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        best[r] = INFINITY;
        blk[r] = -1;
    }

    for (int k = 0; k < ntiles; ++k) {
        const int s = k % kStages;
        mbar_wait(&full_bar[s], (k / kStages) & 1);
        const float4* tb = sm[s];
        float* cv = colv[k & 1][warp];
        unsigned char* cl = coll[k & 1][warp];
        const int jt = j0 + k * kTile;
        const int kend = min(kTile, j1b - jt);   // this tile's targets (a multiple of 32)
        for (int kb = 0; kb < kTile; kb += kBlockK) {
            if (kPartial && kb >= kend) break;   // partial last tile of a block-granular split
            static_assert(kBlockK == 32, "one column result per lane per block");
            float old[R];
#pragma unroll
            for (int r = 0; r < R; ++r) old[r] = best[r];
            unsigned keep_m = 0x7f800000u, keep_e = 0u;  // this lane's target (kb + lane) results
#pragma unroll kFusedUnroll
            for (int jj = 0; jj < kBlockK; jj += 2) {
                const float4 t0 = tb[kb + jj];
                const float4 t1 = tb[kb + jj + 1];
                const u64 t0x = pk2(t0.x, t0.x), t0y = pk2(t0.y, t0.y), t0z = pk2(t0.z, t0.z);
                const u64 t1x = pk2(t1.x, t1.x), t1y = pk2(t1.y, t1.y), t1z = pk2(t1.z, t1.z);
#ifndef CD_COLMIN_TREE
                float ca[2], cb[2];   // column partials: two FMNMX3 accumulators per target (depth 4)
#else
                float ca[R / 2], cb[R / 2];
#endif
#pragma unroll
                for (int r = 0; r < R / 2; ++r) {
                    u64 dx = sub2(qx[r], t0x), dy = sub2(qy[r], t0y), dz = sub2(qz[r], t0z);
                    u64 s0 = mul2(dx, dx);
                    s0 = fma2(dy, dy, s0);
                    s0 = fma2(dz, dz, s0);
                    dx = sub2(qx[r], t1x);
                    dy = sub2(qy[r], t1y);
                    dz = sub2(qz[r], t1z);
                    u64 s1 = mul2(dx, dx);
                    s1 = fma2(dy, dy, s1);
                    s1 = fma2(dz, dz, s1);
                    float a0, a1, b0, b1;
                    upk2(s0, a0, a1);
                    upk2(s1, b0, b1);
                    best[2 * r] = fmin3(best[2 * r], a0, b0);      // row mins
                    best[2 * r + 1] = fmin3(best[2 * r + 1], a1, b1);
#ifndef CD_COLMIN_TREE
                    if (r < 2) {
                        ca[r] = fminf(a0, a1);
                        cb[r] = fminf(b0, b1);
                    } else {
                        ca[r & 1] = fmin3(ca[r & 1], a0, a1);
                        cb[r & 1] = fmin3(cb[r & 1], b0, b1);
                    }
#else
                    ca[r] = fminf(a0, a1);                           // column partials (tree below)
                    cb[r] = fminf(b0, b1);
#endif
                }
#ifndef CD_COLMIN_TREE
                const float c0 = fminf(ca[0], ca[1]), c1 = fminf(cb[0], cb[1]);
#else
                // column min over this thread's 16 rows: FMNMX3 tree (depth 2 instead of a chain)
                const float c0 = fmin3(fmin3(ca[0], ca[1], ca[2]), fmin3(ca[3], ca[4], ca[5]), fminf(ca[6], ca[7]));
                const float c1 = fmin3(fmin3(cb[0], cb[1], cb[2]), fmin3(cb[3], cb[4], cb[5]), fminf(cb[6], cb[7]));
#endif
                // warp min (REDUX on the bits: d >= 0, so unsigned order == float order, NaN > inf)
                const unsigned u0 = __float_as_uint(c0), u1 = __float_as_uint(c1);
                const unsigned m0 = __reduce_min_sync(0xffffffffu, u0);
                const unsigned m1 = __reduce_min_sync(0xffffffffu, u1);
                const unsigned e0 = __ballot_sync(0xffffffffu, u0 == m0);  // lanes holding the min
                const unsigned e1 = __ballot_sync(0xffffffffu, u1 == m1);
                keep_m = lane == jj ? m0 : keep_m;
                keep_e = lane == jj ? e0 : keep_e;
                keep_m = lane == jj + 1 ? m1 : keep_m;
                keep_e = lane == jj + 1 ? e1 : keep_e;
            }
            cv[kb + lane] = __uint_as_float(keep_m);
            cl[kb + lane] = (unsigned char)(__ffs(keep_e) - 1);  // lowest lane; 255 if none (NaN)
#pragma unroll
            for (int r = 0; r < R; ++r) blk[r] = best[r] < old[r] ? jt + kb : blk[r];
        }
        __syncthreads();  // every warp is done with stage s and has written colv[k & 1]
        if (threadIdx.x == 0 && k + kStages < ntiles) {
            const int jn = jt + kStages * kTile;
            const uint32_t bytes = (uint32_t)min(kTile, j1b - jn) * 16;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[s], bytes);
            tma_load_1d(sm[s], T + jn, bytes, &full_bar[s]);
        }
        // combine the 4 warps per target and publish one key per (CTA, target)
        for (int t = threadIdx.x; t < kTile; t += kFwdThreads) {
            const int j = jt + t;
            if (j >= j1) break;
            float m = colv[k & 1][0][t];
            int w = 0;
#pragma unroll
            for (int ww = 1; ww < kFwdThreads / 32; ++ww) {
                const float v = colv[k & 1][ww][t];
                if (v < m || m != m) {  // strict <: the lowest warp keeps ties (NaN never wins)
                    m = v;
                    w = ww;
                }
            }
            const unsigned l = coll[k & 1][w][t];
            if (l < 32u) {
                const unsigned row0 = (unsigned)(a.q0 + tile * (kFwdThreads * R) + (w * 32 + (int)l) * R);
                const long long key = (long long)(((unsigned long long)__float_as_uint(m) << 32) | row0);
                atomicMin(&a.colkey[(int64_t)b * a.M + j], key);  // keys >= 0: signed min == lexicographic
            }
        }
    }

    const int slen = a.q1 - a.q0;
    const int64_t rowbase = (int64_t)b * slen;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int q = qbase + r;
        if (q < a.q1) atomicMin(&a.rowkey[rowbase + (q - a.q0)], row_key(best[r], blk[r]));
    }
}

// ------------------------------------------------------------------------------------------------
// ------------------------------------------------------------------------------------------------
int fused_ctas_per_sm(int rows) {
    static std::atomic<int> big[kMaxDevices], small[kMaxDevices];
    return rows == kR ? occupancy_of(big, nn_fused_kernel<false, kR>, kFwdThreads, 0, 3)
                      : occupancy_of(small, nn_fused_kernel<false, kRSmall>, kFwdThreads, 0, 3);
}

cudaError_t launch_fused_rows(const FwdPlan& p, const float4* xp, const float4* yp, long long* colkey,
                              long long* rowkey, cudaStream_t st) {
    FusedArgs a;
    a.xp = xp;
    a.yp = yp;
    a.N = p.npts[0];
    a.M = p.npts[1];
    a.xpad = p.ppad[0];
    a.ypad = p.ppad[1];
    a.q0 = p.qlo[0];
    a.q1 = p.qhi[0];
    a.qtiles = p.qtiles[0];
    a.splits = p.splits[0];
    a.ttiles = p.ttiles[0];
    a.split_unit = p.split_unit;
    a.slice_total = p.slice_total;
    a.rowkey = rowkey;
    a.colkey = colkey;
    const int gx = p.qtiles[0] * p.splits[0];
    if (gx > 0) {
        if (g_prof_start) record_profile_event(g_prof_start, st);
        const dim3 grid(gx, p.B);
        if (p.fused_rows == kR) {
            if (p.split_unit == kTile)
                launch_pdl(nn_fused_kernel<false, kR>, grid, dim3(kFwdThreads), 0, st, a);
            else
                launch_pdl(nn_fused_kernel<true, kR>, grid, dim3(kFwdThreads), 0, st, a);
        } else {   // small clouds: 1024-row query tiles (twice the CTAs per batch element)
            if (p.split_unit == kTile)
                launch_pdl(nn_fused_kernel<false, kRSmall>, grid, dim3(kFwdThreads), 0, st, a);
            else
                launch_pdl(nn_fused_kernel<true, kRSmall>, grid, dim3(kFwdThreads), 0, st, a);
        }
        if (g_prof_stop) record_profile_event(g_prof_stop, st);
    }
    return cudaGetLastError();
}

}  // namespace cdk
