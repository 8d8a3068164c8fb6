// nn_forward.cu — forward of the batched exact nearest-neighbour search.
//
// Kernels (one launch each, on the caller's stream):
//   pack_kernel      AoS (x,y,z) fp32 clouds -> padded float4 clouds in the workspace (a.1); also
//                    resets the 64-bit row / column keys to the identity of min.
//   nn_fused_kernel  (nn_fused.cu) the default hot loop for full problems: both directions from one
//                    evaluation of every distance.
//   nn_fwd_kernel    the per-direction hot loop (query slices; a.2 + a.3, both directions in one
//                    grid): every thread keeps kR = 16 queries in packed f32x2 registers and sweeps
//                    the targets of its split, staged through a 3-stage shared-memory ring by 1-D TMA
//                    bulk copies (cp.async.bulk + mbarrier).  Distances use FADD2/FMUL2/FFMA2 with
//                    the target coordinate as broadcast operand; the running minimum is value-only
//                    (FMNMX3 folding two targets per op) and the argmin is tracked per block of kBlockK
//                    targets (the block where the minimum last strictly decreased).  Splits merge with
//                    a 64-bit atomicMin on (distance bits << 32 | block start): order-independent.
//   nn_epilogue_kernel  one launch for both directions' epilogues (a.4): row blocks re-scan the
//                    winning 32-target block with the same .rn ops (exact lowest index), column blocks
//                    re-scan the winning 16-row group of the fused kernel's column keys; d / idx
//                    stores and per-chunk fp64 sums + hit counts.
//   partials_kernel  fixed-order reduction of the chunk partials into partials[B][4] (a.4/a.5).
// plus finalize_kernel (cd_finalize, a.5) and the cd_fscore path (stats_kernel).
#include "cd_device.cuh"
#include "cd_internal.h"

#include <algorithm>
#include <cmath>

namespace cdk {

thread_local cudaEvent_t g_prof_start = nullptr;
thread_local cudaEvent_t g_prof_stop = nullptr;

// ------------------------------------------------------------------------------------------------
struct PackArgs {
    const float* src[2];
    float4* dst[2];
    int npts[2];
    int ppad[2];
    int vec[2];          // cloud c packs 4 points per thread (n % 4 == 0, 16-B aligned source)
    int B;
    long long* colkey;   // optional: column keys to reset to the identity of min (fused modes)
    int64_t ncolkey;
    long long* rowkey;   // row keys (min over target splits) to reset
    int64_t nrowkey;
};

// grid (x: point blocks of one row, y: batch element, z: cloud) — no per-element division; the key
// resets are spread over the whole grid
#ifndef CD_PACK_VEC
#define CD_PACK_VEC 1
#endif
__global__ void __launch_bounds__(256) pack_kernel(PackArgs a) {
    pdl_wait();
    const int c = blockIdx.z, b = blockIdx.y;
    const int n = a.npts[c], pad = a.ppad[c];
    const float* __restrict__ src = a.src[c] + (int64_t)b * n * 3;
    float4* __restrict__ dst = a.dst[c] + (int64_t)b * pad;
    // padding targets: +inf coordinates give d = +inf, never selected by min / strict <
    const float4 inf4 = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
    if (a.vec[c]) {
        // 4 points per thread: three 16-B loads (48 B = 4 AoS points; n % 4 == 0 and a 16-B aligned
        // cloud, so every group is whole and aligned), four float4 stores; pad % 4 == 0
        const float4* __restrict__ s4 = reinterpret_cast<const float4*>(src);
        for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < pad / 4; g += gridDim.x * blockDim.x) {
            float4 o0 = inf4, o1 = inf4, o2 = inf4, o3 = inf4;
            if (4 * g < n) {
                const float4 u = __ldg(s4 + 3 * g), v = __ldg(s4 + 3 * g + 1), w = __ldg(s4 + 3 * g + 2);
                o0 = make_float4(u.x, u.y, u.z, 0.f);
                o1 = make_float4(u.w, v.x, v.y, 0.f);
                o2 = make_float4(v.z, v.w, w.x, 0.f);
                o3 = make_float4(w.y, w.z, w.w, 0.f);
            }
            dst[4 * g] = o0;
            dst[4 * g + 1] = o1;
            dst[4 * g + 2] = o2;
            dst[4 * g + 3] = o3;
        }
    } else {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pad; i += gridDim.x * blockDim.x) {
            float4 v = inf4;
            if (i < n) v = make_float4(__ldg(src + 3 * i), __ldg(src + 3 * i + 1), __ldg(src + 3 * i + 2), 0.f);
            dst[i] = v;
        }
    }
    const int64_t nthreads = (int64_t)gridDim.x * gridDim.y * gridDim.z * blockDim.x;
    const int64_t tid = (((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * blockDim.x +
                        threadIdx.x;
    for (int64_t e = tid; e < a.ncolkey; e += nthreads) a.colkey[e] = kColKeyEmpty;
    for (int64_t e = tid; e < a.nrowkey; e += nthreads) a.rowkey[e] = kColKeyEmpty;
}

// ------------------------------------------------------------------------------------------------
struct FwdArgs {
    const float4* pack[2];
    int npts[2], ppad[2];
    int qlo[2], qhi[2];
    int qtiles[2], splits[2], ttiles[2];
    int64_t slice_off[2], slice_total;
    long long* rowkey;   // [slice_total]: min over splits of (best bits << 32 | block start)
};

__global__ void __launch_bounds__(kFwdThreads, 4) nn_fwd_kernel(FwdArgs a) {
    __shared__ __align__(128) float4 sm[kStages][kTile];
    __shared__ __align__(8) u64 full_bar[kStages];

    int u = blockIdx.x;
    const int b = blockIdx.y;
    int dir = 0;
    const int units0 = a.qtiles[0] * a.splits[0];
    if (u >= units0) {
        dir = 1;
        u -= units0;
    }
    const int tile = u / a.splits[dir];
    const int split = u - tile * a.splits[dir];
    const int tdir = 1 - dir;
    const float4* __restrict__ Q = a.pack[dir] + (int64_t)b * a.ppad[dir];
    const float4* __restrict__ T = a.pack[tdir] + (int64_t)b * a.ppad[tdir];
    const int nq = a.npts[dir];
    const int nt = a.npts[tdir];
    // split s covers target tiles [s*T/S, (s+1)*T/S): equal work up to one tile
    const int j0 = (int)((int64_t)split * a.ttiles[dir] / a.splits[dir]) * kTile;
    const int j1 = min((int)((int64_t)(split + 1) * a.ttiles[dir] / a.splits[dir]) * kTile, nt);
    const int ntiles = (j1 - j0 + kTile - 1) / kTile;  // >= 1 (host guarantees non-empty splits)

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int pre = min(kStages, ntiles);
        for (int k = 0; k < pre; ++k) {
            mbar_arrive_expect_tx(&full_bar[k], kTile * 16);
            tma_load_1d(sm[k], T + j0 + (int64_t)k * kTile, kTile * 16, &full_bar[k]);
        }
    }

    // queries: kR consecutive points per thread, packed in pairs (r, r+1) -> one f32x2 register
    const int qbase = a.qlo[dir] + tile * kQTile + threadIdx.x * kR;
    u64 qx[kR / 2], qy[kR / 2], qz[kR / 2];
#pragma unroll
    for (int r = 0; r < kR / 2; ++r) {
        const float4 p0 = Q[min(qbase + 2 * r, nq - 1)];
        const float4 p1 = Q[min(qbase + 2 * r + 1, nq - 1)];
        qx[r] = pk2(p0.x, p1.x);
        qy[r] = pk2(p0.y, p1.y);
        qz[r] = pk2(p0.z, p1.z);
    }
    float best[kR];
    int blk[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        best[r] = INFINITY;
        blk[r] = -1;
    }

    for (int k = 0; k < ntiles; ++k) {
        const int s = k % kStages;
        mbar_wait(&full_bar[s], (k / kStages) & 1);
        const float4* tb = sm[s];
        const int jt = j0 + k * kTile;
        for (int kb = 0; kb < kTile; kb += kBlockK) {
            float old[kR];
#pragma unroll
            for (int r = 0; r < kR; ++r) old[r] = best[r];
#pragma unroll 2
            for (int jj = 0; jj < kBlockK; jj += 2) {
                const float4 t0 = tb[kb + jj];
                const float4 t1 = tb[kb + jj + 1];
                const u64 t0x = pk2(t0.x, t0.x), t0y = pk2(t0.y, t0.y), t0z = pk2(t0.z, t0.z);
                const u64 t1x = pk2(t1.x, t1.x), t1y = pk2(t1.y, t1.y), t1z = pk2(t1.z, t1.z);
#pragma unroll
                for (int r = 0; r < kR / 2; ++r) {
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
                    float a0, a1, c0, c1;
                    upk2(s0, a0, a1);
                    upk2(s1, c0, c1);
                    best[2 * r] = fmin3(best[2 * r], a0, c0);
                    best[2 * r + 1] = fmin3(best[2 * r + 1], a1, c1);
                }
            }
#pragma unroll
            for (int r = 0; r < kR; ++r) blk[r] = best[r] < old[r] ? jt + kb : blk[r];
        }
        __syncthreads();  // every warp is done with stage s
        if (threadIdx.x == 0 && k + kStages < ntiles) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[s], kTile * 16);
            tma_load_1d(sm[s], T + jt + (int64_t)kStages * kTile, kTile * 16, &full_bar[s]);
        }
    }

    const int qhi = a.qhi[dir];
    const int slen = qhi - a.qlo[dir];
    const int64_t rowbase = a.slice_off[dir] + (int64_t)b * slen;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        const int q = qbase + r;
        if (q < qhi) atomicMin(&a.rowkey[rowbase + (q - a.qlo[dir])], row_key(best[r], blk[r]));
    }
}

// ------------------------------------------------------------------------------------------------
// Fixed-order block reduction of (fp64 sum, int hits) over kMergeThreads threads.
__device__ __forceinline__ void block_sum_hits(double v, int h, double* out_sum, int* out_hits) {
    __shared__ double ssum[kMergeThreads / 32];
    __shared__ int shit[kMergeThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_down_sync(0xffffffffu, v, o);
        h += __shfl_down_sync(0xffffffffu, h, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        ssum[w] = v;
        shit[w] = h;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        int t = 0;
        for (int i = 0; i < kMergeThreads / 32; ++i) {
            s += ssum[i];
            t += shit[i];
        }
        *out_sum = s;
        *out_hits = t;
    }
}

struct MergeArgs {
    const float4* pack[2];
    int npts[2];
    int ppad[2];
    int qlo[2], qhi[2];
    int splits[2];
    int64_t slice_off[2], slice_total;
    int nchunks[2];
    int64_t chunk_off[2];
    int B;
    const long long* rowkey;   // [slice_total] merged (over splits) row keys
    float* d_out[2];
    int32_t* idx_out[2];
    double* chunk_sum;
    int* chunk_hits;
    double tau2;  // < 0: no hits
};

// Row direction: per query row, unpack the merged key and find the lowest index inside the winning
// 32-target block with d == min (same .rn ops as the kernel).  Warp-cooperative: the warp walks its
// rows four at a time; for each, the 32 lanes load the block's 32 targets (one coalesced 512-B
// read) and a ballot picks the first match.
__device__ __forceinline__ void row_merge_block(const MergeArgs& a, int blk) {
    int u = blk;
    int dir = 0;
    if (u >= a.B * a.nchunks[0]) {
        dir = 1;
        u -= a.B * a.nchunks[0];
    }
    const int b = u / a.nchunks[dir];
    const int chunk = u - b * a.nchunks[dir];
    const int slen = a.qhi[dir] - a.qlo[dir];
    const int sq = chunk * kMergeThreads + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool valid = sq < slen;
    float best = INFINITY;
    int bb = -1;
    float4 qp = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
        // the atomicMin over splits kept the smallest distance, then the lowest block start
        const unsigned long long key = (unsigned long long)a.rowkey[a.slice_off[dir] + (int64_t)b * slen + sq];
        best = __uint_as_float((unsigned)(key >> 32));
        bb = (int)(unsigned)(key & 0xffffffffull);   // 0xffffffff -> -1: no finite distance
        if (bb >= 0) qp = a.pack[dir][(int64_t)b * a.ppad[dir] + a.qlo[dir] + sq];
    }
    const int tdir = 1 - dir;
    const float4* T = a.pack[tdir] + (int64_t)b * a.ppad[tdir];
    asm("" : "+l"(T));   // one opaque base pointer: each gather address is a single IMAD.WIDE.U32
    CD_CHECK(bb < 0 || (bb < a.npts[tdir] && bb % kBlockK == 0));
    // the warp's 32 rows staged in shared memory: (query, minimum) and block start, read back as
    // warp-wide broadcasts; targets past the cloud are the +inf padding (bb + 31 < ppad)
    __shared__ float4 s_q[kMergeThreads];
    __shared__ int s_b[kMergeThreads];
    s_q[threadIdx.x] = make_float4(qp.x, qp.y, qp.z, best);
    s_b[threadIdx.x] = bb;
    __syncwarp();
    const int wb = threadIdx.x & ~31;
    unsigned myc = 32u;   // this lane's row: the lowest matching lane of its block (32: none)
    constexpr int kRowsInFlight = 8;
    for (int r0 = 0; r0 < 32; r0 += kRowsInFlight) {
        int base[kRowsInFlight];
        float4 t[kRowsInFlight];
#pragma unroll
        for (int k = 0; k < kRowsInFlight; ++k) {
            base[k] = s_b[wb + r0 + k];
            t[k] = __ldg(T + (unsigned)(max(base[k], 0) + lane));   // 32-bit index: one IMAD.WIDE per address
        }
#pragma unroll
        for (int k = 0; k < kRowsInFlight; ++k) {
            const float4 q = s_q[wb + r0 + k];
            const float d = dist_rn(q.x, q.y, q.z, t[k].x, t[k].y, t[k].z);
            const unsigned c = __reduce_min_sync(0xffffffffu, d == q.w ? (unsigned)lane : 32u);
            myc = lane == r0 + k ? c : myc;
        }
    }
    const int idx = (bb >= 0 && myc < 32u) ? bb + (int)myc : -1;
    double v = 0.0;
    int h = 0;
    if (valid) {
        a.d_out[dir][(int64_t)b * slen + sq] = best;
        a.idx_out[dir][(int64_t)b * slen + sq] = idx;
        v = (double)best;
        h = (a.tau2 >= 0.0 && (double)best <= a.tau2) ? 1 : 0;
    }
    double s;
    int t;
    block_sum_hits(v, h, &s, &t);
    if (threadIdx.x == 0) {
        const int64_t c = a.chunk_off[dir] + (int64_t)b * a.nchunks[dir] + chunk;
        a.chunk_sum[c] = s;
        a.chunk_hits[c] = t;
    }
}

struct ResolveArgs {
    const float4* xp;
    const float4* yp;
    int N, M, xpad, ypad;
    int q0, q1;            // X rows that took part in the column minima
    int r0, r1;            // Y rows to resolve
    int B, nchunks;
    const long long* colkey;
    const long long* colkey_peers[kMaxPeers];   // npeers > 0: key = MIN over these arrays (peer reads)
    int npeers;
    float* d_out;          // [B][r1-r0]
    int32_t* idx_out;
    double* chunk_sum;     // dir-1 chunk partials
    int* chunk_hits;
    double tau2;
};

// column direction of the fused forward: per Y row, unpack the key and re-evaluate the winning
// thread's 16 rows with the same .rn ops (lowest index with d == min); `blk` = this CTA's chunk.
// Warp-cooperative: two columns per step, each half-warp loading one column's 16 rows (coalesced).
__device__ __forceinline__ void col_resolve_block(const ResolveArgs& a, int blk) {
    const int b = blk / a.nchunks;
    const int chunk = blk - b * a.nchunks;
    const int slen = a.r1 - a.r0;
    const int sj = chunk * kMergeThreads + threadIdx.x;
    const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
    float m = INFINITY;
    int i0 = -1;
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    if (sj < slen) {
        const int j = a.r0 + sj;
        long long kk;
        if (a.npeers > 0) {
            // the fused all-reduce: this column's keys from every rank's array (peer loads over
            // NVLink), MIN on read — only the resolved slice's keys cross the fabric
            kk = __ldcv(a.colkey_peers[0] + (int64_t)b * a.M + j);
            for (int q = 1; q < a.npeers; ++q) kk = min(kk, __ldcv(a.colkey_peers[q] + (int64_t)b * a.M + j));
        } else {
            kk = a.colkey[(int64_t)b * a.M + j];
        }
        const unsigned long long key = (unsigned long long)kk;
        // a +inf minimum is no finite candidate (R6): (+inf, -1) like the row direction
        if ((long long)key != kColKeyEmpty && __uint_as_float((unsigned)(key >> 32)) < INFINITY) {
            m = __uint_as_float((unsigned)(key >> 32));
            i0 = (int)(unsigned)(key & 0xffffffffull);
            CD_CHECK(i0 >= a.q0 && i0 < a.q1);
            t = a.yp[(int64_t)b * a.ypad + j];
        }
    }
    const float4* X = a.xp + (int64_t)b * a.xpad;
    asm("" : "+l"(X));   // one opaque base pointer (as in the row merge)
    static_assert(kR == 16, "the column resolve re-scans 16-row groups with half-warps");
    // the warp's 32 columns staged in shared memory: (target, minimum) and group start
    __shared__ float4 sc[kMergeThreads];
    __shared__ int si[kMergeThreads];
    sc[threadIdx.x] = make_float4(t.x, t.y, t.z, m);
    si[threadIdx.x] = i0;
    __syncwarp();
    const int wb = threadIdx.x & ~31;
    unsigned myc = 16u;   // this lane's column: the lowest matching row of its group (16: none)
    constexpr int kStepsInFlight = 4;   // steps of two columns (one per half-warp) in flight
    for (int r0 = 0; r0 < 32; r0 += 2 * kStepsInFlight) {
        int g[kStepsInFlight];
        float4 q[kStepsInFlight];
#pragma unroll
        for (int k = 0; k < kStepsInFlight; ++k) {
            g[k] = si[wb + r0 + 2 * k + half];
            q[k] = __ldg(X + (unsigned)min(max(g[k], 0) + hl, max(a.q1 - 1, 0)));   // past the slice end: row q1 - 1
        }
#pragma unroll
        for (int k = 0; k < kStepsInFlight; ++k) {
            const float4 c = sc[wb + r0 + 2 * k + half];
            const float d = dist_rn(q[k].x, q[k].y, q[k].z, c.x, c.y, c.z);  // same operand order as the kernel
            const unsigned v = (g[k] + hl < a.q1 && d == c.w) ? (unsigned)hl : 16u;
            const unsigned c0 = __reduce_min_sync(0xffffffffu, half == 0 ? v : 16u);
            const unsigned c1 = __reduce_min_sync(0xffffffffu, half == 1 ? v : 16u);
            myc = lane == r0 + 2 * k ? c0 : (lane == r0 + 2 * k + 1 ? c1 : myc);
        }
    }
    int idx = (i0 >= 0 && myc < 16u) ? i0 + (int)myc : -1;
    if (idx < 0) m = INFINITY;  // no finite candidate, or every distance was NaN
    double v = 0.0;
    int h = 0;
    if (sj < slen) {
        a.d_out[(int64_t)b * slen + sj] = m;
        a.idx_out[(int64_t)b * slen + sj] = idx;
        v = (double)m;
        h = (a.tau2 >= 0.0 && (double)m <= a.tau2) ? 1 : 0;
    }
    double s;
    int hs;
    block_sum_hits(v, h, &s, &hs);
    if (threadIdx.x == 0) {
        a.chunk_sum[(int64_t)b * a.nchunks + chunk] = s;
        a.chunk_hits[(int64_t)b * a.nchunks + chunk] = hs;
    }
}

// ------------------------------------------------------------------------------------------------

// a.4 epilogue of the forward in ONE launch: blocks [0, merge_blocks) merge the row splits, the rest
// resolve the fused kernel's column keys (independent work, so the two overlap on the GPU).
__global__ void __launch_bounds__(kMergeThreads) nn_epilogue_kernel(MergeArgs m, ResolveArgs r, int merge_blocks) {
    pdl_wait();
    if ((int)blockIdx.x < merge_blocks)
        row_merge_block(m, blockIdx.x);
    else
        col_resolve_block(r, blockIdx.x - merge_blocks);
}

// Per-chunk stats of given distance arrays (cd_fscore path).
struct StatsArgs {
    const float* d[2];
    int n[2];
    int nchunks[2];
    int64_t chunk_off[2];
    int B;
    double* chunk_sum;
    int* chunk_hits;
    double tau2;
};

__global__ void __launch_bounds__(kMergeThreads) stats_kernel(StatsArgs a) {
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
        h = (double)d <= a.tau2 ? 1 : 0;
    }
    double s;
    int t;
    block_sum_hits(v, h, &s, &t);
    if (threadIdx.x == 0) {
        const int64_t c = a.chunk_off[dir] + (int64_t)b * a.nchunks[dir] + chunk;
        a.chunk_sum[c] = s;
        a.chunk_hits[c] = t;
    }
}

// partials[b][0..3] = (sum d_xy, sum d_yx, hits_xy, hits_yx), fixed-order reduction over chunks.
struct PartialsArgs {
    const double* chunk_sum;
    const int* chunk_hits;
    int nchunks[2];
    int64_t chunk_off[2];
    double* partials;
    int dirmask;   // bit d set: write partials[b][d] and partials[b][2+d]
};

__global__ void __launch_bounds__(256) partials_kernel(PartialsArgs a) {
    pdl_wait();
    __shared__ double ssum[256];
    __shared__ long long shit[256];
    const int b = blockIdx.x;
    for (int dir = 0; dir < 2; ++dir) {
        if (!((a.dirmask >> dir) & 1)) continue;
        double s = 0.0;
        long long h = 0;
        const int64_t base = a.chunk_off[dir] + (int64_t)b * a.nchunks[dir];
        for (int c = threadIdx.x; c < a.nchunks[dir]; c += 256) {
            s += a.chunk_sum[base + c];
            h += a.chunk_hits[base + c];
        }
        ssum[threadIdx.x] = s;
        shit[threadIdx.x] = h;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) {
                ssum[threadIdx.x] += ssum[threadIdx.x + w];
                shit[threadIdx.x] += shit[threadIdx.x + w];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            a.partials[b * 4 + dir] = ssum[0];
            a.partials[b * 4 + 2 + dir] = (double)shit[0];
        }
        __syncthreads();
    }
}

// cd_finalize: CD_b, loss, P/R/F from partials (fp64 internally, fp32 outputs).
struct FinalizeArgs {
    const double* partials;
    int B, N, M;
    double w1, w2;
    float *cd, *loss, *fscore, *precision, *recall;
};

__global__ void __launch_bounds__(256) finalize_kernel(FinalizeArgs a) {
    pdl_wait();
    __shared__ double sl[256];
    double acc = 0.0;
    for (int b = threadIdx.x; b < a.B; b += 256) {
        const double* p = a.partials + 4 * b;
        const double cdb = a.w1 * (p[0] / a.N) + a.w2 * (p[1] / a.M);
        acc += cdb;
        if (a.cd) a.cd[b] = (float)cdb;
        const double P = p[2] / a.N, R = p[3] / a.M;
        const double F = (P + R) > 0.0 ? 2.0 * P * R / (P + R) : 0.0;
        if (a.fscore) a.fscore[b] = (float)F;
        if (a.precision) a.precision[b] = (float)P;
        if (a.recall) a.recall[b] = (float)R;
    }
    sl[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sl[threadIdx.x] += sl[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0 && a.loss) a.loss[0] = (float)(sl[0] / a.B);
}

// ------------------------------------------------------------------------------------------------
// Host side.
static int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

static int device_sm_count() { return current_sm_count(); }

// Choose the target-split count S so that (query-tile units x S) CTAs fill the SMs in waves of
// near-equal work: minimise ceil(U*S / slots) * (Mt/S + c0), c0 = per-unit overhead in target-
// equivalents (query load + epilogue).
int unfused_ctas_per_sm() {
    static std::atomic<int> table[kMaxDevices];
    return occupancy_of(table, nn_fwd_kernel, kFwdThreads, 0, 4);
}

// Choose the target-split count S: every (query tile, split) is one CTA; split s covers target
// tiles [s*T/S, (s+1)*T/S).  Minimise waves(U*S) * (ceil(T/S) + c0), with c0 = per-CTA overhead
// in tile units, and prefer at least one full wave of CTAs (a partly filled SM is latency-bound).
static int choose_splits(int64_t units, int ttiles, int ctas_per_sm) {
    const int64_t slots = (int64_t)device_sm_count() * ctas_per_sm;
    const double c0 = 0.25;
    const int smax = std::max(1, std::min(64, ttiles));
    int best_s = 1;
    double best_t = 1e300;
    for (int s = 1; s <= smax; ++s) {
        const int64_t ctas = units * s;
        const double waves = (double)ceil_div(ctas, slots);
        double t = waves * ((double)ceil_div(ttiles, s) + c0);
        if (ctas < slots && s < smax) t *= 1.15;  // under one wave: idle SM slots
        if (t < best_t * 0.999) {
            best_t = t;
            best_s = s;
        }
    }
    return best_s;
}

// Fused kernel, whole 512-target tiles per split: t(S) = U (T + S c0) / slots + (ceil(T/S) + c0) / 2 —
// the work spread over all CTA slots plus half a CTA of tail — with c0 = 0.1 tile of per-CTA cost.
// Fitted to forced-split sweeps (tools/sweep_splits.py): c3 best S = 16 (1.897 ms vs 1.903 at S = 8,
// the ceil-wave model's choice), c4 best S = 32 (17.47 vs 17.60 ms).
static int choose_splits_fused(int64_t units, int ttiles, int ctas_per_sm) {
    const double slots = (double)device_sm_count() * ctas_per_sm;
    const double c0 = 0.1;
    const int smax = std::max(1, std::min(64, ttiles));
    int best_s = 1;
    double best_t = 1e300;
    for (int s = 1; s <= smax; ++s) {
        const double t = (double)units * (ttiles + s * c0) / slots + 0.5 * ((double)ceil_div(ttiles, s) + c0);
        if (t < best_t * 0.999) {
            best_t = t;
            best_s = s;
        }
    }
    return best_s;
}

// Block-granular version for the fused kernel: a CTA's work is ceil(nb/S) 32-target blocks (plus a
// fixed overhead of ~4 tiles' worth: the 2048-row load, the per-tile column combine, the row keys).
static int choose_splits_blocks(int64_t units, int nb, int ctas_per_sm) {
    const int64_t slots = (int64_t)device_sm_count() * ctas_per_sm;
    const double c0 = 4.0;   // in blocks
    const int smax = std::max(1, std::min(128, nb));
    int best_s = 1;
    double best_t = 1e300;
    for (int s = 1; s <= smax; ++s) {
        const int64_t ctas = units * s;
        const double waves = (double)ceil_div(ctas, slots);
        double t = waves * ((double)ceil_div(nb, s) + c0);
        if (ctas < slots && s < smax) t *= 1.15;
        if (t < best_t * 0.999) {
            best_t = t;
            best_s = s;
        }
    }
    return best_s;
}

#ifndef CD_FUSED_SMALL
#define CD_FUSED_SMALL 1
#endif
#ifndef CD_SPLITS_FUSED_MODEL
#define CD_SPLITS_FUSED_MODEL 1
#endif

void plan_forward(FwdPlan& p, int mode, int B, int N, int M, int q0, int q1, int r0, int r1, int forced_splits) {
    if (mode == kTensor) {   // full problems only (q = [0,N), r = [0,M)); the tensor plan carves its own workspace
        plan_forward(p, kFusedFull, B, N, M, q0, q1, r0, r1, forced_splits);
        TcPlan t;
        plan_tc(t, B, N, M, forced_splits);
        p.mode = kTensor;
        p.bytes = t.bytes;
        p.forced_splits = forced_splits;
        return;
    }
    p.mode = mode;
    p.forced_splits = forced_splits;
    p.split_unit = kTile;
    p.B = B;
    p.npts[0] = N;
    p.npts[1] = M;
    p.qlo[0] = q0;
    p.qhi[0] = q1;
    p.qlo[1] = r0;
    p.qhi[1] = r1;
    int64_t units = 0;
    for (int d = 0; d < 2; ++d) {
        p.ppad[d] = ceil_div(p.npts[d], kPad) * kPad;
        const int slen = p.qhi[d] - p.qlo[d];
        p.qtiles[d] = slen > 0 ? ceil_div(slen, kQTile) : 0;
        if (mode != kUnfused && d == 1) p.qtiles[d] = 0;  // dir 1 comes from the column keys
        units += (int64_t)B * p.qtiles[d];
    }
    p.fused_rows = kR;
    if (CD_FUSED_SMALL && mode != kUnfused && p.qtiles[0] > 0 && (int64_t)B * p.qtiles[0] < device_sm_count()) {
        // fewer 2048-row units than SMs: 1024-row query tiles (the per-CTA fixed cost — query load,
        // per-tile column combine, row keys — over half the rows, twice the units to spread)
        p.fused_rows = kRSmall;
        units -= (int64_t)B * p.qtiles[0];
        p.qtiles[0] = ceil_div(p.qhi[0] - p.qlo[0], kFwdThreads * kRSmall);
        units += (int64_t)B * p.qtiles[0];
    }
    const int occ = mode == kUnfused ? unfused_ctas_per_sm() : fused_ctas_per_sm(p.fused_rows);
    if (mode == kUnfused) {
        const int S = forced_splits > 0 ? forced_splits : choose_splits(units, ceil_div(std::max(N, M), kTile), occ);
        for (int d = 0; d < 2; ++d) {
            p.ttiles[d] = ceil_div(p.npts[1 - d], kTile);
            p.splits[d] = std::max(1, std::min(S, p.ttiles[d]));  // <= T: every split non-empty
            if (p.qtiles[d] == 0) p.splits[d] = 1;
        }
    } else {
        // the fused kernel splits the targets in 512-target tiles, or in 32-target blocks when even
        // one tile per CTA cannot fill the GPU (small M, e.g. c2: 4 tiles per batch element)
        const int tt = ceil_div(M, kTile), nb = ceil_div(M, kBlockK);
        const bool blocks = forced_splits <= 0 && units * tt < (int64_t)device_sm_count() * occ;
        p.split_unit = blocks ? kBlockK : kTile;
        const int nu = blocks ? nb : tt;
        const int S = forced_splits > 0 ? forced_splits
                                        : (blocks ? choose_splits_blocks(units, nb, occ)
                                                  : CD_SPLITS_FUSED_MODEL ? choose_splits_fused(units, tt, occ)
                                                                          : choose_splits(units, tt, occ));
        for (int d = 0; d < 2; ++d) {
            p.ttiles[d] = ceil_div(p.npts[1 - d], kTile);
            p.splits[d] = std::max(1, std::min(S, nu));   // <= units: every split non-empty
            if (p.qtiles[d] == 0) p.splits[d] = 1;
        }
    }
    const int64_t sq = (int64_t)(q1 - q0), sr = (int64_t)(r1 - r0);
    p.slice_off[0] = 0;
    p.slice_off[1] = (int64_t)B * sq;
    p.slice_total = (int64_t)B * (sq + sr);
    p.nchunks[0] = ceil_div(sq, kMergeThreads);
    p.nchunks[1] = ceil_div(sr, kMergeThreads);
    p.chunk_off[0] = 0;
    p.chunk_off[1] = (int64_t)B * p.nchunks[0];
    p.chunk_total = (int64_t)B * (p.nchunks[0] + p.nchunks[1]);
    const int smax = std::max(p.splits[0], p.splits[1]);
    size_t off = 0;
    for (int d = 0; d < 2; ++d) {
        p.off_pack[d] = off;
        off = align_up(off + (size_t)B * p.ppad[d] * 16, 256);
    }
    (void)smax;
    p.off_rowkey = off;
    off = align_up(off + (size_t)std::max<int64_t>(p.slice_total, 1) * 8, 256);
    p.off_chunk_sum = off;
    off = align_up(off + (size_t)std::max<int64_t>(p.chunk_total, 1) * 8, 256);
    p.off_chunk_hits = off;
    off = align_up(off + (size_t)std::max<int64_t>(p.chunk_total, 1) * 4, 256);
    p.off_colkey = off;
    if (mode == kFusedFull) off = align_up(off + (size_t)B * M * 8, 256);
    p.bytes = off;
}

cudaError_t launch_forward(const FwdPlan& p, const float* x, const float* y, const FwdOutputs& o, void* ws,
                           cudaStream_t st) {
    if (p.mode == kTensor) {
        TcPlan t;
        plan_tc(t, p.B, p.npts[0], p.npts[1], p.forced_splits);
        return launch_tc(t, x, y, o, ws, st);
    }
    char* w = static_cast<char*>(ws);
    float4* pack0 = reinterpret_cast<float4*>(w + p.off_pack[0]);
    float4* pack1 = reinterpret_cast<float4*>(w + p.off_pack[1]);
    long long* colkey = p.mode == kFusedFull ? reinterpret_cast<long long*>(w + p.off_colkey) : o.colkey;
    long long* rowkey = reinterpret_cast<long long*>(w + p.off_rowkey);
    {
        PackArgs a;
        a.src[0] = x;
        a.src[1] = y;
        a.dst[0] = pack0;
        a.dst[1] = pack1;
        for (int d = 0; d < 2; ++d) {
            a.npts[d] = p.npts[d];
            a.ppad[d] = p.ppad[d];
            a.vec[d] = CD_PACK_VEC && p.npts[d] % 4 == 0 && p.ppad[d] % 4 == 0 &&
                       reinterpret_cast<uintptr_t>(a.src[d]) % 16 == 0;
        }
        a.B = p.B;
        const bool init = p.mode == kFusedFull || p.mode == kFusedRows;
        a.colkey = init ? colkey : nullptr;
        a.ncolkey = init ? (int64_t)p.B * p.npts[1] : 0;
        a.rowkey = rowkey;
        a.nrowkey = p.mode == kFusedCols ? 0 : p.slice_total;
        // one row (cloud, batch element) per (y, z); enough x blocks for ~16 CTAs per SM overall
        const int pmax = std::max(p.ppad[0], p.ppad[1]);
        const int64_t want = (int64_t)device_sm_count() * 16 / std::max<int64_t>(1, 2 * (int64_t)p.B);
        const int per = a.vec[0] && a.vec[1] ? 4 : 1;   // points per thread
        const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((pmax / per + 255) / 256, want));
        launch_pdl(pack_kernel, dim3(gx, p.B, 2), dim3(256), 0, st, a);
    }
    if (p.mode == kUnfused) {
        const int gx = p.qtiles[0] * p.splits[0] + p.qtiles[1] * p.splits[1];
        if (gx > 0) {
            FwdArgs a;
            a.pack[0] = pack0;
            a.pack[1] = pack1;
            for (int d = 0; d < 2; ++d) {
                a.npts[d] = p.npts[d];
                a.ppad[d] = p.ppad[d];
                a.qlo[d] = p.qlo[d];
                a.qhi[d] = p.qhi[d];
                a.qtiles[d] = p.qtiles[d];
                a.splits[d] = p.splits[d];
                a.ttiles[d] = p.ttiles[d];
                a.slice_off[d] = p.slice_off[d];
            }
            a.slice_total = p.slice_total;
            a.rowkey = rowkey;
            if (g_prof_start) record_profile_event(g_prof_start, st);
            nn_fwd_kernel<<<dim3(gx, p.B), kFwdThreads, 0, st>>>(a);
            if (g_prof_stop) record_profile_event(g_prof_stop, st);
        }
    } else if (p.mode == kFusedFull || p.mode == kFusedRows) {
        cudaError_t e = launch_fused_rows(p, pack0, pack1, colkey, rowkey, st);
        if (e != cudaSuccess) return e;
    }
    double* chunk_sum = reinterpret_cast<double*>(w + p.off_chunk_sum);
    int* chunk_hits = reinterpret_cast<int*>(w + p.off_chunk_hits);
    // rows (and, unfused, both directions): merge splits + exact index re-scan + chunk partials;
    // columns of the fused modes: resolve the Y rows from the (reduced) column keys — one launch
    const int64_t merge_chunks = p.mode == kUnfused ? p.chunk_total : (int64_t)p.B * p.nchunks[0];
    MergeArgs ma;
    ma.pack[0] = pack0;
    ma.pack[1] = pack1;
    for (int d = 0; d < 2; ++d) {
        ma.npts[d] = p.npts[d];
        ma.ppad[d] = p.ppad[d];
        ma.qlo[d] = p.qlo[d];
        ma.qhi[d] = p.qhi[d];
        ma.splits[d] = p.splits[d];
        ma.slice_off[d] = p.slice_off[d];
        ma.nchunks[d] = p.nchunks[d];
        ma.chunk_off[d] = p.chunk_off[d];
        ma.d_out[d] = o.d[d];
        ma.idx_out[d] = o.idx[d];
    }
    ma.slice_total = p.slice_total;
    ma.B = p.B;
    ma.rowkey = rowkey;
    ma.chunk_sum = chunk_sum;
    ma.chunk_hits = chunk_hits;
    ma.tau2 = o.tau >= 0.f ? (double)o.tau * (double)o.tau : -1.0;
    ResolveArgs ra;
    int64_t resolve_chunks = 0;
    if ((p.mode == kFusedFull || p.mode == kFusedCols) && p.nchunks[1] > 0) {
        ra.xp = pack0;
        ra.yp = pack1;
        ra.N = p.npts[0];
        ra.M = p.npts[1];
        ra.xpad = p.ppad[0];
        ra.ypad = p.ppad[1];
        ra.q0 = 0;
        ra.q1 = p.npts[0];
        ra.r0 = p.qlo[1];
        ra.r1 = p.qhi[1];
        ra.B = p.B;
        ra.nchunks = p.nchunks[1];
        ra.colkey = colkey;
        ra.npeers = o.npeers;
        for (int q = 0; q < kMaxPeers; ++q) ra.colkey_peers[q] = q < o.npeers ? o.colkey_peers[q] : nullptr;
        ra.d_out = o.d[1];
        ra.idx_out = o.idx[1];
        ra.chunk_sum = chunk_sum + p.chunk_off[1];
        ra.chunk_hits = chunk_hits + p.chunk_off[1];
        ra.tau2 = ma.tau2;
        resolve_chunks = (int64_t)p.B * p.nchunks[1];
    }
    if (merge_chunks + resolve_chunks > 0)
        launch_pdl(nn_epilogue_kernel, dim3((unsigned)(merge_chunks + resolve_chunks)), dim3(kMergeThreads), 0, st, ma,
                   ra, (int)merge_chunks);
    if (o.partials) {
        PartialsArgs a;
        a.chunk_sum = chunk_sum;
        a.chunk_hits = chunk_hits;
        for (int d = 0; d < 2; ++d) {
            a.nchunks[d] = p.nchunks[d];
            a.chunk_off[d] = p.chunk_off[d];
        }
        a.partials = o.partials;
        a.dirmask = p.mode == kFusedRows ? 1 : (p.mode == kFusedCols ? 2 : 3);
        launch_pdl(partials_kernel, dim3(p.B), dim3(256), 0, st, a);
    }
    return cudaGetLastError();
}

cudaError_t launch_partials(const double* chunk_sum, const int* chunk_hits, const int nchunks[2],
                            const int64_t chunk_off[2], int B, double* partials, int dirmask, cudaStream_t st) {
    PartialsArgs a;
    a.chunk_sum = chunk_sum;
    a.chunk_hits = chunk_hits;
    for (int d = 0; d < 2; ++d) {
        a.nchunks[d] = nchunks[d];
        a.chunk_off[d] = chunk_off[d];
    }
    a.partials = partials;
    a.dirmask = dirmask;
    partials_kernel<<<B, 256, 0, st>>>(a);
    return cudaGetLastError();
}

int forward_launches(const FwdPlan& p) {
    if (p.mode == kTensor) {
        TcPlan t;
        plan_tc(t, p.B, p.npts[0], p.npts[1], p.forced_splits);
        return tc_launches(t);
    }
    int n = 1;                                                      // pack (+ column-key reset)
    if (p.mode == kUnfused) n += 2;                                 // nn_fwd + epilogue (merge)
    if (p.mode == kFusedFull) n += 2;                               // fused + epilogue (merge | resolve)
    if (p.mode == kFusedRows) n += 2;                               // fused + epilogue (merge)
    if (p.mode == kFusedCols) n += 1;                               // epilogue (resolve)
    return n + 1;                                                   // partials
}

size_t fscore_workspace(int B, int N, int M) {
    const int64_t chunks = (int64_t)B * (ceil_div(N, kMergeThreads) + ceil_div(M, kMergeThreads));
    return align_up((size_t)chunks * 8, 256) + align_up((size_t)chunks * 4, 256) + align_up((size_t)B * 32, 256);
}

cudaError_t launch_fscore(const float* d_xy, const float* d_yx, int B, int N, int M, float tau, float* fscore,
                          float* precision, float* recall, void* ws, cudaStream_t st) {
    StatsArgs s;
    s.d[0] = d_xy;
    s.d[1] = d_yx;
    s.n[0] = N;
    s.n[1] = M;
    s.nchunks[0] = ceil_div(N, kMergeThreads);
    s.nchunks[1] = ceil_div(M, kMergeThreads);
    s.chunk_off[0] = 0;
    s.chunk_off[1] = (int64_t)B * s.nchunks[0];
    s.B = B;
    const int64_t chunks = (int64_t)B * (s.nchunks[0] + s.nchunks[1]);
    char* w = static_cast<char*>(ws);
    s.chunk_sum = reinterpret_cast<double*>(w);
    s.chunk_hits = reinterpret_cast<int*>(w + align_up((size_t)chunks * 8, 256));
    double* partials =
        reinterpret_cast<double*>(w + align_up((size_t)chunks * 8, 256) + align_up((size_t)chunks * 4, 256));
    s.tau2 = (double)tau * (double)tau;
    stats_kernel<<<(unsigned)chunks, kMergeThreads, 0, st>>>(s);
    PartialsArgs a;
    a.chunk_sum = s.chunk_sum;
    a.chunk_hits = s.chunk_hits;
    for (int d = 0; d < 2; ++d) {
        a.nchunks[d] = s.nchunks[d];
        a.chunk_off[d] = s.chunk_off[d];
    }
    a.partials = partials;
    a.dirmask = 3;
    partials_kernel<<<B, 256, 0, st>>>(a);
    FinalizeArgs f;
    f.partials = partials;
    f.B = B;
    f.N = N;
    f.M = M;
    f.w1 = 1.0;
    f.w2 = 1.0;
    f.cd = nullptr;
    f.loss = nullptr;
    f.fscore = fscore;
    f.precision = precision;
    f.recall = recall;
    launch_pdl(finalize_kernel, dim3(1), dim3(256), 0, st, f);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const double* partials, int B, int N, int M, float w1, float w2, float* cd,
                            float* loss, float* fscore, float* precision, float* recall, cudaStream_t st) {
    FinalizeArgs f;
    f.partials = partials;
    f.B = B;
    f.N = N;
    f.M = M;
    f.w1 = w1;
    f.w2 = w2;
    f.cd = cd;
    f.loss = loss;
    f.fscore = fscore;
    f.precision = precision;
    f.recall = recall;
    launch_pdl(finalize_kernel, dim3(1), dim3(256), 0, st, f);
    return cudaGetLastError();
}

}  // namespace cdk
