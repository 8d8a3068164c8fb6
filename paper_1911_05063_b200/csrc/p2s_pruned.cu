// p2s_pruned.cu — culled point-to-surface forward (SURVEY.md §8.f NEXT-3 at scale).
//
// The same outputs as p2s.cu (cd_p2s_forward) with far fewer (point, face) evaluations, built from
// the pruned nearest-neighbour machinery of nn_pruned.cu (R26):
//   bbox (nn_pruned.cu)  per batch element: sample boxes of the points and of the vertices (they only
//                        set the Hilbert quantisation).
//   ps_hilbert_kernel     key = (set | batch | Hilbert code) for every point (set 0) and every face
//                        centroid (set 1); value = flat row.
//   radix sort           (nn_backward.cu)
//   ps_gather_kernel     Hilbert-sorted packed points + permutation; face order (sorted pos -> face).
//   ps_prep_kernel       the 24-float face records (p2s_common.cuh) in Hilbert face order, padded to
//                        the 64-face tile by repeating the last sorted face.
//   ps_aabb_kernel       boxes of every 64-point query tile and of every 64-face tile and 32-face
//                        block (over the faces' vertices), each widened by delta = 2^-14 max|coord| of
//                        the box so that a box gap bounds the fp32-evaluated distances (R26).
//   ps_candidates_kernel per query tile: LB = gap^2 (1 - 1e-5) to every face tile, bitonic-sorted.
//   p2s_pruned_kernel    one warp per query tile (2 points per lane), face tiles in LB order through a
//                        2-stage TMA ring.  A tile is fetched, and a 32-face block evaluated, only if
//                        some lane may still improve: LB(lane's 2-point box, face box) <= the lane's
//                        current maximum (a vote); value-only running minimum of face_dist2 + block
//                        argmin.  Two phases for load balance: phase 0 visits each list's first
//                        kPsFirst tiles (tight upper bounds for most rows) and stores 64-bit row keys
//                        (distance bits << 32 | block); phase 1 splits the rest of every list into
//                        chunks, one CTA each, that start from those bounds, stop once the list's LB
//                        exceeds every row's bound and merge improvements with atomicMin on the keys
//                        (order-independent: deterministic).
//                        Exact ties between blocks (a block minimum EQUAL to the current one, or an
//                        equal key from another chunk, seen in atomicMin's return value) flag the
//                        point and queue it once.
//   ps_tie_kernel        flagged points: re-walk the LB-sorted candidate tiles while LB <= the minimum
//                        and keep the lowest ORIGINAL face index at the minimum (R3', the brute
//                        force's rule; persistent warps over the queue).
//   ps_resolve_kernel    the face: the tie result, else the lowest original index at the minimum inside
//                        the winning block (same fp32 ops); fp64 closest point / barycentrics /
//                        distance on that face, outputs in the original point order, fp64 chunk
//                        sums; then p2s_finalize (p2s.cu).  Outputs are bit-identical to p2s.cu's.
#include "cd_internal.h"
#include "p2s_common.cuh"

#include <algorithm>
#include <cstdio>

namespace cdk {

constexpr int kPsR = 2;                          // points per thread (one packed pair)
#ifndef CD_PS_THREADS
#define CD_PS_THREADS 32
#endif
#ifndef CD_PS_STAGES
#define CD_PS_STAGES 2
#endif
#ifndef CD_PS_TILE
#define CD_PS_TILE 64
#endif
#ifndef CD_PS_MINB
#define CD_PS_MINB 16
#endif
constexpr int kPsThreads = CD_PS_THREADS;
constexpr int kPsStages = CD_PS_STAGES;          // TMA ring depth
constexpr int kPsTile = CD_PS_TILE;              // faces per shared-memory stage
constexpr int kPsQ = kPsThreads * kPsR;          // 64 sorted points per query tile
constexpr int kPsBlocks = kPsTile / kBlockK;   // blocks of 32 faces per face tile
constexpr int kPsMaxTiles = 8192;                // face tiles per batch element (LB sort in smem)
constexpr float kPsLbScale = 0.99999f;
#ifndef CD_PS_FIRST
#define CD_PS_FIRST 16
#endif
#ifndef CD_PS_CHUNK
#define CD_PS_CHUNK 16
#endif
constexpr int kPsFirst = CD_PS_FIRST;            // phase-0 face tiles per query tile
constexpr int kPsChunk = CD_PS_CHUNK;            // phase-1 face tiles per CTA (at least)
constexpr int kPsMaxChunks = 32;                 // phase-1 CTAs per query tile (at most)
constexpr float kPsMargin = 1.0f / 16384.0f;     // delta = 2^-14 * max |coord| of the box

// ------------------------------------------------------------------------------------------ hilbert keys

struct PsHilbertArgs {
    const float* points;
    const float* verts;
    const int* faces;
    int B, N, Nv, Nf, kbits;
    const float* bbox;   // [2][B][6]
    uint32_t* keys;
    uint32_t* vals;
};

__global__ void __launch_bounds__(256) ps_hilbert_kernel(PsHilbertArgs a) {
    const int64_t L0 = (int64_t)a.B * a.N;
    const int64_t L = L0 + (int64_t)a.B * a.Nf;
    const float qmax = (float)((1 << a.kbits) - 1);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = e < L0 ? 0 : 1;
        float p[3];
        int b;
        if (c == 0) {
            b = (int)(e / a.N);
            for (int k = 0; k < 3; ++k) p[k] = __ldg(a.points + e * 3 + k);
        } else {
            const int64_t f = e - L0;
            b = (int)(f / a.Nf);
            const int fi = (int)(f - (int64_t)b * a.Nf);
            const float* v = a.verts + (int64_t)b * a.Nv * 3;
            const int i0 = min(max(a.faces[3 * fi], 0), a.Nv - 1), i1 = min(max(a.faces[3 * fi + 1], 0), a.Nv - 1),
                      i2 = min(max(a.faces[3 * fi + 2], 0), a.Nv - 1);
            for (int k = 0; k < 3; ++k) p[k] = (__ldg(v + 3 * i0 + k) + __ldg(v + 3 * i1 + k) + __ldg(v + 3 * i2 + k)) * (1.0f / 3.0f);
        }
        const float* bb = a.bbox + ((int64_t)c * a.B + b) * 6;
        uint32_t q[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float ext = bb[3 + k] - bb[k];
            float t = ext > 0.f ? (p[k] - bb[k]) / ext : 0.f;
            t = fminf(fmaxf(t, 0.f), 1.f);
            q[k] = (uint32_t)(t * qmax + 0.5f);
        }
        const uint32_t code = hilbert3(q[0], q[1], q[2], a.kbits);
        a.keys[e] = code;   // segment-local: the (points | faces, batch) segment is the sort's SegSpec
        a.vals[e] = (uint32_t)e;
    }
}

// ------------------------------------------------------------------------------------------ gather
struct PsGatherArgs {
    const float* points;
    int B, N, Nf;
    const uint32_t* vals;
    float4* spts;    // [B][N] sorted points
    int* perm_p;     // [B][N] sorted position -> original point
    int* perm_f;     // [B][Nf] sorted position -> face
};

__global__ void __launch_bounds__(256) ps_gather_kernel(PsGatherArgs a) {
    const int64_t L0 = (int64_t)a.B * a.N;
    const int64_t L = L0 + (int64_t)a.B * a.Nf;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = a.vals[s];
        if (s < L0) {
            const int b = (int)(s / a.N);
            const float* q = a.points + v * 3;
            a.spts[s] = make_float4(__ldg(q), __ldg(q + 1), __ldg(q + 2), 0.f);
            a.perm_p[s] = (int)(v - (int64_t)b * a.N);
        } else {
            const int64_t f = s - L0;
            const int b = (int)(f / a.Nf);
            a.perm_f[f] = (int)(v - L0 - (int64_t)b * a.Nf);
        }
    }
}

// ------------------------------------------------------------------------------------------ face records
struct PsPrepArgs {
    const float* verts;
    const int* faces;
    const int* perm_f;
    int B, Nv, Nf, Fpad;
    float* fd;   // [B][Fpad][24] in sorted face order
};

__global__ void __launch_bounds__(256) ps_prep_kernel(PsPrepArgs a) {
    const int64_t total = (int64_t)a.B * a.Fpad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(e / a.Fpad);
        const int pos = min((int)(e - (int64_t)b * a.Fpad), a.Nf - 1);
        const int f = a.perm_f[(int64_t)b * a.Nf + pos];
        write_face_record(a.verts + (int64_t)b * a.Nv * 3, a.Nv, a.faces, f, a.fd + e * kFaceFloats);
    }
}

// ------------------------------------------------------------------------------------------ boxes
__device__ __forceinline__ void warp_box(float lo[3], float hi[3]) {
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[q] = fminf(lo[q], __shfl_xor_sync(0xffffffffu, lo[q], o));
            hi[q] = fmaxf(hi[q], __shfl_xor_sync(0xffffffffu, hi[q], o));
        }
}

// widen a (non-empty) box by delta = 2^-14 * max |coord| (R26); an empty box stays empty
__device__ __forceinline__ void widen(float lo[3], float hi[3]) {
    if (!(lo[0] <= hi[0])) return;
    float m = 0.f;
#pragma unroll
    for (int q = 0; q < 3; ++q) m = fmaxf(m, fmaxf(fabsf(lo[q]), fabsf(hi[q])));
    const float d = m * kPsMargin + 1e-30f;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        lo[q] -= d;
        hi[q] += d;
    }
}

struct PsAabbArgs {
    const float4* spts;
    const float* verts;
    const int* faces;
    const int* perm_f;
    int B, N, Nv, Nf, qtiles, ftiles;
    float4* qbox;     // [B][qtiles][2]
    float4* fbox;     // [B][ftiles][2]
    float4* fbox32;   // [B][ftiles*4][2]
};

// One warp per query tile (lane reduces kPsQ / 32 points) or per face tile (kPsBlocks blocks of 32).
__global__ void __launch_bounds__(256) ps_aabb_kernel(PsAabbArgs a) {
    const int64_t TQ = (int64_t)a.B * a.qtiles, T = TQ + (int64_t)a.B * a.ftiles;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= T) return;
    if (wid < TQ) {
        const int b = (int)(wid / a.qtiles), t = (int)(wid - (int64_t)b * a.qtiles);
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int k = 0; k < kPsQ / 32; ++k) {
            const int p = t * kPsQ + k * 32 + lane;
            if (p < a.N) {
                const float4 v = a.spts[(int64_t)b * a.N + p];
                lo[0] = fminf(lo[0], v.x); hi[0] = fmaxf(hi[0], v.x);
                lo[1] = fminf(lo[1], v.y); hi[1] = fmaxf(hi[1], v.y);
                lo[2] = fminf(lo[2], v.z); hi[2] = fmaxf(hi[2], v.z);
            }
        }
        warp_box(lo, hi);
        widen(lo, hi);
        if (lane == 0) {
            float4* o = a.qbox + wid * 2;
            o[0] = make_float4(lo[0], lo[1], lo[2], 0.f);
            o[1] = make_float4(hi[0], hi[1], hi[2], 0.f);
        }
        return;
    }
    const int64_t f = wid - TQ;
    const int b = (int)(f / a.ftiles), t = (int)(f - (int64_t)b * a.ftiles);
    const float* vv = a.verts + (int64_t)b * a.Nv * 3;
    float tlo[3] = {INFINITY, INFINITY, INFINITY}, thi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = 0; k < kPsBlocks; ++k) {
        const int pos = t * kPsTile + k * kBlockK + lane;
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        if (pos < a.Nf) {
            const int fi = a.perm_f[(int64_t)b * a.Nf + pos];
            for (int c = 0; c < 3; ++c) {
                const int vi = min(max(a.faces[3 * fi + c], 0), a.Nv - 1);
                for (int q = 0; q < 3; ++q) {
                    const float x = vv[3 * vi + q];
                    lo[q] = fminf(lo[q], x);
                    hi[q] = fmaxf(hi[q], x);
                }
            }
        }
        warp_box(lo, hi);
        widen(lo, hi);
        if (lane == 0) {
            float4* o = a.fbox32 + ((int64_t)b * a.ftiles * kPsBlocks + t * kPsBlocks + k) * 2;
            o[0] = make_float4(lo[0], lo[1], lo[2], 0.f);
            o[1] = make_float4(hi[0], hi[1], hi[2], 0.f);
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            tlo[q] = fminf(tlo[q], lo[q]);
            thi[q] = fmaxf(thi[q], hi[q]);
        }
    }
    if (lane == 0) {
        float4* o = a.fbox + f * 2;
        o[0] = make_float4(tlo[0], tlo[1], tlo[2], 0.f);
        o[1] = make_float4(thi[0], thi[1], thi[2], 0.f);
    }
}

__device__ __forceinline__ float ps_gap(float qlo, float qhi, float tlo, float thi) {
    return fmaxf(fmaxf(tlo - qhi, qlo - thi), 0.f);
}
// squared box-box gap scaled down by 1e-5 (empty target box: +inf)
__device__ __forceinline__ float ps_box_lb(const float qlo[3], const float qhi[3], float4 lo, float4 hi) {
    if (lo.x > hi.x) return INFINITY;
    const float gx = ps_gap(qlo[0], qhi[0], lo.x, hi.x);
    const float gy = ps_gap(qlo[1], qhi[1], lo.y, hi.y);
    const float gz = ps_gap(qlo[2], qhi[2], lo.z, hi.z);
    return (gx * gx + gy * gy + gz * gz) * kPsLbScale;
}

// ------------------------------------------------------------------------------------------ candidates
struct PsCandArgs {
    const float4* qbox;
    const float4* fbox;
    int qtiles, ftiles;
    unsigned long long* cand;   // [B][qtiles][ftiles]: (LB bits << 32) | face tile, ascending
    unsigned* tiecount;         // zeroed here (the tie queue of this call is filled by the NN kernel)
};

__global__ void __launch_bounds__(256) ps_candidates_kernel(PsCandArgs a) {
    extern __shared__ unsigned long long keys[];
    const int u = blockIdx.x;
    const int b = u / a.qtiles;
    if (u == 0 && threadIdx.x == 0) *a.tiecount = 0u;
    const float4 ql = a.qbox[(int64_t)u * 2], qh = a.qbox[(int64_t)u * 2 + 1];
    const float qlo[3] = {ql.x, ql.y, ql.z}, qhi[3] = {qh.x, qh.y, qh.z};
    int npow = 1;
    while (npow < a.ftiles) npow <<= 1;
    for (int t = threadIdx.x; t < npow; t += 256) {
        unsigned long long key = ~0ull;
        if (t < a.ftiles) {
            const float4* bx = a.fbox + ((int64_t)b * a.ftiles + t) * 2;
            const float lb = ps_box_lb(qlo, qhi, bx[0], bx[1]);
            key = ((unsigned long long)__float_as_uint(lb) << 32) | (unsigned)t;
        }
        keys[t] = key;
    }
    __syncthreads();
    for (int k = 2; k <= npow; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < npow; i += 256) {
                const int l = i ^ j;
                if (l > i) {
                    const unsigned long long x = keys[i], y = keys[l];
                    if ((x > y) == ((i & k) == 0)) {
                        keys[i] = y;
                        keys[l] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
    unsigned long long* out = a.cand + (int64_t)u * a.ftiles;
    for (int t = threadIdx.x; t < a.ftiles; t += 256) out[t] = keys[t];
}

// ------------------------------------------------------------------------------------------ main kernel
#ifdef CD_PS_STATS   // experiment build only: visit statistics
__device__ unsigned long long g_ps_stats[4];
#endif
struct PsArgs {
    const float4* spts;
    const float* fd;        // [B][Fpad][24] sorted faces
    const float4* fbox;     // [B][ftiles][2] face tile boxes
    const float4* fbox32;
    const unsigned long long* cand;
    int N, Fpad, qtiles, ftiles;
    int k0, klen, nchunk;   // candidate range of chunk c: [k0 + c klen, k0 + (c+1) klen)
    int phase;              // 0: first tiles, plain store of the row keys; 1: refine from the row keys
    long long* rowkey;      // [B][N] sorted order: (best bits << 32) | sorted block position
    int* tieflag;           // [B][N] sorted order: 1 if a block other than the key's may hold the minimum
    int* tiequeue;          // flagged sorted rows, each once (the 0 -> 1 transition of its flag appends it)
    unsigned* tiecount;
};

// Per-lane lower bound: the lane's two points (widened box) against a face box; a tile or block is
// evaluated iff some thread of the CTA / lane of the warp may still improve (LB <= its own max best).
__device__ __forceinline__ float lane_lb(const float llo[3], const float lhi[3], float4 lo, float4 hi) {
    return ps_box_lb(llo, lhi, lo, hi);
}

__global__ void __launch_bounds__(kPsThreads, CD_PS_MINB) p2s_pruned_kernel(PsArgs a) {
    __shared__ __align__(128) float sm[kPsStages][kPsTile * kFaceFloats];
    __shared__ __align__(128) float4 smb[kPsStages][kPsBlocks * 2];
    __shared__ __align__(8) u64 full_bar[kPsStages];
    __shared__ unsigned s_wmax[kPsThreads / 32];

    const int u = blockIdx.x / a.nchunk, chunk = blockIdx.x - (blockIdx.x / a.nchunk) * a.nchunk;
    const int b = blockIdx.y;
    const int nt = a.ftiles;
    const int kbeg = min(nt, a.k0 + chunk * a.klen), kend = min(nt, kbeg + a.klen);
    const float* FD = a.fd + (int64_t)b * a.Fpad * kFaceFloats;
    const float4* FB = a.fbox32 + (int64_t)b * nt * kPsBlocks * 2;
    const float4* FT = a.fbox + (int64_t)b * nt * 2;
    const unsigned long long* __restrict__ cand = a.cand + ((int64_t)b * a.qtiles + u) * nt;
    const uint32_t fbytes = kPsTile * kFaceFloats * 4, bbytes = kPsBlocks * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPsStages; ++s) mbar_init(&full_bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const int P = a.N;
    const float4* Q = a.spts + (int64_t)b * P;
    const int qbase = u * kPsQ + threadIdx.x * kPsR;
    const float4 p0 = Q[min(qbase, P - 1)], p1 = Q[min(qbase + 1, P - 1)];
    const u64 qx = pk2(p0.x, p1.x), qy = pk2(p0.y, p1.y), qz = pk2(p0.z, p1.z);
    float best0 = INFINITY, best1 = INFINITY;
    const int64_t rowbase = (int64_t)b * P;
    if (a.phase == 1) {   // refine: start from the first phase's minima (upper bounds of the final ones)
        if (qbase < P) best0 = __uint_as_float((unsigned)((unsigned long long)a.rowkey[rowbase + qbase] >> 32));
        if (qbase + 1 < P) best1 = __uint_as_float((unsigned)((unsigned long long)a.rowkey[rowbase + qbase + 1] >> 32));
    }
    if (qbase >= P) best0 = -1.0f;       // padding rows: never need anything
    if (qbase + 1 >= P) best1 = -1.0f;
    const float init0 = best0, init1 = best1;
    int blk0 = -1, blk1 = -1;
    bool tie0 = false, tie1 = false;
    // widened box of the lane's (valid) points
    float llo[3] = {INFINITY, INFINITY, INFINITY}, lhi[3] = {-INFINITY, -INFINITY, -INFINITY};
    if (qbase < P) {
        llo[0] = p0.x; llo[1] = p0.y; llo[2] = p0.z;
        lhi[0] = p0.x; lhi[1] = p0.y; lhi[2] = p0.z;
    }
    if (qbase + 1 < P) {
        llo[0] = fminf(llo[0], p1.x); lhi[0] = fmaxf(lhi[0], p1.x);
        llo[1] = fminf(llo[1], p1.y); lhi[1] = fmaxf(lhi[1], p1.y);
        llo[2] = fminf(llo[2], p1.z); lhi[2] = fmaxf(lhi[2], p1.z);
    }
    widen(llo, lhi);

    // next face tile that some thread may still need, in the query tile's LB order (-1: none).  Block-
    // uniform: every thread walks the same list; one barrier per candidate considered.
    int pos = kbeg;
    auto advance = [&]() -> int {
        // CTA maximum of the rows' current minima: the sorted list ends the walk once LB exceeds it
        unsigned m = __float_as_uint(fmaxf(fmaxf(best0, best1), 0.f));
        m = __reduce_max_sync(0xffffffffu, m);
        if (lane == 0) s_wmax[warp] = m;
        __syncthreads();
        unsigned mm = s_wmax[0];
#pragma unroll
        for (int w = 1; w < kPsThreads / 32; ++w) mm = max(mm, s_wmax[w]);
        const float maxbest = __uint_as_float(mm);
        const float mine = fmaxf(best0, best1);
        int found = -1;
        while (pos < kend) {
            const unsigned long long e = cand[pos];
            if (__uint_as_float((unsigned)(e >> 32)) > maxbest) {
                pos = kend;
                break;
            }
            const int t = (int)(e & 0xffffffffull);
            ++pos;
            const bool need = lane_lb(llo, lhi, FT[2 * t], FT[2 * t + 1]) <= mine;
            if (__syncthreads_or(need)) {
                found = t;
                break;
            }
        }
        __syncthreads();   // s_wmax reuse
        return found;
    };

    int tiles[kPsStages];
    int tail = 0;
#ifdef CD_PS_STATS
    unsigned long long nblk_stat = 0;
#endif
#pragma unroll
    for (int k = 0; k < kPsStages; ++k) {
        const int t = advance();
        tiles[k] = t;
        if (t < 0) break;
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(&full_bar[k], fbytes + bbytes);
            tma_load_1d(sm[k], FD + (int64_t)t * kPsTile * kFaceFloats, fbytes, &full_bar[k]);
            tma_load_1d(smb[k], FB + (int64_t)t * kPsBlocks * 2, bbytes, &full_bar[k]);
        }
        ++tail;
    }
    for (int head = 0; head < tail; ++head) {
        const int s = head % kPsStages;
        int t = tiles[0];
#pragma unroll
        for (int q = 1; q < kPsStages; ++q) t = s == q ? tiles[q] : t;
        mbar_wait(&full_bar[s], (head / kPsStages) & 1);
#ifdef CD_PS_STATS
        if (threadIdx.x == 0) atomicAdd(&g_ps_stats[0], 1ull);
#endif
        const float* tb = sm[s];
        const float4* bb = smb[s];
        const int ft = t * kPsTile;
        const float mine = fmaxf(best0, best1);
        for (int kb = 0; kb < kPsBlocks; ++kb) {
            const bool need = lane_lb(llo, lhi, bb[2 * kb], bb[2 * kb + 1]) <= mine;
            if (!__any_sync(0xffffffffu, need)) continue;
#ifdef CD_PS_STATS
            if (lane == 0) atomicAdd(&g_ps_stats[1], 1ull);
            ++nblk_stat;
#endif
            float m0 = INFINITY, m1 = INFINITY;   // block minima
#pragma unroll 2
            for (int j = 0; j < kBlockK; ++j) {
                float d0, d1;
                face_dist2(tb + (kb * kBlockK + j) * kFaceFloats, qx, qy, qz, d0, d1);
                m0 = fminf(m0, d0);
                m1 = fminf(m1, d1);
            }
            // a block whose minimum equals the current one: an exact tie across blocks (R3'); the
            // flag is reset whenever the minimum strictly improves
            tie0 = m0 < best0 ? false : (m0 == best0 && m0 < INFINITY ? true : tie0);
            tie1 = m1 < best1 ? false : (m1 == best1 && m1 < INFINITY ? true : tie1);
            blk0 = m0 < best0 ? ft + kb * kBlockK : blk0;
            blk1 = m1 < best1 ? ft + kb * kBlockK : blk1;
            best0 = fminf(best0, m0);
            best1 = fminf(best1, m1);
        }
        __syncthreads();   // stage s consumed by every warp
        const int tn = advance();
        if (tn >= 0) {
#pragma unroll
            for (int q = 0; q < kPsStages; ++q) tiles[q] = s == q ? tn : tiles[q];
            if (threadIdx.x == 0) {
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&full_bar[s], fbytes + bbytes);
                tma_load_1d(sm[s], FD + (int64_t)tn * kPsTile * kFaceFloats, fbytes, &full_bar[s]);
                tma_load_1d(smb[s], FB + (int64_t)tn * kPsBlocks * 2, bbytes, &full_bar[s]);
            }
            ++tail;
        }
    }
#ifdef CD_PS_STATS
    if (threadIdx.x == 0) atomicMax(&g_ps_stats[2], (unsigned long long)tail);
    if (lane == 0) atomicMax(&g_ps_stats[3], nblk_stat);
#endif

    if (a.phase == 0) {
        if (qbase < P) {
            a.rowkey[rowbase + qbase] = row_key(best0, blk0);
            a.tieflag[rowbase + qbase] = tie0;
            if (tie0) a.tiequeue[atomicAdd(a.tiecount, 1u)] = (int)(rowbase + qbase);
        }
        if (qbase + 1 < P) {
            a.rowkey[rowbase + qbase + 1] = row_key(best1, blk1);
            a.tieflag[rowbase + qbase + 1] = tie1;
            if (tie1) a.tiequeue[atomicAdd(a.tiecount, 1u)] = (int)(rowbase + qbase + 1);
        }
    } else {
        // strictly improved rows only; the 64-bit minimum over chunks is order-independent.  A tie
        // between chunks shows in the value atomicMin returns (equal distance, other block): the
        // second of the two writers sees it.  Flags are only ever set here (a flag that a later,
        // strictly smaller minimum makes moot costs a re-scan, never a wrong face).
        if (qbase < P) {
            bool t = tie0;
            if (best0 < init0) {
                const long long k = row_key(best0, blk0);
                const long long old = atomicMin(a.rowkey + rowbase + qbase, k);
                t |= (old >> 32) == (k >> 32) && old != k;
            }
            if (t && atomicExch(a.tieflag + rowbase + qbase, 1) == 0)
                a.tiequeue[atomicAdd(a.tiecount, 1u)] = (int)(rowbase + qbase);
        }
        if (qbase + 1 < P) {
            bool t = tie1;
            if (best1 < init1) {
                const long long k = row_key(best1, blk1);
                const long long old = atomicMin(a.rowkey + rowbase + qbase + 1, k);
                t |= (old >> 32) == (k >> 32) && old != k;
            }
            if (t && atomicExch(a.tieflag + rowbase + qbase + 1, 1) == 0)
                a.tiequeue[atomicAdd(a.tiecount, 1u)] = (int)(rowbase + qbase + 1);
        }
    }
}

// Rows flagged with a possible cross-block tie: one warp re-walks the row's query-tile candidate list
// (tiles in LB order while LB <= the row's minimum: every face whose fp32 distance equals the minimum
// has LB <= it, R26) and returns the lowest ORIGINAL face index among the faces at the minimum — the
// brute force's choice (R3').
struct PsTieArgs {
    const float4* spts;
    const float* fd;
    const float4* fbox32;
    const unsigned long long* cand;
    const int* perm_f;
    int B, N, Nf, Fpad, qtiles, ftiles;
    const long long* rowkey;
    const int* tiequeue;
    const unsigned* tiecount;
    int* tieface;           // [B][N] sorted order: original face index (flagged rows)
};

// Persistent warps over the queue of flagged rows (a few % of the rows; the order of the queue does
// not matter: every row's result is its own).
__device__ __forceinline__ void ps_tie_row(const PsTieArgs& a, int64_t srow, int lane) {
    const int b = (int)(srow / a.N);
    const int pr = (int)(srow - (int64_t)b * a.N);
    const int u = pr / kPsQ;
    const float best = __uint_as_float((unsigned)((unsigned long long)a.rowkey[srow] >> 32));
    const float4 pp = a.spts[srow];
    float llo[3] = {pp.x, pp.y, pp.z}, lhi[3] = {pp.x, pp.y, pp.z};
    widen(llo, lhi);
    const int nt = a.ftiles;
    const unsigned long long* cand = a.cand + ((int64_t)b * a.qtiles + u) * nt;
    const float* FD = a.fd + (int64_t)b * a.Fpad * kFaceFloats;
    const float4* FB = a.fbox32 + (int64_t)b * nt * kPsBlocks * 2;
    const int* PF = a.perm_f + (int64_t)b * a.Nf;
    int low = 0x7fffffff;
#ifdef CD_PS_STATS
    int nblk_row = 0;
#endif
    // 32 candidates per step, one per lane: the tile LB (sorted) and the point's block LBs decide
    // which 32-face blocks hold a face that can equal the minimum; each such block is then evaluated
    // lane-parallel (two faces per lane: block halves)
    for (int k0 = 0; k0 < nt; k0 += 32) {
        const int k = k0 + lane;
        const unsigned long long e = k < nt ? cand[k] : ~0ull;
        const bool live = k < nt && __uint_as_float((unsigned)(e >> 32)) <= best;
        const int t = (int)(e & 0xffffffffull);
        static_assert(kPsBlocks == 2, "two 32-face blocks per face tile");
        const bool n0 = live && lane_lb(llo, lhi, FB[(t * 2) * 2], FB[(t * 2) * 2 + 1]) <= best;
        const bool n1 = live && lane_lb(llo, lhi, FB[(t * 2 + 1) * 2], FB[(t * 2 + 1) * 2 + 1]) <= best;
        // needed blocks as bits (kb * 32 + lane), two per step: half-warp h takes the h-th
        unsigned long long mm = ((unsigned long long)__ballot_sync(0xffffffffu, n1) << 32) | __ballot_sync(0xffffffffu, n0);
        while (mm) {
            const int i0 = __ffsll((long long)mm) - 1;
            mm &= mm - 1;
            const int i1 = mm ? __ffsll((long long)mm) - 1 : -1;
            if (mm) mm &= mm - 1;
            const int t0 = __shfl_sync(0xffffffffu, t, i0 & 31), t1 = __shfl_sync(0xffffffffu, t, i1 & 31);
            const int mine = lane < 16 ? i0 : i1;
            const int tm = lane < 16 ? t0 : t1;
#ifdef CD_PS_STATS
            if (lane == 0) atomicAdd(&g_ps_stats[1], i1 >= 0 ? 2ull : 1ull);
            nblk_row += i1 >= 0 ? 2 : 1;
#endif
            if (mine >= 0) {
                const int f = tm * kPsTile + (mine >> 5) * kBlockK + (lane & 15) * 2;   // faces f, f + 1
                CD_CHECK(tm >= 0 && tm < nt && f + 1 < a.Fpad);
                float fa[kFaceFloats], fb[kFaceFloats];
                load_face_record(FD + (int64_t)f * kFaceFloats, fa);
                load_face_record(FD + (int64_t)(f + 1) * kFaceFloats, fb);
                float d0, d1;
                face_dist2_2f(fa, fb, pp.x, pp.y, pp.z, d0, d1);
                if (d0 == best) low = min(low, PF[min(f, a.Nf - 1)]);
                if (d1 == best) low = min(low, PF[min(f + 1, a.Nf - 1)]);
            }
        }
        if (__ballot_sync(0xffffffffu, live) != 0xffffffffu) break;   // sorted: the rest are above the minimum
    }
    low = __reduce_min_sync(0xffffffffu, low);
    if (lane == 0) a.tieface[srow] = low;
#ifdef CD_PS_STATS
    if (lane == 0) atomicAdd(&g_ps_stats[0], 1ull);
    if (lane == 0) atomicMax(&g_ps_stats[2], (unsigned long long)(nblk_row));
    if (lane == 0) atomicMax(&g_ps_stats[3], (unsigned long long)__float_as_uint(best));
#endif
}

__global__ void __launch_bounds__(256) ps_tie_kernel(PsTieArgs a) {
    const int lane = threadIdx.x & 31;
    const unsigned count = *a.tiecount;
    CD_CHECK(count <= (unsigned)((int64_t)a.B * a.N));
    for (unsigned qi = blockIdx.x * 8 + (threadIdx.x >> 5); qi < count; qi += gridDim.x * 8)
        ps_tie_row(a, a.tiequeue[qi], lane);
}

// ------------------------------------------------------------------------------------------ resolve
struct PsResolveArgs {
    const float4* spts;
    const int* perm_p;
    const int* perm_f;
    const float* fd;
    const float* verts;
    const int* faces;
    int B, N, Nv, Nf, Fpad, nchunks;
    const long long* rowkey;
    const int* tieflag;
    const int* tieface;
    float* d_out;
    int* face_out;
    float* closest;
    float* bary;
    double* chunk_sum;
};

__global__ void __launch_bounds__(kMergeThreads) ps_resolve_kernel(PsResolveArgs a) {
    const int b = blockIdx.x / a.nchunks;
    const int chunk = blockIdx.x - b * a.nchunks;
    const int p = chunk * kMergeThreads + threadIdx.x;
    double v = 0.0;
    if (p < a.N) {
        const int64_t srow = (int64_t)b * a.N + p;
        const unsigned long long key = (unsigned long long)a.rowkey[srow];
        const float best = __uint_as_float((unsigned)(key >> 32));
        const int bb = (int)(unsigned)(key & 0xffffffffull);   // 0xffffffff -> -1
        const float4 pp = a.spts[srow];
        int face = a.perm_f[(int64_t)b * a.Nf];
        if (bb >= 0 && a.tieflag[srow] && a.tieface[srow] != 0x7fffffff) {
            face = a.tieface[srow];   // cross-block tie: lowest original index over all faces at the minimum
        } else if (bb >= 0) {
            // lowest original index among the winning block's faces at the minimum (R3')
            const float* FD = a.fd + (int64_t)b * a.Fpad * kFaceFloats;
            const int fend = min(bb + kBlockK, a.Nf);
            int low = 0x7fffffff;
            for (int f = bb; f < fend; f += 2) {   // two faces per packed evaluation
                const int g = min(f + 1, fend - 1);
                float fa[kFaceFloats], fb[kFaceFloats];
                load_face_record(FD + (int64_t)f * kFaceFloats, fa);
                load_face_record(FD + (int64_t)g * kFaceFloats, fb);
                float d0, d1;
                face_dist2_2f(fa, fb, pp.x, pp.y, pp.z, d0, d1);
                if (d0 == best) low = min(low, a.perm_f[(int64_t)b * a.Nf + f]);
                if (d1 == best) low = min(low, a.perm_f[(int64_t)b * a.Nf + g]);
            }
            face = low != 0x7fffffff ? low : a.perm_f[(int64_t)b * a.Nf + min(bb, a.Nf - 1)];
        }
        // no finite candidate (a non-finite point, R6): (+inf, face -1, closest 0, bary 0) as the oracle
        const float* vv = a.verts + (int64_t)b * a.Nv * 3;
        double A[3], Bv[3], C[3], q[3] = {pp.x, pp.y, pp.z}, c[3] = {0.0, 0.0, 0.0}, lam[3] = {0.0, 0.0, 0.0};
        double dd = INFINITY;
        if (bb >= 0) {
            const int ia = min(max(a.faces[3 * face], 0), a.Nv - 1), ib = min(max(a.faces[3 * face + 1], 0), a.Nv - 1),
                      ic = min(max(a.faces[3 * face + 2], 0), a.Nv - 1);
            for (int k = 0; k < 3; ++k) {
                A[k] = vv[3 * ia + k];
                Bv[k] = vv[3 * ib + k];
                C[k] = vv[3 * ic + k];
            }
            dd = face_foot64(q, A, Bv, C, c, lam);
        } else {
            face = -1;
        }
        const int64_t row = (int64_t)b * a.N + a.perm_p[srow];
        a.d_out[row] = (float)dd;
        a.face_out[row] = face;
        if (a.closest)
            for (int k = 0; k < 3; ++k) a.closest[3 * row + k] = (float)c[k];
        if (a.bary)
            for (int k = 0; k < 3; ++k) a.bary[3 * row + k] = (float)lam[k];
        v = (double)(float)dd;
    }
    __shared__ double ssum[kMergeThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) ssum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kMergeThreads / 32; ++w) s += ssum[w];
        a.chunk_sum[(int64_t)b * a.nchunks + chunk] = s;
    }
}

// ------------------------------------------------------------------------------------------ host
static int ps_cdiv(int64_t x, int64_t y) { return (int)((x + y - 1) / y); }

struct PsPlan {
    int B, N, Nv, Nf, Fpad, qtiles, ftiles, nchunks, kbits, nbits;
    SegSpec segs;
    int64_t L;
    size_t off_bbox, off_keys[2], off_vals[2], off_counts, off_totals, off_spts, off_perm_p, off_perm_f, off_fd,
        off_qbox, off_fbox, off_fbox32, off_cand, off_rowkey, off_tieflag, off_tieface, off_tiequeue, off_tiecount, off_chunk, bytes;
    int k_first, klen, nchunk;   // phase 0: candidates [0, k_first); phase 1: nchunk chunks of klen
    bool supported;
};

static void plan_ps(PsPlan& p, int B, int N, int Nv, int Nf) {
    p.B = B;
    p.N = N;
    p.Nv = Nv;
    p.Nf = Nf;
    p.Fpad = ps_cdiv(Nf, kPsTile) * kPsTile;
    p.qtiles = ps_cdiv(N, kPsQ);
    p.ftiles = p.Fpad / kPsTile;
    p.nchunks = ps_cdiv(N, kMergeThreads);
    p.kbits = hilbert_bits(std::max(N, Nf));
    p.nbits = 3 * p.kbits;
    p.segs = SegSpec{B, N, B, Nf};
    p.L = (int64_t)B * N + (int64_t)B * Nf;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    p.off_bbox = take((size_t)2 * B * 6 * 4);
    for (int i = 0; i < 2; ++i) {
        p.off_keys[i] = take((size_t)p.L * 4);
        p.off_vals[i] = take((size_t)p.L * 4);
    }
    p.off_counts = take(radix_sort_counts_words(p.segs, p.nbits, true) * 4);
    p.off_totals = take(radix_sort_totals_words(p.segs, p.nbits, true) * 4);
    p.off_spts = take((size_t)B * N * 16);
    p.off_perm_p = take((size_t)B * N * 4);
    p.off_perm_f = take((size_t)B * Nf * 4);
    p.off_fd = take((size_t)B * p.Fpad * kFaceFloats * 4);
    p.off_qbox = take((size_t)B * p.qtiles * 32);
    p.off_fbox = take((size_t)B * p.ftiles * 32);
    p.off_fbox32 = take((size_t)B * p.ftiles * kPsBlocks * 32);
    p.off_cand = take((size_t)B * p.qtiles * p.ftiles * 8);
    p.off_rowkey = take((size_t)B * N * 8);
    p.off_tieflag = take((size_t)B * N * 4);
    p.off_tieface = take((size_t)B * N * 4);
    p.off_tiequeue = take((size_t)B * N * 4);
    p.off_tiecount = take(256);
    p.off_chunk = take((size_t)B * p.nchunks * 8);
    p.bytes = off;
    // phase 0 visits each query tile's nearest kPsFirst face tiles (tight upper bounds for most rows);
    // phase 1 spreads the rest of every list over chunks of klen tiles, one CTA each (load balance:
    // the work of a far or straddling query tile is split instead of serialised in one CTA)
    p.k_first = std::min(p.ftiles, kPsFirst);
    const int rest = p.ftiles - p.k_first;
    p.klen = std::max(kPsChunk, ps_cdiv(rest, kPsMaxChunks));
    p.nchunk = rest > 0 ? ps_cdiv(rest, p.klen) : 0;
    p.supported = (double)B * p.qtiles * p.ftiles * 8.0 <= 4294967296.0 && p.ftiles <= kPsMaxTiles && p.L <= 0x7fffffffLL;
}

size_t p2s_pruned_workspace(int B, int N, int Nv, int Nf) {
    PsPlan p;
    plan_ps(p, B, N, Nv, Nf);
    return p.supported ? p.bytes : 0;
}

int p2s_pruned_launches(int B, int N, int Nv, int Nf) {
    PsPlan p;
    plan_ps(p, B, N, Nv, Nf);
    return 2 + radix_sort_launches(p.segs, p.nbits, true) + 7 + (p.nchunk > 0 ? 1 : 0) + 1;   // + ties + finalize
}

cudaError_t launch_p2s_pruned(const float* points, const float* verts, const int* faces, int B, int N, int Nv, int Nf,
                              float* d, int* face, float* closest, float* bary, float* per_batch, float* loss,
                              void* ws, cudaStream_t st) {
    PsPlan p;
    plan_ps(p, B, N, Nv, Nf);
    if (!p.supported) return cudaErrorInvalidValue;
    char* w = static_cast<char*>(ws);
    const int sms = current_sm_count();
    float* bbox = reinterpret_cast<float*>(w + p.off_bbox);
    launch_bbox(points, N, verts, Nv, B, bbox, st);
    uint32_t* keys[2] = {reinterpret_cast<uint32_t*>(w + p.off_keys[0]), reinterpret_cast<uint32_t*>(w + p.off_keys[1])};
    uint32_t* vals[2] = {reinterpret_cast<uint32_t*>(w + p.off_vals[0]), reinterpret_cast<uint32_t*>(w + p.off_vals[1])};
    const int grid_l = (int)std::min<int64_t>((p.L + 255) / 256, (int64_t)sms * 16);
    {
        PsHilbertArgs a{points, verts, faces, B, N, Nv, Nf, p.kbits, bbox, keys[0], vals[0]};
        ps_hilbert_kernel<<<grid_l, 256, 0, st>>>(a);
    }
    const int cur = radix_sort_pairs(keys, vals, p.segs, p.nbits, reinterpret_cast<uint32_t*>(w + p.off_counts),
                                     reinterpret_cast<uint32_t*>(w + p.off_totals), st, false, true);
    float4* spts = reinterpret_cast<float4*>(w + p.off_spts);
    int* perm_p = reinterpret_cast<int*>(w + p.off_perm_p);
    int* perm_f = reinterpret_cast<int*>(w + p.off_perm_f);
    float* fd = reinterpret_cast<float*>(w + p.off_fd);
    float4* qbox = reinterpret_cast<float4*>(w + p.off_qbox);
    float4* fbox = reinterpret_cast<float4*>(w + p.off_fbox);
    float4* fbox32 = reinterpret_cast<float4*>(w + p.off_fbox32);
    unsigned long long* cand = reinterpret_cast<unsigned long long*>(w + p.off_cand);
    long long* rowkey = reinterpret_cast<long long*>(w + p.off_rowkey);
    int* tieflag = reinterpret_cast<int*>(w + p.off_tieflag);
    int* tieface = reinterpret_cast<int*>(w + p.off_tieface);
    int* tiequeue = reinterpret_cast<int*>(w + p.off_tiequeue);
    unsigned* tiecount = reinterpret_cast<unsigned*>(w + p.off_tiecount);
    double* chunk = reinterpret_cast<double*>(w + p.off_chunk);
    {
        PsGatherArgs a{points, B, N, Nf, vals[cur], spts, perm_p, perm_f};
        ps_gather_kernel<<<grid_l, 256, 0, st>>>(a);
    }
    {
        PsPrepArgs a{verts, faces, perm_f, B, Nv, Nf, p.Fpad, fd};
        ps_prep_kernel<<<std::min(ps_cdiv((int64_t)B * p.Fpad, 256), sms * 16), 256, 0, st>>>(a);
    }
    {
        PsAabbArgs a{spts, verts, faces, perm_f, B, N, Nv, Nf, p.qtiles, p.ftiles, qbox, fbox, fbox32};
        const int64_t tasks = (int64_t)B * (p.qtiles + p.ftiles);
        ps_aabb_kernel<<<ps_cdiv(tasks * 32, 256), 256, 0, st>>>(a);
    }
    {
        PsCandArgs a{qbox, fbox, p.qtiles, p.ftiles, cand, tiecount};
        int npow = 1;
        while (npow < p.ftiles) npow <<= 1;
        ensure_smem_attr((const void*)ps_candidates_kernel, kPsMaxTiles * 8);
        ps_candidates_kernel<<<B * p.qtiles, 256, (size_t)npow * 8, st>>>(a);
    }
    {
        PsArgs a{spts, fd, fbox, fbox32, cand, N, p.Fpad, p.qtiles, p.ftiles, 0, p.k_first, 1, 0, rowkey, tieflag, tiequeue, tiecount};
        if (g_prof_start) record_profile_event(g_prof_start, st);
        p2s_pruned_kernel<<<dim3(p.qtiles, B), kPsThreads, 0, st>>>(a);
        if (p.nchunk > 0) {
            a.k0 = p.k_first;
            a.klen = p.klen;
            a.nchunk = p.nchunk;
            a.phase = 1;
            p2s_pruned_kernel<<<dim3(p.qtiles * p.nchunk, B), kPsThreads, 0, st>>>(a);
        }
        if (g_prof_stop) record_profile_event(g_prof_stop, st);
#ifdef CD_PS_STATS
        unsigned long long h[4];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_ps_stats, sizeof(h));
        printf("ps_stats tiles=%llu warp_blocks=%llu maxtiles=%llu maxwarpblocks=%llu ctas=%d ftiles=%d (full warp_blocks=%lld)\n", h[0], h[1], h[2], h[3],
               p.qtiles * B, p.ftiles, (long long)p.qtiles * B * p.ftiles * kPsBlocks * (kPsThreads / 32));
        unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(g_ps_stats, z, sizeof(z));
#endif
    }
    {
        PsTieArgs a{spts, fd, fbox32, cand, perm_f, B, N, Nf, p.Fpad, p.qtiles, p.ftiles, rowkey, tiequeue, tiecount,
                    tieface};
        ps_tie_kernel<<<std::min(ps_cdiv((int64_t)B * N, 8), sms * 8), 256, 0, st>>>(a);
#ifdef CD_PS_STATS
        unsigned long long h[4];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_ps_stats, sizeof(h));
        printf("ps_tie_stats flagged_rows=%llu blocks=%llu of rows=%d maxblocks=%llu maxbest=%g\n", h[0], h[1], B * N, h[2],
               (double)__builtin_bit_cast(float, (unsigned)h[3]));
        unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(g_ps_stats, z, sizeof(z));
#endif
    }
    {
        PsResolveArgs a{spts, perm_p, perm_f, fd, verts, faces, B, N, Nv, Nf, p.Fpad, p.nchunks,
                        rowkey, tieflag, tieface, d, face, closest, bary, chunk};
        ps_resolve_kernel<<<B * p.nchunks, kMergeThreads, 0, st>>>(a);
    }
    launch_p2s_finalize(chunk, B, N, p.nchunks, per_batch, loss, st);
    return cudaGetLastError();
}

}  // namespace cdk
