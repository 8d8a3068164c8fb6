// nn_pruned.cu — exact pruned nearest-neighbour forward.
//
// Same results as the brute force (the fixed fp32 distance formula of DESIGN.md §4.2 evaluated on
// every pair that could matter), far fewer pairs on large clouds:
//   bbox_kernel        per (cloud, batch) bounding box of a fixed-stride sample (min/max: order-free;
//                      only the Hilbert quantisation depends on it).
//   hilbert_kernel      key = 3k-bit Hilbert index per point, value = row.
//   radix sort         (nn_backward.cu) every (cloud, batch) segment on its own -> Hilbert order.
//   gather_kernel      sorted packed float4 clouds + permutation (sorted position -> original row).
//   aabb_kernel        bounding box of every 512-point tile of the sorted clouds.
//   candidates_kernel  per query tile (128 sorted rows): lower bound LB of the squared distance to
//                      every target tile (box-box gap, scaled by (1 - 1e-5) so it is a strict lower
//                      bound of the fp32-evaluated distances; large clouds: via 16-tile super tiles),
//                      sorted ascending.
//   nn_pruned_kernel   per query tile: target tiles in LB order through the 2-stage TMA ring, the
//                      same packed-FP32 value-only min + block argmin tracking as nn_fwd_kernel; stops
//                      at the first tile with LB > max over the CTA's rows of the current minimum:
//                      every skipped pair has d > that row's minimum, so the minimum is exact.
//   pruned_resolve_kernel  exact index inside the winning 32-target block (same .rn ops), mapped back
//                      to original rows; outputs in original order; chunk partials.
// Tie-break: among EXACTLY equal distances the index found first in LB-tile order wins (the brute
// force returns the lowest index); any such index is an exact nearest neighbour (R3').
#include "cd_device.cuh"
#include "cd_internal.h"
#include "seg_sort.cuh"

#include <algorithm>
#include <cstdio>

namespace cdk {

// Geometry (the -D overrides exist for tools/build_variant.py sweeps; the defaults are the measured
// best of profiles/r02_experiments.txt): 2 rows x 64 threads = 128-row query tiles, own candidate lists.
#ifndef CD_PR_R
#define CD_PR_R 2
#endif
#ifndef CD_PR_THREADS
#define CD_PR_THREADS 64
#endif
constexpr int kPrR = CD_PR_R;                   // query rows per thread (packed f32x2 pairs)
constexpr int kPrThreads = CD_PR_THREADS;       // threads per query-tile CTA
constexpr int kPrQ = kPrThreads * kPrR;         // sorted rows per query tile of the main kernel
#ifndef CD_CAND_Q
#define CD_CAND_Q kPrQ
#endif
constexpr int kCandQ = CD_CAND_Q;               // sorted rows per candidate list (query tiles may share one)
static_assert(kCandQ % kPrQ == 0, "a candidate list covers whole query tiles");
constexpr int kPrMaxTiles = 8192;               // target tiles per batch supported by the LB sort
static_assert(kPrMaxTiles <= (1 << 13), "candidate keys hold a 13-bit tile index");
constexpr float kLbScale = 0.99999f;            // LB' = LB * (1 - 1e-5): strict lower bound margin
// Candidate keys: the top 19 bits of LB' (>= 0: sign, exponent, 10 mantissa bits — truncation rounds
// DOWN, so the key's LB is still a lower bound) above the 13-bit tile index (< kPrMaxTiles); ascending
// keys = ascending LB, ties by tile.  32 bits halve the sort's shared memory (more CTAs per SM).
__device__ __forceinline__ uint32_t cand_key(float lb, int t) {
    return (__float_as_uint(lb) & 0xFFFFE000u) | (uint32_t)t;
}
__device__ __forceinline__ float cand_lb(uint32_t k) { return __uint_as_float(k & 0xFFFFE000u); }
__device__ __forceinline__ int cand_tile(uint32_t k) { return (int)(k & 0x1FFFu); }

// --------------------------------------------------------------------------------------------- bbox
struct BoxArgs {
    const float* src[2];
    int npts[2];
    int B;
    float* bbox;   // [2][B][6]: lo xyz, hi xyz
};

__global__ void __launch_bounds__(256) bbox_kernel(BoxArgs a) {
    const int c = blockIdx.x / a.B, b = blockIdx.x - (blockIdx.x / a.B) * a.B;
    const float* p = a.src[c] + (int64_t)b * a.npts[c] * 3;
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    // The box only sets the Hilbert quantisation (codes are clamped), never correctness: a fixed-
    // stride sample of ~4K points per cloud is enough and keeps this O(4K) per batch element.
    const int stride = max(1, a.npts[c] / 4096);
    for (int i = threadIdx.x * stride; i < a.npts[c]; i += 256 * stride) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float v = __ldg(p + (int64_t)i * 3 + k);
            lo[k] = fminf(lo[k], v);
            hi[k] = fmaxf(hi[k], v);
        }
    }
    __shared__ float s[8][6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
    }
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 3; ++k) {
            s[threadIdx.x >> 5][k] = lo[k];
            s[threadIdx.x >> 5][3 + k] = hi[k];
        }
    __syncthreads();
    if (threadIdx.x < 6) {
        float v = s[0][threadIdx.x];
        for (int w = 1; w < 8; ++w) v = threadIdx.x < 3 ? fminf(v, s[w][threadIdx.x]) : fmaxf(v, s[w][threadIdx.x]);
        a.bbox[((int64_t)c * a.B + b) * 6 + threadIdx.x] = v;
    }
}

void launch_bbox(const float* src0, int n0, const float* src1, int n1, int B, float* bbox, cudaStream_t st) {
    BoxArgs a;
    a.src[0] = src0;
    a.src[1] = src1;
    a.npts[0] = n0;
    a.npts[1] = n1;
    a.B = B;
    a.bbox = bbox;
    bbox_kernel<<<2 * B, 256, 0, st>>>(a);
}

// --------------------------------------------------------------------------------------------- hilbert keys

struct HilbertArgs {
    const float* src[2];
    int npts[2];
    int B, kbits;
    const float* bbox;
    uint32_t* keys;
    uint32_t* vals;
    unsigned* fb_count;   // tie queue of the resolve, reset here
};

__global__ void __launch_bounds__(256) hilbert_kernel(HilbertArgs a) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.fb_count) *a.fb_count = 0u;
    // L = B (N + M) < 2^31 (cd_forward_pruned's size limit): 32-bit index arithmetic
    const int L0 = a.B * a.npts[0];
    const int L = L0 + a.B * a.npts[1];
    const float qmax = (float)((1 << a.kbits) - 1);
    for (int64_t e64 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e64 < L; e64 += (int64_t)gridDim.x * blockDim.x) {
        const int e = (int)e64;
        const int c = e < L0 ? 0 : 1;
        const int f = c == 0 ? e : e - L0;
        const int b = f / a.npts[c];
        const float* bb = a.bbox + ((int64_t)c * a.B + b) * 6;
        const float* p = a.src[c] + (int64_t)f * 3;
        uint32_t q[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            // any quantisation is valid (the order only steers the culling): fast division
            const float ext = bb[3 + k] - bb[k];
            float t = ext > 0.f ? __fdividef(__ldg(p + k) - bb[k], ext) : 0.f;
            t = fminf(fmaxf(t, 0.f), 1.f);          // NaN -> 0 via fmaxf
            q[k] = (uint32_t)(t * qmax + 0.5f);
        }
        const uint32_t code = hilbert3(q[0], q[1], q[2], a.kbits);
        a.keys[e] = code;   // segment-local: the (cloud, batch) segment is the sort's SegSpec
        a.vals[e] = (uint32_t)e;
    }
}

// --------------------------------------------------------------------------------------------- gather
struct GatherArgs {
    const float* src[2];
    int npts[2], ppad[2];
    int B;
    const uint32_t* vals;   // sorted flat rows (cloud 0 rows first)
    float4* sorted[2];      // [B][ppad]
    int* perm[2];           // [B][npts]: sorted position -> original row within the batch element
};

__global__ void __launch_bounds__(256) gather_kernel(GatherArgs a) {
    const int64_t L0 = (int64_t)a.B * a.npts[0];
    const int64_t L = L0 + (int64_t)a.B * a.npts[1];
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L; s += (int64_t)gridDim.x * blockDim.x) {
        const int c = s < L0 ? 0 : 1;
        const int f = (int)(c == 0 ? s : s - L0);       // (b, p) of the sorted position (< 2^31)
        const int b = f / a.npts[c];
        const int p = f - b * a.npts[c];
        const int64_t v = (int64_t)a.vals[s] - (c == 0 ? 0 : L0);  // original flat row of the same cloud
        const float* q = a.src[c] + v * 3;
        a.sorted[c][(int64_t)b * a.ppad[c] + p] = make_float4(__ldg(q), __ldg(q + 1), __ldg(q + 2), 0.f);
        a.perm[c][(int64_t)b * a.npts[c] + p] = (int)(v - (int64_t)b * a.npts[c]);
    }
    // padding rows of every batch element: +inf (never a nearest neighbour)
    const int64_t pad0 = (int64_t)a.B * (a.ppad[0] - a.npts[0]);
    const int64_t padL = pad0 + (int64_t)a.B * (a.ppad[1] - a.npts[1]);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < padL; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = e < pad0 ? 0 : 1;
        const int64_t f = c == 0 ? e : e - pad0;
        const int w = a.ppad[c] - a.npts[c];
        const int b = (int)(f / w);
        const int p = a.npts[c] + (int)(f - (int64_t)b * w);
        a.sorted[c][(int64_t)b * a.ppad[c] + p] = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
    }
}


// ------------------------------------------------------------------------------ on-chip Hilbert sort
// Clouds of <= kSegMax points: one CTA per (cloud, batch element) computes 14-bit Hilbert keys (a 32^3
// grid over the element's box, top 14 of 15 bits), sorts them stably on chip (seg_sort.cuh: two 7-bit
// passes) and writes the sorted packed points, the permutation and the +inf padding directly —
// replacing hilbert_kernel + the global radix passes + gather_kernel.  Any order is correct (the
// culling is exact for every permutation); the order only sets how tight the tile boxes are.
constexpr int kPrSegKeyBits = 14;

struct PrSegArgs {
    const float* src[2];
    int npts[2], ppad[2];
    int B, nmax;
    float4* sorted[2];
    int* perm[2];
    float4* box[2];       // [B][ppad/kTile][2] tile boxes (as aabb_kernel)
    float4* bbox32[2];    // [B][ppad/kBlockK][2] 32-point block boxes
    unsigned* fb_count;   // tie queue of the resolve, reset here
};

__global__ void __launch_bounds__(kSegThreads) pr_segsort_kernel(PrSegArgs a) {
    extern __shared__ __align__(16) uint32_t smem_pr[];
    uint32_t* wcur = smem_pr;
    uint32_t* wnext = wcur + kSegWarps * kSegD;
    uint16_t* kA = reinterpret_cast<uint16_t*>(wnext + kSegWarps * kSegD);
    uint16_t* kB = kA + a.nmax;
    uint16_t* vA = kB + a.nmax;
    uint16_t* vB = vA + a.nmax;
    __shared__ uint32_t dstart[kSegD];
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.fb_count) *a.fb_count = 0u;
    __shared__ float s_box[kSegWarps][6];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = blockIdx.x / a.B, b = blockIdx.x - c * a.B;
    const int n = a.npts[c];
    const float* P = a.src[c] + (int64_t)b * n * 3;
    // the element's box (it only sets the quantisation; NaN coordinates are ignored by fminf/fmaxf)
    float bb[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll 4
    for (int i = threadIdx.x; i < n; i += kSegThreads)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float v = __ldg(P + (int64_t)i * 3 + k);
            bb[k] = fminf(bb[k], v);
            bb[3 + k] = fmaxf(bb[3 + k], v);
        }
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            bb[k] = fminf(bb[k], __shfl_xor_sync(0xffffffffu, bb[k], o));
            bb[3 + k] = fmaxf(bb[3 + k], __shfl_xor_sync(0xffffffffu, bb[3 + k], o));
        }
    if (lane == 0)
        for (int k = 0; k < 6; ++k) s_box[warp][k] = bb[k];
    __syncthreads();
    for (int w = 0; w < kSegWarps; ++w)
        for (int k = 0; k < 3; ++k) {
            bb[k] = fminf(bb[k], s_box[w][k]);
            bb[3 + k] = fmaxf(bb[3 + k], s_box[w][3 + k]);
        }
    const int passes = 2, db = kPrSegKeyBits / 2, D = 1 << db;
    int lspan = 5;   // warp w owns [w*span, (w+1)*span), span a power of two
    while (kSegWarps << lspan < n) ++lspan;
    const int R = 1 << (lspan - 5);
    for (int i = threadIdx.x; i < 2 * kSegWarps * kSegD; i += kSegThreads) wcur[i] = 0;
    float lo[3], sc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float ext = bb[3 + k] - bb[k];
        lo[k] = bb[k];
        sc[k] = ext > 0.f ? 31.f / ext : 0.f;   // (no finite point: ext is NaN or -inf -> 0)
    }
    __syncthreads();
#pragma unroll 4
    for (int i = threadIdx.x; i < n; i += kSegThreads) {
        uint32_t q[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float t = fminf(fmaxf((__ldg(P + (int64_t)i * 3 + k) - lo[k]) * sc[k], 0.f), 31.f);   // NaN -> 0
            q[k] = (uint32_t)(t + 0.5f);
        }
        const uint16_t key = (uint16_t)(hilbert3(q[0], q[1], q[2], 5) >> (15 - kPrSegKeyBits));
        kA[i] = key;
        vA[i] = (uint16_t)i;
        atomicAdd(&wcur[(i >> lspan) * D + (key & (D - 1))], 1u);
    }
    seg_lsd_passes(kA, vA, kB, vB, wcur, wnext, dstart, n, passes, db, lspan, R);
    __syncthreads();
    float4* S = a.sorted[c] + (int64_t)b * a.ppad[c];
    int* PM = a.perm[c] + (int64_t)b * n;
    for (int pos = threadIdx.x; pos < a.ppad[c]; pos += kSegThreads) {
        if (pos < n) {
            const int i = vA[pos];
            const float* q = P + (int64_t)i * 3;
            S[pos] = make_float4(__ldg(q), __ldg(q + 1), __ldg(q + 2), 0.f);
            PM[pos] = i;
        } else {
            S[pos] = make_float4(INFINITY, INFINITY, INFINITY, 0.f);   // padding: never a neighbour
        }
    }
    // block and tile boxes of the sorted element (one warp per 512-point tile, as aabb_kernel)
    const int nt = a.ppad[c] / kTile;
    for (int t = warp; t < nt; t += kSegWarps) {
        float tlo[3] = {INFINITY, INFINITY, INFINITY}, thi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int k = 0; k < (kTile / kBlockK); ++k) {
            const int pos = t * kTile + k * kBlockK + lane;
            float lo3[3] = {INFINITY, INFINITY, INFINITY}, hi3[3] = {-INFINITY, -INFINITY, -INFINITY};
            if (pos < n) {
                const float* q = P + (int64_t)vA[pos] * 3;
#pragma unroll
                for (int d = 0; d < 3; ++d) lo3[d] = hi3[d] = __ldg(q + d);
            }
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    lo3[d] = fminf(lo3[d], __shfl_xor_sync(0xffffffffu, lo3[d], o));
                    hi3[d] = fmaxf(hi3[d], __shfl_xor_sync(0xffffffffu, hi3[d], o));
                }
            if (lane == 0) {
                float4* o = a.bbox32[c] + (((int64_t)b * nt + t) * (kTile / kBlockK) + k) * 2;
                o[0] = make_float4(lo3[0], lo3[1], lo3[2], 0.f);
                o[1] = make_float4(hi3[0], hi3[1], hi3[2], 0.f);
            }
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                tlo[d] = fminf(tlo[d], lo3[d]);
                thi[d] = fmaxf(thi[d], hi3[d]);
            }
        }
        if (lane == 0) {
            float4* o = a.box[c] + ((int64_t)b * nt + t) * 2;
            o[0] = make_float4(tlo[0], tlo[1], tlo[2], 0.f);
            o[1] = make_float4(thi[0], thi[1], thi[2], 0.f);
        }
    }
}

// --------------------------------------------------------------------------------------------- tile boxes
constexpr int kBlocksPerTile = kTile / kBlockK;  // 16 blocks of 32 points per 512-point tile

struct AabbArgs {
    const float4* sorted[2];
    int npts[2], ppad[2];
    int B;
    float4* box[2];         // [B][ppad/kTile][2]: tile lo, hi (empty: lo = +inf, hi = -inf)
    float4* bbox32[2];      // [B][ppad/kBlockK][2]: 32-point block lo, hi
};

// One warp per 512-point tile: lane l reduces point l of each 32-point block.
__global__ void __launch_bounds__(256) aabb_kernel(AabbArgs a) {
    const int nt0 = a.ppad[0] / kTile, nt1 = a.ppad[1] / kTile;
    const int64_t T0 = (int64_t)a.B * nt0, T = T0 + (int64_t)a.B * nt1;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= T) return;
    const int c = wid < T0 ? 0 : 1;
    const int64_t f = c == 0 ? wid : wid - T0;
    const int nt = c == 0 ? nt0 : nt1;
    const int b = (int)(f / nt);
    const int t = (int)(f - (int64_t)b * nt);
    float tlo[3] = {INFINITY, INFINITY, INFINITY}, thi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = 0; k < kBlocksPerTile; ++k) {
        const int p = t * kTile + k * kBlockK + lane;
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        if (p < a.npts[c]) {
            const float4 v = a.sorted[c][(int64_t)b * a.ppad[c] + p];
            lo[0] = hi[0] = v.x;
            lo[1] = hi[1] = v.y;
            lo[2] = hi[2] = v.z;
        }
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo[q] = fminf(lo[q], __shfl_xor_sync(0xffffffffu, lo[q], o));
                hi[q] = fmaxf(hi[q], __shfl_xor_sync(0xffffffffu, hi[q], o));
            }
        if (lane == 0) {
            float4* o = a.bbox32[c] + (((int64_t)b * nt + t) * kBlocksPerTile + k) * 2;
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
        float4* o = a.box[c] + ((int64_t)b * nt + t) * 2;
        o[0] = make_float4(tlo[0], tlo[1], tlo[2], 0.f);
        o[1] = make_float4(thi[0], thi[1], thi[2], 0.f);
    }
}

// --------------------------------------------------------------------------------------------- candidates
struct CandArgs {
    const float4* box[2];
    const float4* box32[2];   // 32-point block boxes: the query tile box is their union
    int ppad[2];
    int B;
    int qtiles[2];            // candidate lists (kCandQ rows) per batch element, per dir
    int64_t cand_off[2];      // offset of dir's lists in `cand` (u64 entries)
    uint32_t* cand;           // per (dir, b, query tile): up to ttiles(1-dir) keys (cand_key: LB' | tile)
    int* ccount;              // per list: number of entries (LB <= UB), lists of dir 1 after dir 0's
    const float4* sbox[2];    // [B][nst][2] super-tile boxes (kSuper tiles), or null: flat scan
};

// Super tiles: kSuper consecutive 512-point tiles of a Hilbert-sorted cloud (8192 points, spatially
// compact).  superbox_kernel: their boxes (union of the non-empty tile boxes; empty: lo = +inf).
constexpr int kSuper = 16;
constexpr int kHierMinTiles = 64;   // target clouds of >= 64 tiles use the two-level candidate search
#ifndef CD_PR_HIER
#define CD_PR_HIER 1   // two-level candidate search for clouds of >= kHierMinTiles tiles
#endif

__global__ void __launch_bounds__(256) superbox_kernel(const float4* box0, const float4* box1, int nt0, int nt1,
                                                       int B, float4* sbox0, float4* sbox1) {
    const int ns0 = (nt0 + kSuper - 1) / kSuper, ns1 = (nt1 + kSuper - 1) / kSuper;
    const int64_t S0 = (int64_t)B * ns0, S = S0 + (int64_t)B * ns1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = i < S0 ? 0 : 1;
        const int64_t f = c == 0 ? i : i - S0;
        const int ns = c == 0 ? ns0 : ns1, nt = c == 0 ? nt0 : nt1;
        const int bb = (int)(f / ns), sidx = (int)(f - (int64_t)bb * ns);
        const float4* bx = (c == 0 ? box0 : box1) + (int64_t)bb * nt * 2;
        float4 lo = make_float4(INFINITY, INFINITY, INFINITY, 0.f), hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
        for (int t = sidx * kSuper; t < min(nt, (sidx + 1) * kSuper); ++t) {
            const float4 l = bx[2 * t], h = bx[2 * t + 1];
            if (l.x > h.x) continue;   // empty tile
            lo.x = fminf(lo.x, l.x); lo.y = fminf(lo.y, l.y); lo.z = fminf(lo.z, l.z);
            hi.x = fmaxf(hi.x, h.x); hi.y = fmaxf(hi.y, h.y); hi.z = fmaxf(hi.z, h.z);
        }
        float4* o = (c == 0 ? sbox0 : sbox1) + f * 2;
        o[0] = lo;
        o[1] = hi;
    }
}

__device__ __forceinline__ float gap(float qlo, float qhi, float tlo, float thi) {
    return fmaxf(fmaxf(tlo - qhi, qlo - thi), 0.f);
}

#ifndef CD_CAND_THREADS
#define CD_CAND_THREADS 128
#endif
constexpr int kCandThreads = CD_CAND_THREADS;
__global__ void __launch_bounds__(kCandThreads) candidates_kernel(CandArgs a) {
    extern __shared__ uint32_t keys[];
    int u = blockIdx.x;
    int dir = 0;
    if (u >= a.B * a.qtiles[0]) {
        dir = 1;
        u -= a.B * a.qtiles[0];
    }
    const int b = u / a.qtiles[dir];
    const int q = u - b * a.qtiles[dir];
    const int qc = dir, tc = 1 - dir;
    const int qnt = a.ppad[qc] / kTile, tnt = a.ppad[tc] / kTile;
    // query box = union of its kCandQ / kBlockK 32-point block boxes
    float qlo[3] = {INFINITY, INFINITY, INFINITY}, qhi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int s = 0; s < kCandQ / kBlockK; ++s) {
        const float4* bx = a.box32[qc] + ((int64_t)b * qnt * kBlocksPerTile + q * (kCandQ / kBlockK) + s) * 2;
        const float4 lo = bx[0], hi = bx[1];
        qlo[0] = fminf(qlo[0], lo.x); qlo[1] = fminf(qlo[1], lo.y); qlo[2] = fminf(qlo[2], lo.z);
        qhi[0] = fmaxf(qhi[0], hi.x); qhi[1] = fmaxf(qhi[1], hi.y); qhi[2] = fmaxf(qhi[2], hi.z);
    }
    // Upper bound UB of every row's final minimum: each row's nearest target is at most as far as any
    // point of any non-empty tile, i.e. the farthest box-to-box corner distance (x (1 + 1e-5): an
    // upper bound of the fp32-evaluated distance too).  Tiles with LB > UB can never be visited
    // (the kernel stops at LB > max over rows of the current minimum <= UB): the list keeps only
    // LB <= UB, compacted, then sorted (keys are unique, so the order is deterministic).
    __shared__ float s_ub[kCandThreads / 32];
    __shared__ int s_cnt;
    const float4* tbox = a.box[tc] + (int64_t)b * tnt * 2;
    auto far2 = [&](float4 lo, float4 hi) {   // farthest box-to-box corner distance, x (1 + 1e-5)
        const float fx = fmaxf(fabsf(hi.x - qlo[0]), fabsf(qhi[0] - lo.x));
        const float fy = fmaxf(fabsf(hi.y - qlo[1]), fabsf(qhi[1] - lo.y));
        const float fz = fmaxf(fabsf(hi.z - qlo[2]), fabsf(qhi[2] - lo.z));
        return (fx * fx + fy * fy + fz * fz) * 1.00001f;
    };
    auto tile_lb = [&](float4 lo, float4 hi) {
        if (lo.x > hi.x) return INFINITY;   // empty tile (all padding)
        const float gx = gap(qlo[0], qhi[0], lo.x, hi.x);
        const float gy = gap(qlo[1], qhi[1], lo.y, hi.y);
        const float gz = gap(qlo[2], qhi[2], lo.z, hi.z);
        return (gx * gx + gy * gy + gz * gz) * kLbScale;
    };
    auto block_min = [&](float v) {   // min over the CTA (all threads call it)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
        __syncthreads();
        if ((threadIdx.x & 31) == 0) s_ub[threadIdx.x >> 5] = v;
        __syncthreads();
        v = s_ub[0];
        for (int w = 1; w < kCandThreads / 32; ++w) v = fminf(v, s_ub[w]);
        return v;
    };
    if (threadIdx.x == 0) s_cnt = 0;
    float ub = INFINITY;
    if (a.sbox[tc] == nullptr) {
        // flat: every tile's farthest corner, then every tile's LB
        for (int t = threadIdx.x; t < tnt; t += kCandThreads) {
            const float4 lo = tbox[2 * t], hi = tbox[2 * t + 1];
            if (lo.x <= hi.x) ub = fminf(ub, far2(lo, hi));
        }
        ub = block_min(ub);
        for (int t = threadIdx.x; t < tnt; t += kCandThreads) {
            const float lb = tile_lb(tbox[2 * t], tbox[2 * t + 1]);
            if (lb <= ub) keys[atomicAdd(&s_cnt, 1)] = cand_key(lb, t);
        }
    } else {
        // two levels (large clouds): LB of every super tile (kSuper tiles; a tile's LB >= its super
        // tile's), UB from the tiles of the nearest super tile only (a minimum over fewer tiles: >= the
        // flat UB, so the list below is a superset of the flat one whose extra entries all have LB > the
        // flat UB — after the kernel's stopping point: the same tiles are visited in the same order),
        // then the tiles of the super tiles with LB <= UB
        const int tns = (tnt + kSuper - 1) / kSuper;
        const float4* sb = a.sbox[tc] + (int64_t)b * tns * 2;
        float* slb = reinterpret_cast<float*>(keys + tnt);   // [tns] super LBs (after the key area)
        __shared__ int s_sup[kPrMaxTiles / kSuper];
        __shared__ int s_nsup;
        float mlb = INFINITY;
        for (int t = threadIdx.x; t < tns; t += kCandThreads) {
            const float lb = tile_lb(sb[2 * t], sb[2 * t + 1]);
            slb[t] = lb;
            mlb = fminf(mlb, lb);
        }
        mlb = block_min(mlb);   // (contains the barriers slb needs)
        if (threadIdx.x == 0) s_nsup = 0;
        // UB over the tiles of every super tile at the minimum LB (usually one: the query's own region)
        for (int t = threadIdx.x; t < tnt; t += kCandThreads) {
            if (slb[t / kSuper] != mlb) continue;
            const float4 lo = tbox[2 * t], hi = tbox[2 * t + 1];
            if (lo.x <= hi.x) ub = fminf(ub, far2(lo, hi));
        }
        ub = block_min(ub);
        for (int t = threadIdx.x; t < tns; t += kCandThreads)
            if (slb[t] <= ub) s_sup[atomicAdd(&s_nsup, 1)] = t;
        __syncthreads();
        const int nsup = s_nsup;
        for (int i = threadIdx.x; i < nsup * kSuper; i += kCandThreads) {
            const int t = s_sup[i / kSuper] * kSuper + (i % kSuper);
            if (t >= tnt) continue;
            const float lb = tile_lb(tbox[2 * t], tbox[2 * t + 1]);
            if (lb <= ub) keys[atomicAdd(&s_cnt, 1)] = cand_key(lb, t);
        }
    }
    __syncthreads();
    const int n = s_cnt;
    const int64_t list = (int64_t)(dir == 0 ? 0 : a.B * a.qtiles[0]) + (int64_t)b * a.qtiles[dir] + q;
    uint32_t* out = a.cand + a.cand_off[dir] + ((int64_t)b * a.qtiles[dir] + q) * tnt;
    if (n <= 64) {
        // short list (the common case): one warp sorts it in registers, two keys per lane (bitonic
        // network over 64 slots by shuffles and an in-lane exchange; no block barriers)
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            uint32_t v0 = lane < n ? keys[lane] : ~0u;        // slot lane
            uint32_t v1 = lane + 32 < n ? keys[lane + 32] : ~0u;   // slot lane + 32
            for (int k = 2; k <= 64; k <<= 1) {
                for (int j = k >> 1; j > 0; j >>= 1) {
                    if (j == 32) {   // partner slot is in the same lane
                        const bool up = (lane & k) == 0;   // k == 64: ascending
                        const uint32_t lo = min(v0, v1), hi = max(v0, v1);
                        v0 = up ? lo : hi;
                        v1 = up ? hi : lo;
                    } else {
                        const uint32_t o0 = __shfl_xor_sync(0xffffffffu, v0, j);
                        const uint32_t o1 = __shfl_xor_sync(0xffffffffu, v1, j);
                        const bool lower = (lane & j) == 0;
                        const bool up0 = (lane & k) == 0, up1 = ((lane + 32) & k) == 0;
                        v0 = (lower == up0) ? min(v0, o0) : max(v0, o0);
                        v1 = (lower == up1) ? min(v1, o1) : max(v1, o1);
                    }
                }
            }
            if (lane < n) out[lane] = v0;
            if (lane + 32 < n) out[lane + 32] = v1;
            if (lane == 0) a.ccount[list] = n;
        }
        return;
    }
    int npow = 1;
    while (npow < n) npow <<= 1;
    for (int t = n + threadIdx.x; t < npow; t += kCandThreads) keys[t] = ~0u;
    __syncthreads();
    // bitonic sort ascending (npow <= kPrMaxTiles)
    for (int k = 2; k <= npow; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < npow; i += kCandThreads) {
                const int l = i ^ j;
                if (l > i) {
                    const uint32_t x = keys[i], y = keys[l];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        keys[i] = y;
                        keys[l] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int t = threadIdx.x; t < n; t += kCandThreads) out[t] = keys[t];
    if (threadIdx.x == 0) a.ccount[list] = n;
}

// --------------------------------------------------------------------------------------------- main kernel
struct PrunedArgs {
    const float4* sorted[2];
    const float4* bbox32[2];
    const float4* tbox[2];    // 512-point tile boxes
    int npts[2], ppad[2];
    int qtiles[2];        // query tiles (kPrQ rows)
    int cqtiles[2];       // candidate lists (kCandQ rows): query tile u reads list u / (kCandQ / kPrQ)
    int64_t cand_off[2];
    const uint32_t* cand;
    const int* ccount;    // entries per list (candidates_kernel)
    float* best_d[2];     // [B][npts] sorted order
    int* best_blk[2];     // sorted target position of the winning block
};

__device__ __forceinline__ float box_lb(const float wlo[3], const float whi[3], float4 lo, float4 hi) {
    const float gx = gap(wlo[0], whi[0], lo.x, hi.x);
    const float gy = gap(wlo[1], whi[1], lo.y, hi.y);
    const float gz = gap(wlo[2], whi[2], lo.z, hi.z);
    return (gx * gx + gy * gy + gz * gz) * kLbScale;
}

#ifdef CD_PR_STATS
__device__ unsigned long long g_pr_stats[4];
#endif
#ifndef CD_PR_STAGES
#define CD_PR_STAGES 2
#endif
constexpr int kPrStages = CD_PR_STAGES;   // TMA ring depth of the pruned kernel
#ifndef CD_PR_MINB
#define CD_PR_MINB 4
#endif
__global__ void __launch_bounds__(kPrThreads, CD_PR_MINB) nn_pruned_kernel(PrunedArgs a) {
    __shared__ __align__(128) float4 sm[kPrStages][kTile];
    __shared__ __align__(128) float4 smb[kPrStages][kBlocksPerTile * 2];   // the tile's 32-point block boxes
    __shared__ __align__(8) u64 full_bar[kPrStages];
    __shared__ unsigned s_wmax[kPrThreads / 32];
#ifdef CD_PR_STATS
    __shared__ int s_used;
    if (threadIdx.x == 0) s_used = 0;
#endif

    int u = blockIdx.x;
    const int b = blockIdx.y;
    int dir = 0;
    if (u >= a.qtiles[0]) {
        dir = 1;
        u -= a.qtiles[0];
    }
    const int qc = dir, tc = 1 - dir;
    const int P = a.npts[qc];
    const int tnt = a.ppad[tc] / kTile;
    const float4* __restrict__ Q = a.sorted[qc] + (int64_t)b * a.ppad[qc];
    const float4* __restrict__ T = a.sorted[tc] + (int64_t)b * a.ppad[tc];
    const float4* __restrict__ TB = a.bbox32[tc] + (int64_t)b * tnt * kBlocksPerTile * 2;
    // the list of the kCandQ-row group holding this tile: sorted by the group box's LB, a lower bound
    // of this tile's (the group box contains it) — every skipped tile still has LB > every row's minimum
    const int cu = u / (kCandQ / kPrQ);
    const uint32_t* __restrict__ cand =
        a.cand + a.cand_off[dir] + ((int64_t)b * a.cqtiles[dir] + cu) * tnt;
    const int ncand = a.ccount[(int64_t)(dir == 0 ? 0 : (int64_t)gridDim.y * a.cqtiles[0]) + (int64_t)b * a.cqtiles[dir] + cu];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPrStages; ++s) mbar_init(&full_bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const int qbase = u * kPrQ + threadIdx.x * kPrR;
    u64 qx[kPrR / 2], qy[kPrR / 2], qz[kPrR / 2];
#pragma unroll
    for (int r = 0; r < kPrR / 2; ++r) {
        const float4 p0 = Q[min(qbase + 2 * r, P - 1)];
        const float4 p1 = Q[min(qbase + 2 * r + 1, P - 1)];
        qx[r] = pk2(p0.x, p1.x);
        qy[r] = pk2(p0.y, p1.y);
        qz[r] = pk2(p0.z, p1.z);
    }
    float best[kPrR];
    int blk[kPrR];
    bool tie[kPrR];
#pragma unroll
    for (int r = 0; r < kPrR; ++r) {
        best[r] = INFINITY;
        blk[r] = -1;
        tie[r] = false;
    }
    // box of this lane's rows (valid rows only): a tile is fetched, and a 32-target block inside it
    // evaluated, only if some lane may still improve (or tie) one of its rows
    float llo[3] = {INFINITY, INFINITY, INFINITY}, lhi[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int r = 0; r < kPrR / 2; ++r) {
        float v0, v1;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            upk2(q == 0 ? qx[r] : (q == 1 ? qy[r] : qz[r]), v0, v1);
            if (qbase + 2 * r < P) { llo[q] = fminf(llo[q], v0); lhi[q] = fmaxf(lhi[q], v0); }
            if (qbase + 2 * r + 1 < P) { llo[q] = fminf(llo[q], v1); lhi[q] = fmaxf(lhi[q], v1); }
        }
    }
    // the warp's union box (all its lanes' rows): a block whose LB against it exceeds the warp's largest
    // row minimum is needed by no lane (each lane box lies inside it)
    float wlo[3], whi[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        wlo[q] = llo[q];
        whi[q] = lhi[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            wlo[q] = fminf(wlo[q], __shfl_xor_sync(0xffffffffu, wlo[q], o));
            whi[q] = fmaxf(whi[q], __shfl_xor_sync(0xffffffffu, whi[q], o));
        }
    }
    auto lane_max = [&]() {
        float lmax = -1.0f;   // no valid row: never needs anything
#pragma unroll
        for (int r = 0; r < kPrR; ++r)
            if (qbase + r < P) lmax = fmaxf(lmax, best[r]);
        return lmax;
    };
    const float4* __restrict__ TT = a.tbox[tc] + (int64_t)b * tnt * 2;
    // next candidate tile that some thread still needs (list order = ascending LB of the query tile;
    // the walk ends at the first LB above every row's minimum).  CTA-uniform; one barrier per
    // candidate considered.
    int pos = 0;
    auto advance = [&]() -> int {
        unsigned m = 0u;
#pragma unroll
        for (int r = 0; r < kPrR; ++r)
            if (qbase + r < P) m = max(m, __float_as_uint(best[r]));
        m = __reduce_max_sync(0xffffffffu, m);
        if (lane == 0) s_wmax[warp] = m;
        __syncthreads();
        unsigned mm = s_wmax[0];
#pragma unroll
        for (int w = 1; w < kPrThreads / 32; ++w) mm = max(mm, s_wmax[w]);
        const float maxbest = __uint_as_float(mm);
        const float lmax = lane_max();
        int found = -1;
        while (pos < ncand) {
            const uint32_t e = cand[pos];
            if (cand_lb(e) > maxbest) {
                pos = ncand;
                break;
            }
            const int t = cand_tile(e);
            ++pos;
#ifdef CD_PR_STATS
            if (threadIdx.x == 0) atomicAdd(&g_pr_stats[3], 1ull);
#endif
            const bool need = box_lb(llo, lhi, TT[2 * t], TT[2 * t + 1]) <= lmax;
            if (__syncthreads_or(need)) {
                found = t;
                break;
            }
        }
        __syncthreads();   // s_wmax reuse
        return found;
    };
    auto issue = [&](int t, int s) {
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[s], kTile * 16 + kBlocksPerTile * 32);
            tma_load_1d(sm[s], T + (int64_t)t * kTile, kTile * 16, &full_bar[s]);
            tma_load_1d(smb[s], TB + (int64_t)t * kBlocksPerTile * 2, kBlocksPerTile * 32, &full_bar[s]);
        }
    };
    int tiles[kPrStages];
    int tail = 0;
#pragma unroll
    for (int k = 0; k < kPrStages; ++k) {
        const int t = advance();
        tiles[k] = t;
        if (t < 0) break;
        issue(t, k);
        ++tail;
    }
    for (int head = 0; head < tail; ++head) {
        const int s = head % kPrStages;
        int t = tiles[0];
#pragma unroll
        for (int q = 1; q < kPrStages; ++q) t = s == q ? tiles[q] : t;
        mbar_wait(&full_bar[s], (head / kPrStages) & 1);
        const float4* tb = sm[s];
        const float4* bb = smb[s];
        const int jt = t * kTile;
        // the tile's blocks some lane may still need, one lane per block against the warp's union box
        // and largest row minimum (a superset: the exact per-lane test below decides)
        unsigned bmask;
        {
            const float wmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(lane_max(), 0.f))));
            bool wneed = false;
            if (lane < kBlocksPerTile) wneed = box_lb(wlo, whi, bb[2 * lane], bb[2 * lane + 1]) <= wmax;
            bmask = __ballot_sync(0xffffffffu, wneed);
        }
        while (bmask) {
            const int kb = (__ffs(bmask) - 1) * kBlockK;
            bmask &= bmask - 1;
            // skip unless some lane may improve or tie: LB(lane box, block) <= the lane's largest minimum
            {
                float lmax = -1.0f;   // no valid row: never needs a block
#pragma unroll
                for (int r = 0; r < kPrR; ++r)
                    if (qbase + r < P) lmax = fmaxf(lmax, best[r]);
                const bool need = box_lb(llo, lhi, bb[2 * (kb / kBlockK)], bb[2 * (kb / kBlockK) + 1]) <= lmax;
                if (!__any_sync(0xffffffffu, need)) continue;
#ifdef CD_PR_STATS
                if (lane == 0) { atomicAdd(&g_pr_stats[1], 1ull); s_used = 1; }
#endif
            }
            float cur[kPrR], cur2[kPrR];   // this block's minimum per row: two independent fold chains
#pragma unroll
            for (int r = 0; r < kPrR; ++r) {
                cur[r] = INFINITY;
                cur2[r] = INFINITY;
            }
            auto fold_pair = [&](const float4 t0, const float4 t1, float* acc) {
                const u64 t0x = pk2(t0.x, t0.x), t0y = pk2(t0.y, t0.y), t0z = pk2(t0.z, t0.z);
                const u64 t1x = pk2(t1.x, t1.x), t1y = pk2(t1.y, t1.y), t1z = pk2(t1.z, t1.z);
#pragma unroll
                for (int r = 0; r < kPrR / 2; ++r) {
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
                    acc[2 * r] = fmin3(acc[2 * r], a0, c0);
                    acc[2 * r + 1] = fmin3(acc[2 * r + 1], a1, c1);
                }
            };
#pragma unroll 2
            for (int jj = 0; jj < kBlockK; jj += 4) {
                fold_pair(tb[kb + jj], tb[kb + jj + 1], cur);
                fold_pair(tb[kb + jj + 2], tb[kb + jj + 3], cur2);
            }
#pragma unroll
            for (int r = 0; r < kPrR; ++r) cur[r] = fminf(cur[r], cur2[r]);   // min: order-free, exact
            // a strictly smaller block minimum takes over; an EQUAL finite one is an exact tie across
            // blocks (Hilbert order is not index order): flagged, the resolve then scans the row
#pragma unroll
            for (int r = 0; r < kPrR; ++r) {
                const bool lt = cur[r] < best[r];
                const bool eq = cur[r] == best[r] && cur[r] < INFINITY;
                blk[r] = lt ? jt + kb : blk[r];
                tie[r] = lt ? false : (eq || tie[r]);
                best[r] = fminf(best[r], cur[r]);
            }
        }
        __syncthreads();   // stage s consumed by every warp
        const int tn = advance();
        if (tn >= 0) {
#pragma unroll
            for (int q = 0; q < kPrStages; ++q) tiles[q] = s == q ? tn : tiles[q];
            issue(tn, s);
            ++tail;
        }
    }

    const int64_t rowbase = (int64_t)b * P;
#pragma unroll
    for (int r = 0; r < kPrR; ++r) {
        const int q = qbase + r;
        if (q < P) {
            a.best_d[dir][rowbase + q] = best[r];
            a.best_blk[dir][rowbase + q] = (blk[r] >= 0 && tie[r]) ? (blk[r] | (int)0x80000000) : blk[r];
        }
    }
}

// --------------------------------------------------------------------------------------------- resolve
struct PrResolveArgs {
    const float4* sorted[2];
    const int* perm[2];
    int npts[2], ppad[2];
    int B;
    int nchunks[2];
    int64_t chunk_off[2];
    const float* best_d[2];
    const int* best_blk[2];
    float* d_out[2];
    int32_t* idx_out[2];
    double* chunk_sum;
    int* chunk_hits;
    double tau2;
    unsigned* fb_count;    // rows with an exact tie across blocks (full scan: lowest original index)
    unsigned* fb_list;     // (dir << 31) | b * P + p
};

__global__ void __launch_bounds__(kMergeThreads) pruned_resolve_kernel(PrResolveArgs a) {
    int u = blockIdx.x;
    int dir = 0;
    if (u >= a.B * a.nchunks[0]) {
        dir = 1;
        u -= a.B * a.nchunks[0];
    }
    const int b = u / a.nchunks[dir];
    const int chunk = u - b * a.nchunks[dir];
    const int qc = dir, tc = 1 - dir;
    const int P = a.npts[qc];
    const int p = chunk * kMergeThreads + threadIdx.x;
    double v = 0.0;
    int h = 0;
    float best = INFINITY;
    int bb = -1;
    bool tie = false;
    float4 qp = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p < P) {
        best = a.best_d[dir][(int64_t)b * P + p];
        const int bbt = a.best_blk[dir][(int64_t)b * P + p];
        tie = bbt != -1 && (bbt & (int)0x80000000) != 0;
        bb = bbt == -1 ? -1 : (bbt & 0x7fffffff);
        CD_CHECK(bb < a.ppad[tc]);
        if (bb >= 0) qp = a.sorted[qc][(int64_t)b * a.ppad[qc] + p];
    }
    // the lowest ORIGINAL index among the winning block's targets at the minimum distance, warp-
    // cooperatively: the warp's 32 rows staged in shared memory, then per row the 32 lanes load the
    // block's 32 sorted targets (one coalesced 512-B read, 8 rows in flight), the matching lanes their
    // original indices, and one REDUX.MIN; targets past the cloud are the +inf padding (bb + 31 < ppad)
    __shared__ float4 s_q[kMergeThreads];
    __shared__ int s_b[kMergeThreads];
    s_q[threadIdx.x] = make_float4(qp.x, qp.y, qp.z, best);
    s_b[threadIdx.x] = bb;
    __syncwarp();
    const int lane = threadIdx.x & 31, wb = threadIdx.x & ~31;
    const float4* T = a.sorted[tc] + (int64_t)b * a.ppad[tc];
    const int* PT = a.perm[tc] + (int64_t)b * a.npts[tc];
    const int nt = a.npts[tc];
    unsigned myidx = 0xffffffffu;
    constexpr int kRowsInFlight = 8;
    for (int r0 = 0; r0 < 32; r0 += kRowsInFlight) {
        int base[kRowsInFlight];
        float4 t[kRowsInFlight];
#pragma unroll
        for (int k = 0; k < kRowsInFlight; ++k) {
            base[k] = s_b[wb + r0 + k];
            t[k] = T[max(base[k], 0) + lane];
        }
#pragma unroll
        for (int k = 0; k < kRowsInFlight; ++k) {
            const float4 q = s_q[wb + r0 + k];
            const float d = dist_rn(q.x, q.y, q.z, t[k].x, t[k].y, t[k].z);
            const int j = base[k] + lane;
            const bool m = base[k] >= 0 && j < nt && d == q.w;
            const unsigned o = m ? (unsigned)PT[j] : 0xffffffffu;
            const unsigned low = __reduce_min_sync(0xffffffffu, o);
            myidx = lane == r0 + k ? low : myidx;
        }
    }
    if (p < P) {
        const int idx = (bb >= 0 && myidx != 0xffffffffu) ? (int)myidx : -1;
        if (bb >= 0 && tie) {
            const unsigned slot = atomicAdd(a.fb_count, 1u);
            a.fb_list[slot] = ((unsigned)dir << 31) | (unsigned)((int64_t)b * P + p);
        }
        const int i = a.perm[qc][(int64_t)b * P + p];
        a.d_out[dir][(int64_t)b * P + i] = best;
        a.idx_out[dir][(int64_t)b * P + i] = idx;
        v = (double)best;
        h = (a.tau2 >= 0.0 && (double)best <= a.tau2) ? 1 : 0;
    }
    // fixed-order block reduction
    __shared__ double ssum[kMergeThreads / 32];
    __shared__ int shit[kMergeThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_down_sync(0xffffffffu, v, o);
        h += __shfl_down_sync(0xffffffffu, h, o);
    }
    if ((threadIdx.x & 31) == 0) {
        ssum[threadIdx.x >> 5] = v;
        shit[threadIdx.x >> 5] = h;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        int t = 0;
        for (int w = 0; w < kMergeThreads / 32; ++w) {
            s += ssum[w];
            t += shit[w];
        }
        const int64_t c = a.chunk_off[dir] + (int64_t)b * a.nchunks[dir] + chunk;
        a.chunk_sum[c] = s;
        a.chunk_hits[c] = t;
    }
}

// Rows whose minimum is attained in more than one block: scan every target (sorted clouds) for the
// lowest original index at the minimum distance (the distance itself is already final).  One CTA
// per queued row.
__global__ void __launch_bounds__(256) pruned_tie_kernel(PrResolveArgs a) {
    constexpr int kChunk = 256 * 16;   // targets per work item (16 per thread)
    const unsigned count = *a.fb_count;
    const int nchunk = (max(a.npts[0], a.npts[1]) + kChunk - 1) / kChunk;
    __shared__ int sidx[8];
    for (int64_t w = blockIdx.x; w < (int64_t)count * nchunk; w += gridDim.x) {
        const unsigned item = a.fb_list[w / nchunk];
        const int c = (int)(w % nchunk);
        const int dir = (int)(item >> 31);
        const int64_t g = item & 0x7fffffffu;
        const int qc = dir, tc = 1 - dir;
        const int P = a.npts[qc];
        const int b = (int)(g / P);
        const int p = (int)(g - (int64_t)b * P);
        const int nT = a.npts[tc];
        const int j0 = c * kChunk;
        if (j0 >= nT) continue;   // uniform across the CTA
        const float best = a.best_d[dir][g];
        const float4 qp = a.sorted[qc][(int64_t)b * a.ppad[qc] + p];
        const float4* T = a.sorted[tc] + (int64_t)b * a.ppad[tc];
        const int* PT = a.perm[tc] + (int64_t)b * a.npts[tc];
        int idx = 0x7fffffff;
        float4 t[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) t[u] = T[min(j0 + 256 * u + (int)threadIdx.x, nT - 1)];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int j = j0 + 256 * u + (int)threadIdx.x;
            if (j < nT && dist_rn(qp.x, qp.y, qp.z, t[u].x, t[u].y, t[u].z) == best) idx = min(idx, PT[j]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) idx = min(idx, __shfl_xor_sync(0xffffffffu, idx, o));
        if ((threadIdx.x & 31) == 0) sidx[threadIdx.x >> 5] = idx;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < 8; ++k) idx = min(idx, sidx[k]);
            const int i = a.perm[qc][(int64_t)b * P + p];
            // the resolve stored a tie index of the winning block; the minimum over all chunks is the
            // lowest original index at the minimum distance (integer min: order-independent)
            if (idx != 0x7fffffff) atomicMin(&a.idx_out[dir][(int64_t)b * P + i], idx);
        }
        __syncthreads();
    }
}

// --------------------------------------------------------------------------------------------- host
// Bits per axis of the Hilbert codes (segment-local keys of 3k bits): the smallest k that leaves
// <= ~8 points per occupied surface cell (4^k >= n / 48), at least 6 (18-bit keys: 2 radix passes of
// 9 bits), at most 10.  Measured on the pruned forward (r02_experiments.txt): c4 (100k points) k = 5 /
// 6 / 7: 1.050 / 0.972 / 0.998 ms; c5 (1M points) k = 7 / 8 / 9 / 10: 6.34 / 6.17 / 6.42 / 6.50 ms.
// The order only affects how much is culled, never the results.
int hilbert_bits(int nmax) {
    int need = 1;
    while (((int64_t)1 << (2 * need)) * 48 < (int64_t)nmax) ++need;
    return std::min(10, std::max(6, need));
}

static int cdiv(int64_t x, int64_t y) { return (int)((x + y - 1) / y); }

void plan_pruned(PrunedPlan& p, int B, int N, int M) {
    p.B = B;
    p.npts[0] = N;
    p.npts[1] = M;
    for (int c = 0; c < 2; ++c) {
        const int unit = std::max(kPrQ, kTile);
        p.ppad[c] = cdiv(p.npts[c], unit) * unit;
        p.qtiles[c] = cdiv(p.npts[c], kPrQ);
        p.cqtiles[c] = cdiv(p.npts[c], kCandQ);
        p.ttiles[c] = p.ppad[c] / kTile;
    }
    p.kbits = hilbert_bits(std::max(N, M));
    p.nbits = 3 * p.kbits;
    p.segs = SegSpec{B, N, B, M};
    p.L = (int64_t)B * (N + M);
    p.cand_off[0] = 0;
    p.cand_off[1] = (int64_t)B * p.cqtiles[0] * p.ttiles[1];
    const int64_t ncand = p.cand_off[1] + (int64_t)B * p.cqtiles[1] * p.ttiles[0];
    p.nchunks[0] = cdiv(N, kMergeThreads);
    p.nchunks[1] = cdiv(M, kMergeThreads);
    p.chunk_off[0] = 0;
    p.chunk_off[1] = (int64_t)B * p.nchunks[0];
    const int64_t chunks = p.chunk_off[1] + (int64_t)B * p.nchunks[1];
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
    for (int c = 0; c < 2; ++c) {
        p.off_sorted[c] = take((size_t)B * p.ppad[c] * 16);
        p.off_perm[c] = take((size_t)B * p.npts[c] * 4);
        p.off_box[c] = take((size_t)B * p.ttiles[c] * 32);
        p.off_box32[c] = take((size_t)B * p.ttiles[c] * kBlocksPerTile * 32);
        p.off_best_d[c] = take((size_t)B * p.npts[c] * 4);
        p.off_best_blk[c] = take((size_t)B * p.npts[c] * 4);
        p.off_sbox[c] = take((size_t)B * ((p.ttiles[c] + kSuper - 1) / kSuper) * 32);
    }
    p.hier = CD_PR_HIER && std::max(p.ttiles[0], p.ttiles[1]) >= kHierMinTiles;
    p.off_cand = take((size_t)ncand * 4);
    p.off_ccount = take((size_t)B * (p.cqtiles[0] + p.cqtiles[1]) * 4);
    p.off_chunk_sum = take((size_t)chunks * 8);
    p.off_chunk_hits = take((size_t)chunks * 4);
    p.off_fb = take(256 + (size_t)p.L * 4);
    p.bytes = off;
    p.supported = p.ttiles[0] <= kPrMaxTiles && p.ttiles[1] <= kPrMaxTiles;
}

#ifndef CD_PR_SEGSORT
#define CD_PR_SEGSORT 1
#endif
// clouds of <= kSegMax points: the on-chip Hilbert sort (pr_segsort_kernel)
static bool pruned_segsort(const PrunedPlan& p) {
    return CD_PR_SEGSORT && std::max(p.npts[0], p.npts[1]) <= kSegMax;
}

int pruned_launches(const PrunedPlan& p) {
    // segment sort: sort+boxes, candidates, kernel, resolve, tie, partials (+ super boxes)
    return (pruned_segsort(p) ? 6 : 2 + radix_sort_launches(p.segs, p.nbits, true) + 7) + (p.hier ? 1 : 0);
}

cudaError_t launch_pruned(const PrunedPlan& p, const float* x, const float* y, const FwdOutputs& o, void* ws,
                          cudaStream_t st) {
    char* w = static_cast<char*>(ws);
    const int sms = current_sm_count();
    float* bbox = reinterpret_cast<float*>(w + p.off_bbox);
    const bool segsort = pruned_segsort(p);
    if (!segsort) launch_bbox(x, p.npts[0], y, p.npts[1], p.B, bbox, st);
    uint32_t* keys[2] = {reinterpret_cast<uint32_t*>(w + p.off_keys[0]), reinterpret_cast<uint32_t*>(w + p.off_keys[1])};
    uint32_t* vals[2] = {reinterpret_cast<uint32_t*>(w + p.off_vals[0]), reinterpret_cast<uint32_t*>(w + p.off_vals[1])};
    const int grid_l = (int)std::min<int64_t>((p.L + 255) / 256, (int64_t)sms * 16);
    float4* sorted[2];
    int* perm[2];
    float4* box[2];
    float4* box32[2];
    for (int c = 0; c < 2; ++c) {
        sorted[c] = reinterpret_cast<float4*>(w + p.off_sorted[c]);
        perm[c] = reinterpret_cast<int*>(w + p.off_perm[c]);
        box[c] = reinterpret_cast<float4*>(w + p.off_box[c]);
        box32[c] = reinterpret_cast<float4*>(w + p.off_box32[c]);
    }
    if (segsort) {   // sort + element boxes + tile / block boxes in one launch
        PrSegArgs a;
        a.src[0] = x;
        a.src[1] = y;
        a.B = p.B;
        a.nmax = std::max(p.npts[0], p.npts[1]);
        a.fb_count = reinterpret_cast<unsigned*>(w + p.off_fb);
        for (int c = 0; c < 2; ++c) {
            a.npts[c] = p.npts[c];
            a.ppad[c] = p.ppad[c];
            a.sorted[c] = sorted[c];
            a.perm[c] = perm[c];
            a.box[c] = box[c];
            a.bbox32[c] = box32[c];
        }
        const size_t smem = seg_sort_smem(a.nmax);
        ensure_smem_attr((const void*)pr_segsort_kernel, (int)seg_sort_smem(kSegMax));
        pr_segsort_kernel<<<2 * p.B, kSegThreads, smem, st>>>(a);
    } else {
    {
        HilbertArgs a;
        a.src[0] = x;
        a.src[1] = y;
        a.npts[0] = p.npts[0];
        a.npts[1] = p.npts[1];
        a.B = p.B;
        a.kbits = p.kbits;
        a.bbox = bbox;
        a.keys = keys[0];
        a.vals = vals[0];
        a.fb_count = reinterpret_cast<unsigned*>(w + p.off_fb);
        hilbert_kernel<<<grid_l, 256, 0, st>>>(a);
    }
    const int cur = radix_sort_pairs(keys, vals, p.segs, p.nbits, reinterpret_cast<uint32_t*>(w + p.off_counts),
                                     reinterpret_cast<uint32_t*>(w + p.off_totals), st, false, true);
    {
        GatherArgs a;
        a.src[0] = x;
        a.src[1] = y;
        a.B = p.B;
        a.vals = vals[cur];
        for (int c = 0; c < 2; ++c) {
            a.npts[c] = p.npts[c];
            a.ppad[c] = p.ppad[c];
            a.sorted[c] = sorted[c];
            a.perm[c] = perm[c];
        }
        gather_kernel<<<grid_l, 256, 0, st>>>(a);
    }
    }
    if (!segsort) {
        AabbArgs a;
        a.B = p.B;
        for (int c = 0; c < 2; ++c) {
            a.sorted[c] = sorted[c];
            a.npts[c] = p.npts[c];
            a.ppad[c] = p.ppad[c];
            a.box[c] = box[c];
            a.bbox32[c] = box32[c];
        }
        const int64_t tiles = (int64_t)p.B * (p.ttiles[0] + p.ttiles[1]);
        aabb_kernel<<<cdiv(tiles * 32, 256), 256, 0, st>>>(a);
    }
    uint32_t* cand = reinterpret_cast<uint32_t*>(w + p.off_cand);
    float4* sbox[2] = {reinterpret_cast<float4*>(w + p.off_sbox[0]), reinterpret_cast<float4*>(w + p.off_sbox[1])};
    if (p.hier) {
        const int64_t n = (int64_t)p.B * ((p.ttiles[0] + kSuper - 1) / kSuper + (p.ttiles[1] + kSuper - 1) / kSuper);
        superbox_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 4)), 256, 0,
                          st>>>(box[0], box[1], p.ttiles[0], p.ttiles[1], p.B, sbox[0], sbox[1]);
    }
    {
        CandArgs a;
        a.B = p.B;
        for (int c = 0; c < 2; ++c) {
            a.box[c] = box[c];
            a.box32[c] = box32[c];
            a.ppad[c] = p.ppad[c];
            a.qtiles[c] = p.cqtiles[c];
            a.cand_off[c] = p.cand_off[c];
            a.sbox[c] = p.hier ? sbox[c] : nullptr;
        }
        a.cand = cand;
        a.ccount = reinterpret_cast<int*>(w + p.off_ccount);
        int npow = 1;
        while (npow < std::max(p.ttiles[0], p.ttiles[1])) npow <<= 1;
        // keys (npow u64) + the super LBs (two-level search: ceil(T / kSuper) floats)
        const size_t smem = (size_t)npow * 4 + (size_t)(std::max(p.ttiles[0], p.ttiles[1]) / kSuper + 1) * 4;
        ensure_smem_attr((const void*)candidates_kernel, kPrMaxTiles * 4 + (kPrMaxTiles / kSuper + 1) * 4);
        candidates_kernel<<<p.B * (p.cqtiles[0] + p.cqtiles[1]), kCandThreads, smem, st>>>(a);
    }
    float* best_d[2];
    int* best_blk[2];
    for (int c = 0; c < 2; ++c) {
        best_d[c] = reinterpret_cast<float*>(w + p.off_best_d[c]);
        best_blk[c] = reinterpret_cast<int*>(w + p.off_best_blk[c]);
    }
    {
        PrunedArgs a;
        for (int c = 0; c < 2; ++c) {
            a.sorted[c] = sorted[c];
            a.bbox32[c] = box32[c];
            a.tbox[c] = box[c];
            a.npts[c] = p.npts[c];
            a.ppad[c] = p.ppad[c];
            a.qtiles[c] = p.qtiles[c];
            a.cqtiles[c] = p.cqtiles[c];
            a.cand_off[c] = p.cand_off[c];
            a.best_d[c] = best_d[c];
            a.best_blk[c] = best_blk[c];
        }
        a.cand = cand;
        a.ccount = reinterpret_cast<const int*>(w + p.off_ccount);
        if (g_prof_start) record_profile_event(g_prof_start, st);
        nn_pruned_kernel<<<dim3(p.qtiles[0] + p.qtiles[1], p.B), kPrThreads, 0, st>>>(a);
        if (g_prof_stop) record_profile_event(g_prof_stop, st);
    }
    double* chunk_sum = reinterpret_cast<double*>(w + p.off_chunk_sum);
    int* chunk_hits = reinterpret_cast<int*>(w + p.off_chunk_hits);
    {
        PrResolveArgs a;
        a.B = p.B;
        for (int c = 0; c < 2; ++c) {
            a.sorted[c] = sorted[c];
            a.perm[c] = perm[c];
            a.npts[c] = p.npts[c];
            a.ppad[c] = p.ppad[c];
            a.nchunks[c] = p.nchunks[c];
            a.chunk_off[c] = p.chunk_off[c];
            a.best_d[c] = best_d[c];
            a.best_blk[c] = best_blk[c];
            a.d_out[c] = o.d[c];
            a.idx_out[c] = o.idx[c];
        }
        a.chunk_sum = chunk_sum;
        a.chunk_hits = chunk_hits;
        a.tau2 = o.tau >= 0.f ? (double)o.tau * (double)o.tau : -1.0;
        a.fb_count = reinterpret_cast<unsigned*>(w + p.off_fb);
        a.fb_list = a.fb_count + 64;
        pruned_resolve_kernel<<<p.B * (p.nchunks[0] + p.nchunks[1]), kMergeThreads, 0, st>>>(a);
        pruned_tie_kernel<<<sms * 4, 256, 0, st>>>(a);
#ifdef CD_PR_STATS
        unsigned h = 0;
        cudaStreamSynchronize(st);
        cudaMemcpy(&h, a.fb_count, 4, cudaMemcpyDeviceToHost);
        printf("pruned tie rows: %u of %lld\n", h, (long long)p.L);
        unsigned long long st3[4];
        cudaMemcpyFromSymbol(st3, g_pr_stats, sizeof(st3));
        printf("candidates considered %llu, tiles fetched %llu, tiles with >= 1 evaluated block %llu, warp-blocks evaluated %llu\n", st3[3], st3[0], st3[2], st3[1]);
        unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(g_pr_stats, z, sizeof(z));
#endif
    }
    if (o.partials) {
        cudaError_t e = launch_partials(chunk_sum, chunk_hits, p.nchunks, p.chunk_off, p.B, o.partials, 3, st);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

}  // namespace cdk
