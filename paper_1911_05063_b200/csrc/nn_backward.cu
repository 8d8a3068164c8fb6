// nn_backward.cu — backward of the Chamfer per-point distances, argmin held fixed
// (SURVEY.md §8.a.6-a.8).  Deterministic and free of floating-point atomics.
//
// Clouds of <= kSegMax points (c1-c3): seg_sort_grad_kernel, ONE launch: one or 2^p CTAs per
// (direction, batch) segment sort the segment's edges on chip (stable LSD, see below), fill the key
// offsets in shared memory and write the gradients of the part's targets.  Larger clouds (c4, c5),
// the 2B (direction, batch) segments sorted as independent segments with segment-local keys:
//
//   keys_hist_kernel one (key, value) pair per NN edge: xy edge i -> a_i gets key a_i (segment b),
//                    yx edge j -> b_j gets key b_j (segment B + b); value = the source row.  Built in
//                    ascending source order; also the first radix pass's per-tile histogram.
//   radix passes     stable LSD radix sort by key, digits of <= 11 bits (widths from a measured
//                    per-width cost), reduce-then-scan:
//                      radix_hist_kernel   per-tile digit histograms (shared-memory integer adds)
//                      radix_rowscan_kernel exclusive scan of each (segment, digit) row of tile counts
//                                          (one warp per row; the digit bases are scanned inside
//                                          the scatter kernel)
//                      radix_scatter_kernel stable in-tile ranks (warp ballot multisplit + per-warp
//                                          counts in element order) -> scatter.  Stability keeps ascending
//                                          source rows inside every key segment.
//   offsets_kernel   global key offsets from the sorted keys (disjoint gap fills, no atomics).
//   grad_kernel      one thread per output point (batch-major): own term 2 g (p - partner) then the
//                    segment's scatter terms in ascending source order, accumulated in fp64 with
//                    explicit .rn ops (no contraction), one fp32 store.
#include "cd_device.cuh"
#include "cd_internal.h"
#include "seg_sort.cuh"

#include <algorithm>

namespace cdk {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
#ifndef CD_SORT_ITEMS
#define CD_SORT_ITEMS 16
#endif
#ifndef CD_SORT_MINB
#define CD_SORT_MINB 1
#endif
constexpr int kSortItems = CD_SORT_ITEMS;           // elements per thread per tile (digits <= 9 bits)
constexpr int kSortItemsWide = 24;                   // ... for 10-11-bit digits: the per-tile digit scans
                                                     // (8 warps x D counters) amortised over 1.5x the tile
// elements per thread of a sort whose digits have `digit_bits` bits (measured: c4 backward, two
// 11-bit passes, 0.187 -> 0.164 ms with 24; 8-bit digits gain nothing)
inline int sort_items(int digit_bits) { return digit_bits >= 10 ? kSortItemsWide : kSortItems; }
#ifndef CD_SORT_BALLOT
#define CD_SORT_BALLOT 1
#endif
#ifndef CD_SORT_MAXBITS
#define CD_SORT_MAXBITS 11
#endif
constexpr int kMaxDigitBits = CD_SORT_MAXBITS;        // digits of up to 11 bits: 2 passes cover 2^22 keys

// Segmented sorts: the sequence is nA segments of szA elements followed by nB segments of szB, each
// sorted on its own (a plain sort is one segment).  Every tile lies inside one segment; the digit-
// major counts table holds one row of per-tile counts per (segment, digit); a segment's sorted
// output occupies its input range.  The backward's edges form 2B such segments (B of N xy edges keyed
// by a target in [0, M), B of M yx edges keyed in [0, N)), so the keys are segment-LOCAL and need
// ceil(log2(max(N, M))) bits instead of log2(B(N + M)): c5 sorts 20-bit keys in 2 passes, not 23 in 3.
struct SortSegs {
    int nA, nB;
    int64_t szA, szB;
    int ntA, ntB;   // tiles per segment for the pass's tile size
    __host__ __device__ int64_t seg_start(int s) const { return s < nA ? s * szA : nA * szA + (s - nA) * szB; }
    __host__ __device__ int64_t seg_size(int s) const { return s < nA ? szA : szB; }
    __host__ __device__ int seg_tiles(int s) const { return s < nA ? ntA : ntB; }
    __host__ __device__ int ntiles() const { return nA * ntA + nB * ntB; }
    __host__ __device__ int nsegs() const { return nA + nB; }
    __host__ __device__ void locate(int t, int& s, int& lt) const {
        if (t < nA * ntA) {
            s = t / ntA;
            lt = t - s * ntA;
        } else {
            const int u = t - nA * ntA, q = u / ntB;
            s = nA + q;
            lt = u - q * ntB;
        }
    }
    // element range [start, end) of tile t (tile size T)
    __host__ __device__ void range(int t, int T, int& s, int& lt, int64_t& start, int64_t& end) const {
        locate(t, s, lt);
        const int64_t s0 = seg_start(s);
        start = s0 + (int64_t)lt * T;
        end = s0 + seg_size(s);
        if (start + T < end) end = start + T;
    }
    // first word of the (segment, digit) row of per-tile counts
    __host__ __device__ int64_t row(int s, int d, int D) const {
        return s < nA ? ((int64_t)s * D + d) * ntA : (int64_t)nA * D * ntA + ((int64_t)(s - nA) * D + d) * ntB;
    }
};

static SortSegs make_segs(const SegSpec& sp, int tile) {
    SortSegs g;
    g.nA = sp.nA;
    g.nB = sp.nB;
    g.szA = sp.szA;
    g.szB = sp.szB;
    g.ntA = (int)((sp.szA + tile - 1) / tile);
    g.ntB = (int)((sp.szB + tile - 1) / tile);
    return g;
}

// Edge keys fused with the first radix pass's per-tile histogram: one CTA per sort tile writes its
// (key, value) pairs and counts digit 0 (saves a launch and a read of the keys).  Segment s < B holds
// batch s's xy edges (key a_i, value the global x row), s >= B batch (s - B)'s yx edges.
template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads) keys_hist_kernel(const int32_t* __restrict__ idx_xy,
                                                                 const int32_t* __restrict__ idx_yx, int B, int N,
                                                                 int M, int D, SortSegs g, uint32_t* __restrict__ keys,
                                                                 uint32_t* __restrict__ vals,
                                                                 uint32_t* __restrict__ counts) {
    extern __shared__ uint32_t hist[];
    for (int d = threadIdx.x; d < D; d += kSortThreads) hist[d] = 0;
    __syncthreads();
    int sg, lt;
    int64_t start, end;
    g.range(blockIdx.x, kSortThreads * ITEMS, sg, lt, start, end);
    const int64_t L0 = (int64_t)B * N;
    const bool xy = sg < B;
    const int kmaxl = xy ? M - 1 : N - 1;
    const int32_t* idx = xy ? idx_xy : idx_yx - L0;   // idx[p] for p in this segment's range
#pragma unroll 4
    for (int k = 0; k < ITEMS; ++k) {
        const int64_t p = start + (int64_t)k * kSortThreads + threadIdx.x;
        if (p < end) {
            const uint32_t key = (uint32_t)min(max(idx[p], 0), kmaxl);
            keys[p] = key;
            vals[p] = (uint32_t)(xy ? p : p - L0);
            atomicAdd(&hist[key & (D - 1)], 1u);  // integer adds: order-free
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += kSortThreads) counts[g.row(sg, d, D) + lt] = hist[d];
}

// per-tile digit counts into the (segment, digit) rows; D = 1 << digit bits (dynamic smem: D words)
template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const uint32_t* __restrict__ keys, SortSegs g,
                                                                  int shift, int D, uint32_t* __restrict__ counts) {
    extern __shared__ uint32_t hist[];
    for (int d = threadIdx.x; d < D; d += kSortThreads) hist[d] = 0;
    __syncthreads();
    int sg, lt;
    int64_t start, end;
    g.range(blockIdx.x, kSortThreads * ITEMS, sg, lt, start, end);
    uint32_t kk[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {   // all loads in flight before the shared-memory adds
        const int64_t e = min(start + (int64_t)k * kSortThreads + threadIdx.x, end - 1);
        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(kk[k]) : "l"(keys + e));
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int64_t e = start + (int64_t)k * kSortThreads + threadIdx.x;
        if (e < end) atomicAdd(&hist[(kk[k] >> shift) & (D - 1)], 1u);  // integer adds: order-free
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += kSortThreads) counts[g.row(sg, d, D) + lt] = hist[d];
}

// Block-wide exclusive scan of one value per thread (kSortThreads threads); returns the block total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_tot, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint32_t before = 0, all = 0;
    for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t t = warp_tot[w];
        before += w < warp ? t : 0u;
        all += t;
    }
    __syncthreads();
    total = all;
    return before + incl - v;
}

// Row-wise exclusive scan of the counts table, one warp per (segment s, digit d) row: scans the row
// of s's tile counts for d in place (32 tiles per step, shuffle scan) and writes the row total to
// totals[s * D + d].  8 rows per CTA: short rows (many small segments) cost a warp, not a CTA.
__global__ void __launch_bounds__(kSortThreads) radix_rowscan_kernel(uint32_t* __restrict__ counts, SortSegs g, int D,
                                                                     uint32_t* __restrict__ totals) {
    const int lane = threadIdx.x & 31;
    const int64_t rowid = (int64_t)blockIdx.x * kSortWarps + (threadIdx.x >> 5);
    if (rowid >= (int64_t)g.nsegs() * D) return;   // warp-uniform
    const int sg = (int)(rowid / D), d = (int)(rowid - (int64_t)sg * D);
    const int ntiles = g.seg_tiles(sg);
    uint32_t* row = counts + g.row(sg, d, D);
    uint32_t carry = 0;
    for (int base = 0; base < ntiles; base += 32) {
        const int i = base + lane;
        const uint32_t v = i < ntiles ? row[i] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (i < ntiles) row[i] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) totals[rowid] = carry;
}

// Stable scatter of one tile.  Warp w owns elements [w*512, (w+1)*512) of the tile (16 rounds of
// 32), so tile order = (warp, round, lane).  Phase 1: per-warp digit counters in shared memory give
// every element its rank among equal digits of its warp (warp ballot multisplit; only the warp's own counter row
// is touched, no block barrier per round).  Phase 2: per digit, the tile-local start (exclusive scan
// of the tile's digit counts) plus the prefix over the warps; delta[d] = global base - local start.
// Phase 3: the tile is re-ordered by digit in shared memory, then written out so that consecutive
// threads write consecutive addresses of each digit's run (coalesced stores).
// Dynamic shared memory: (kSortWarps + 2) * D + 2 * tile words (tile = kSortThreads * ITEMS).
template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads, CD_SORT_MINB > 1 ? CD_SORT_MINB : 2) radix_scatter_kernel(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, SortSegs g, int shift, int D,
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ totals, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout) {
    extern __shared__ uint32_t smem[];
    uint32_t* wcnt = smem;                       // [kSortWarps][D]
    uint32_t* dbase = smem + kSortWarps * D;     // [D] global base of digit d for this tile
    uint32_t* delta = dbase + D;                 // [D] global base - tile-local start
    uint32_t* skey = delta + D;                  // [(kSortThreads * ITEMS)] tile re-ordered by digit
    uint32_t* sval = skey + (kSortThreads * ITEMS);
    __shared__ uint32_t warp_tot[kSortWarps];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int dbits = __ffs(D) - 1;
    const int per = (D + kSortThreads - 1) / kSortThreads;   // digits owned by this thread in the scans
    const int d0 = threadIdx.x * per;
    for (int i = threadIdx.x; i < kSortWarps * D; i += kSortThreads) wcnt[i] = 0;
    int sg, lt;
    int64_t tbase, L;   // this tile's elements [tbase, L): L is the tile's end, inside its segment
    g.range(blockIdx.x, kSortThreads * ITEMS, sg, lt, tbase, L);
    // digit bases: the segment's start + exclusive scan of its digit totals, plus this tile's
    // row-scan offset
    {
        const uint32_t* tseg = totals + (int64_t)sg * D;
        uint32_t loc = 0;
        for (int d = d0; d < min(d0 + per, D); ++d) loc += tseg[d];
        uint32_t tot;
        uint32_t run = (uint32_t)g.seg_start(sg) + block_exclusive_scan(loc, warp_tot, tot);
        for (int d = d0; d < min(d0 + per, D); ++d) {
            dbase[d] = run + offsets[g.row(sg, d, D) + lt];
            run += tseg[d];
        }
    }
    __syncthreads();
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int64_t wbase = tbase + (int64_t)warp * (ITEMS * 32);
    uint32_t kk[ITEMS], vv[ITEMS], rk[ITEMS];
    uint32_t* my = wcnt + warp * D;
    // all 16 loads first (independent: full memory-level parallelism), then the ranking rounds
    // all loads issued before the ranking rounds, as volatile loads: the compiler would otherwise
    // re-issue (rematerialise) each read-only load at its first use, exposing one memory latency per round
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int64_t e = min(wbase + k * 32 + lane, L - 1);
        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(kk[k]) : "l"(kin + e));
        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(vv[k]) : "l"(vin + e));
    }
    {
        uint32_t all = 0;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) all ^= kk[k];
        asm volatile("" ::"r"(all));   // every key has arrived before the first ranking round
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int64_t e = wbase + k * 32 + lane;
        const bool valid = e < L;
        const int digit = valid ? (int)((kk[k] >> shift) & (D - 1)) : D;  // D: sentinel group
#if CD_SORT_BALLOT
        // warp multisplit: the lanes with an equal digit = AND over the digit bits (and validity) of
        // the matching ballot or its complement.  VOTE issues at ALU rate; MATCH.ANY is a slow,
        // long-latency op (ncu: the match results were the top short-scoreboard stall, c5 scatter
        // 117 -> 100 us with ballots)
        uint32_t peers = __ballot_sync(0xffffffffu, valid);
        if (!valid) peers = ~peers;
        for (int b = 0; b < dbits; ++b) {
            const bool bit = (digit >> b) & 1;
            const uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
#else
        const uint32_t peers = __match_any_sync(0xffffffffu, digit);
#endif
        const uint32_t before = valid ? my[digit] : 0u;
        rk[k] = before + __popc(peers & lt_mask);
        __syncwarp();
        if (valid && (peers & lt_mask) == 0u) my[digit] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // tile-local digit starts (exclusive scan of the tile's digit counts) and warp prefixes
    {
        uint32_t loc = 0;
        for (int d = d0; d < min(d0 + per, D); ++d)
            for (int w = 0; w < kSortWarps; ++w) loc += wcnt[w * D + d];
        uint32_t tot;
        uint32_t run = block_exclusive_scan(loc, warp_tot, tot);
        for (int d = d0; d < min(d0 + per, D); ++d) {
            delta[d] = dbase[d] - run;
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t t = wcnt[w * D + d];
                wcnt[w * D + d] = run;
                run += t;
            }
        }
    }
    __syncthreads();
    const int nvalid = (int)min((int64_t)(kSortThreads * ITEMS), L - tbase);
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int64_t e = wbase + k * 32 + lane;
        if (e < L) {
            const uint32_t lp = my[(kk[k] >> shift) & (D - 1)] + rk[k];
            skey[lp] = kk[k];
            sval[lp] = vv[k];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nvalid; i += kSortThreads) {
        const uint32_t key = skey[i];
        const uint32_t pos = (uint32_t)i + delta[(key >> shift) & (D - 1)];
        CD_CHECK(pos >= (uint64_t)g.seg_start(sg) && pos < (uint64_t)(g.seg_start(sg) + g.seg_size(sg)));
        kout[pos] = key;
        vout[pos] = sval[i];
    }
}

// off[k] = first sorted position with GLOBAL key >= k, for k in [0, kmax]; off[kmax] = L.  The
// sorted keys are segment-local: position p of segment s carries global key kbase(s) + key[p], with
// kbase(s) = s KA (s < nA) or nA KA + (s - nA) KB, and the global keys ascend over all positions.
// Each thread fills the gaps before kOffRun consecutive positions (one segment division per run, the
// run's keys loaded together); the writes of different threads are disjoint (no atomics).
constexpr int kOffRun = 8;
__global__ void __launch_bounds__(256) offsets_kernel(const uint32_t* __restrict__ keys, SortSegs g, int64_t KA,
                                                      int64_t KB, int64_t kmax, uint32_t* __restrict__ off) {
    const int L = (int)g.seg_start(g.nsegs());   // < 2^31 (cd_backward's size limit)
    const int LA = (int)((int64_t)g.nA * g.szA);
    const int szA = (int)g.szA, szB = (int)max(g.szB, (int64_t)1);
    const int nruns = L / kOffRun + 1;            // positions [0, L] inclusive
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nruns; r += gridDim.x * blockDim.x) {
        const int p0 = r * kOffRun;
        // segment of position p0 - 1 (the run's left neighbour) and where it ends
        const int q = max(p0 - 1, 0);
        int s = q < LA ? q / szA : g.nA + (q - LA) / szB;
        int send = (int)g.seg_start(s + 1);
        int64_t kb = s < g.nA ? (int64_t)s * KA : (int64_t)g.nA * KA + (int64_t)(s - g.nA) * KB;
        uint32_t kk[kOffRun + 1];
#pragma unroll
        for (int u = 0; u <= kOffRun; ++u) kk[u] = (p0 - 1 + u >= 0 && p0 - 1 + u < L) ? keys[p0 - 1 + u] : 0u;
        int64_t prev = p0 == 0 ? -1 : kb + kk[0];   // global key at p0 - 1
#pragma unroll
        for (int u = 0; u < kOffRun; ++u) {
            const int p = p0 + u;
            if (p > L) break;
            int64_t hi;
            if (p == L) {
                hi = kmax;
            } else {
                while (p >= send) {   // next segment
                    ++s;
                    send = (int)g.seg_start(s + 1);
                    kb = s < g.nA ? (int64_t)s * KA : (int64_t)g.nA * KA + (int64_t)(s - g.nA) * KB;
                }
                hi = kb + kk[u + 1];
            }
            CD_CHECK(prev + 1 <= hi + 1 && hi <= kmax);
            for (int64_t k = prev + 1; k <= hi; ++k) off[k] = (uint32_t)p;
            prev = hi;
        }
    }
}

struct GradArgs {
    const float* x;
    const float* y;
    int B, N, M, q0, q1, r0, r1;
    const int32_t* idx_xy;
    const int32_t* idx_yx;
    const float* g;
    const float* h;
    float g_scalar, h_scalar;
    const float* upstream;   // optional device scalar u: the fills become RN(u * g_scalar), RN(u * h_scalar)
    const uint32_t* vals;
    const uint32_t* off;
    float* grad_x;
    float* grad_y;
};

// acc += (2 w) * (p - s), fp64, explicit roundings in the oracle's order (no FMA contraction); p is
// the output point, promoted to fp64 once (exactly) by the caller and kept in registers.
__device__ __forceinline__ void acc_term(double acc[3], const double p[3], const float* s, double w) {
    const double w2 = __dmul_rn(2.0, w);
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(w2, __dsub_rn(p[c], (double)s[c])));
}
__device__ __forceinline__ void load_point64(const float* p, double out[3]) {
    out[0] = (double)p[0];
    out[1] = (double)p[1];
    out[2] = (double)p[2];
}

// Segment-local sort (small clouds: max(N, M) <= kSegMax).  The edges of one (direction, batch
// element) segment have keys in one range of T = M (xy) or N (yx) consecutive keys and land in one
// contiguous range of the sorted order, so each segment sorts on its own: one CTA per segment, a
// stable LSD radix sort entirely in shared memory (digits of <= 7 bits; warp w owns a contiguous
// range of the segment and places it in order with warp ballot multisplit ranks; the per-warp digit
// counts of a pass are integer shared-memory adds made while loading / while placing the previous
// pass), then the sorted sources and the segment's key offsets (gap fill) go to global memory.
// Replaces keys_hist + the global passes + offsets_kernel: 2 launches per backward, not 3 passes + 2.
#ifndef CD_SEG_COUNTING
#define CD_SEG_COUNTING 1   // counting sort for part key ranges that fit the counter words (see below)
#endif
constexpr int kRunMax = 32;   // longest key run the counting mode's insertion sort handles


// Exclusive scan of one value per thread over the kSegThreads threads of the CTA (warp shuffles +
// the warp totals in `wtot[kSegWarps]`); contains the barriers it needs.
__device__ __forceinline__ uint32_t seg_block_exclusive_scan(uint32_t v, uint32_t* wtot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    __syncthreads();   // wtot may still be read by an earlier phase
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += wtot[w];
    return before + incl - v;
}

__global__ void __launch_bounds__(kSegThreads) seg_sort_grad_kernel(GradArgs ga, int nmax, int lparts) {
    pdl_wait();
    const int32_t* __restrict__ idx_xy = ga.idx_xy;
    const int32_t* __restrict__ idx_yx = ga.idx_yx;
    const int B = ga.B, N = ga.N, M = ga.M;
    extern __shared__ __align__(16) uint32_t smem_seg[];
    uint32_t* wcur = smem_seg;                   // [kSegWarps][D] this pass's per-warp digit counts
    uint32_t* wnext = wcur + kSegWarps * kSegD;  // next pass's, counted while placing
    uint16_t* kA = reinterpret_cast<uint16_t*>(wnext + kSegWarps * kSegD);   // keys
    uint16_t* kB = kA + nmax;
    uint16_t* vA = kB + nmax;                    // values: the source's index in the segment
    uint16_t* vB = vA + nmax;
    __shared__ uint32_t dstart[kSegD];
    __shared__ uint32_t wsum[2][kSegWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = blockIdx.x >> lparts, part = blockIdx.x & ((1 << lparts) - 1);
    const int dir = seg / B, b = seg - dir * B;
    const int nseg = dir == 0 ? N : M;       // edges (sources) of the segment
    const int T = dir == 0 ? M : N;          // keys (targets) of the segment
    const int32_t* idx = dir == 0 ? idx_xy + (int64_t)b * N : idx_yx + (int64_t)b * M;
    int nb = 1;
    while ((1 << nb) < T) ++nb;
    // part h of the segment's 2^lparts CTAs owns the keys whose top lparts bits are h: [K0, K1)
    const int lp = min(lparts, nb);
    const int kb_low = nb - lp;              // key bits sorted on chip
    const int K0 = min(part << kb_low, T), K1 = min((part + 1) << kb_low, T);
    // phase A: per-warp counts of this part's edges and of the edges of lower parts (the part's
    // global base); warp w scans a contiguous range of the segment in order
    const int lspan_l = max(5, 31 - __clz(max((nseg + kSegWarps - 1) / kSegWarps, 1) - 1) + 1);
    const int spanl = 1 << lspan_l;
    const int wend = min((warp + 1) * spanl, nseg);
    {
        uint32_t mine = 0, lower = 0;
        for (int e0 = warp * spanl; e0 < wend; e0 += 8 * 32) {   // 8 index loads in flight per lane
            int k[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * 32 + lane;
                k[u] = e < wend ? min(max(__ldg(idx + e), 0), T - 1) : -1;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                mine += __popc(__ballot_sync(0xffffffffu, k[u] >= K0 && k[u] < K1));
                lower += __popc(__ballot_sync(0xffffffffu, k[u] >= 0 && k[u] < K0));
            }
        }
        if (lane == 0) {
            wsum[0][warp] = mine;
            wsum[1][warp] = lower;
        }
    }
    for (int i = threadIdx.x; i < 2 * kSegWarps * kSegD; i += kSegThreads) wcur[i] = 0;
    __syncthreads();
    uint32_t wbase = 0, n_u = 0, base_u = 0;
    for (int w = 0; w < kSegWarps; ++w) {
        const uint32_t c = wsum[0][w];
        wbase += w < warp ? c : 0u;
        n_u += c;
        base_u += wsum[1][w];
    }
    const int n = (int)n_u;                  // edges of this part
    CD_CHECK(n <= nmax && (int64_t)base_u + n <= nseg);
    const int passes = kb_low > 0 ? (kb_low + kSegDigitBits - 1) / kSegDigitBits : 0;
    const int db = passes > 0 ? (kb_low + passes - 1) / passes : 1;
    const int D = 1 << db;
    int lspan = 5;   // rounds per warp R = span / 32, a power of two: warp w owns [w*span, (w+1)*span)
    while (kSegWarps << lspan < n) ++lspan;
    const int R = 1 << (lspan - 5);
    // counting mode (the part's key range fits the 2 x 32 x 128 counter words): a counting sort
    // instead of the LSD passes — per-key counts, an exclusive scan, placement by integer shared-memory
    // atomics (unordered inside a key) and each key's run then sorted by source index, which restores
    // the stable order exactly; a part with a run longer than kRunMax falls back to the LSD passes
    const bool counting = CD_SEG_COUNTING && K1 - K0 <= 2 * kSegWarps * kSegD;
    // phase B: ordered compaction of the part's edges + the first pass's per-warp digit counts
    // (integer shared-memory adds: order-free)
    {
        const uint32_t lt_mask = (1u << lane) - 1u;
        uint32_t run = wbase;
        for (int e0 = warp * spanl; e0 < wend; e0 += 8 * 32) {
            int k[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * 32 + lane;
                k[u] = e < wend ? min(max(__ldg(idx + e), 0), T - 1) : -1;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const bool in = k[u] >= K0 && k[u] < K1;
                const uint32_t m = __ballot_sync(0xffffffffu, in);
                if (in) {
                    const uint32_t pos = run + __popc(m & lt_mask);
                    CD_CHECK(pos < (uint32_t)n && (pos >> lspan) < (uint32_t)kSegWarps);
                    kA[pos] = (uint16_t)k[u];
                    vA[pos] = (uint16_t)(e0 + u * 32 + lane);
                    if (counting)
                        atomicAdd(&wcur[k[u] - K0], 1u);   // per-key counts (integer adds: order-free)
                    else if (passes > 0)
                        atomicAdd(&wcur[(pos >> lspan) * D + (k[u] & (D - 1))], 1u);
                }
                run += __popc(m);
            }
        }
    }
    bool counted = false;   // the counting sort produced the grouped sources (in vB, runs from wcur)
    if (counting) {
        __syncthreads();
        const int KK = K1 - K0;
        uint32_t* cnt = wcur;   // [KK]: counts, then exclusive offsets, then (after placement) run ends
        const int per = (KK + kSegThreads - 1) / kSegThreads;
        const int c0 = min(threadIdx.x * per, KK), c1 = min(c0 + per, KK);
        uint32_t loc = 0;
        bool longrun = false;
        for (int i = c0; i < c1; ++i) {
            loc += cnt[i];
            longrun |= cnt[i] > (uint32_t)kRunMax;
        }
        const uint32_t excl = seg_block_exclusive_scan(loc, &wsum[0][0]);
        if (!__syncthreads_or(longrun)) {
            uint32_t run = excl;
            for (int i = c0; i < c1; ++i) {
                const uint32_t c = cnt[i];
                cnt[i] = run;
                run += c;
            }
            __syncthreads();
            for (int e = threadIdx.x; e < n; e += kSegThreads) {
                const uint32_t pos = atomicAdd(&cnt[kA[e] - K0], 1u);   // cnt[k] ends as the end of k's run
                CD_CHECK(pos < (uint32_t)n);
                vB[pos] = vA[e];
            }
            __syncthreads();
            for (int kk = threadIdx.x; kk < KK; kk += kSegThreads) {   // runs of <= kRunMax: insertion sort
                const int r0 = kk == 0 ? 0 : (int)cnt[kk - 1], r1 = (int)cnt[kk];
                for (int i = r0 + 1; i < r1; ++i) {
                    const uint16_t v = vB[i];
                    int j = i - 1;
                    while (j >= r0 && vB[j] > v) {
                        vB[j + 1] = vB[j];
                        --j;
                    }
                    vB[j + 1] = v;
                }
            }
            __syncthreads();
            counted = true;
        } else {
            // fallback: the first LSD pass's per-warp digit counts from the compacted keys
            for (int i = threadIdx.x; i < 2 * kSegWarps * kSegD; i += kSegThreads) wcur[i] = 0;
            __syncthreads();
            if (passes > 0)
                for (int e = threadIdx.x; e < n; e += kSegThreads)
                    atomicAdd(&wcur[(e >> lspan) * D + (kA[e] & (D - 1))], 1u);
        }
    }
    uint16_t* offs = kB;
    if (!counted) {
        seg_lsd_passes(kA, vA, kB, vB, wcur, wnext, dstart, n, passes, db, lspan, R);
        __syncthreads();
        // key offsets of this part in shared memory (the free key buffer): offs[k - K0] = first sorted
        // position with key >= k for k in [K0, K1) (gap fill, disjoint writes); key K1 - 1's run ends at n
        offs = kB;
        for (int p = threadIdx.x; p <= n; p += kSegThreads) {
            const int lo = p == 0 ? K0 : (int)kA[p - 1] + 1;
            const int hi = min(p == n ? K1 : (int)kA[p], K1 - 1);
            CD_CHECK(lo >= K0 && hi < K1);
            for (int k = lo; k <= hi; ++k) offs[k - K0] = (uint16_t)p;
        }
        __syncthreads();
    }
    const uint16_t* srt = counted ? vB : vA;           // sources grouped by key, ascending inside a key
    const uint32_t* cend = wcur;                       // counting: end of key k's run at cend[k - K0]
    // the gradients of this part's targets, as grad_kernel computes them: own term 2 w_t (p - partner)
    // first, then the sources in ascending index (the stable sort's order), fp64 with explicit .rn ops
    float gs = ga.g_scalar, hs = ga.h_scalar;
    if (ga.upstream) {
        const float u = *ga.upstream;
        gs = __fmul_rn(u, gs);
        hs = __fmul_rn(u, hs);
    }
    const int S = dir == 0 ? N : M;                              // sources (and partners) per batch
    const float* tgt = dir == 0 ? ga.y + (int64_t)b * M * 3 : ga.x + (int64_t)b * N * 3;
    const float* src = dir == 0 ? ga.x + (int64_t)b * N * 3 : ga.y + (int64_t)b * M * 3;
    const int32_t* pidx = dir == 0 ? idx_yx + (int64_t)b * M : idx_xy + (int64_t)b * N;
    const float* wt = dir == 0 ? (ga.h ? ga.h + (int64_t)b * M : nullptr) : (ga.g ? ga.g + (int64_t)b * N : nullptr);
    const float* wsrc = dir == 0 ? (ga.g ? ga.g + (int64_t)b * N : nullptr) : (ga.h ? ga.h + (int64_t)b * M : nullptr);
    const float wt_s = dir == 0 ? hs : gs, wsrc_s = dir == 0 ? gs : hs;
    const int t0 = dir == 0 ? ga.r0 : ga.q0, t1 = dir == 0 ? ga.r1 : ga.q1;
    float* out = dir == 0 ? ga.grad_y + (int64_t)b * (ga.r1 - ga.r0) * 3 : ga.grad_x + (int64_t)b * (ga.q1 - ga.q0) * 3;
    const int tlo = max(K0, t0), thi = min(K1, t1);
    // the part's partner rows staged in the 16-bit buffer the sort left free (sources < kSegMax <
    // 2^16), so each target's loads — its point, its partner and its first source — are ONE round
    // trip: the three addresses come from shared memory
    uint16_t* spart = counted ? vA : vB;
    for (int t = tlo + threadIdx.x; t < thi; t += kSegThreads)
        spart[t - K0] = (uint16_t)min(max(__ldg(pidx + t), 0), S - 1);
    __syncthreads();
    for (int t = tlo + threadIdx.x; t < thi; t += kSegThreads) {
        int e0, e1;
        if (counted) {
            e0 = t == K0 ? 0 : (int)cend[t - K0 - 1];
            e1 = (int)cend[t - K0];
        } else {
            e0 = offs[t - K0];
            e1 = t + 1 < K1 ? (int)offs[t + 1 - K0] : n;
        }
        CD_CHECK(e0 <= e1 && e1 <= n);
        const float* pp = tgt + (int64_t)t * 3;
        const float* ps = src + (int64_t)spart[t - K0] * 3;
        const int s0 = e0 < e1 ? (int)srt[e0] : 0;   // an empty run reads row 0 (valid) and ignores it
        const float* pf = src + (int64_t)s0 * 3;
        const float tx = pp[0], ty = pp[1], tz = pp[2];
        const float px = ps[0], py = ps[1], pz = ps[2];
        const float fx = pf[0], fy = pf[1], fz = pf[2];
        const double wtt = wt ? (double)wt[t] : (double)wt_s;
        const double wf = wsrc ? (double)wsrc[s0] : (double)wsrc_s;
        const double pt[3] = {(double)tx, (double)ty, (double)tz};
        double acc[3];
        {
            const double w2 = __dmul_rn(2.0, wtt);
            acc[0] = __dmul_rn(w2, __dsub_rn(pt[0], (double)px));
            acc[1] = __dmul_rn(w2, __dsub_rn(pt[1], (double)py));
            acc[2] = __dmul_rn(w2, __dsub_rn(pt[2], (double)pz));
        }
        if (e0 < e1) {
            const double w2 = __dmul_rn(2.0, wf);
            acc[0] = __dadd_rn(acc[0], __dmul_rn(w2, __dsub_rn(pt[0], (double)fx)));
            acc[1] = __dadd_rn(acc[1], __dmul_rn(w2, __dsub_rn(pt[1], (double)fy)));
            acc[2] = __dadd_rn(acc[2], __dmul_rn(w2, __dsub_rn(pt[2], (double)fz)));
        }
        for (int e = e0 + 1; e < e1; ++e) {
            const int sidx = srt[e];
            acc_term(acc, pt, src + (int64_t)sidx * 3, wsrc ? (double)wsrc[sidx] : (double)wsrc_s);
        }
        float* o = out + (int64_t)(t - t0) * 3;
        o[0] = (float)acc[0];
        o[1] = (float)acc[1];
        o[2] = (float)acc[2];
    }
}

#ifndef CD_SEG_MAXPARTS
#define CD_SEG_MAXPARTS 3   // log2 of the most CTAs per segment
#endif
#ifndef CD_GRAD_MINB
#define CD_GRAD_MINB 1   // min resident CTAs per SM requested from ptxas (register cap)
#endif
#ifndef CD_GRAD_CTAS_PER_SM
#define CD_GRAD_CTAS_PER_SM 0   // 0: the occupancy (one resident wave)
#endif
__global__ void __launch_bounds__(256, CD_GRAD_MINB) grad_kernel(GradArgs a) {
    pdl_wait();
    if (a.upstream) {
        const float u = *a.upstream;
        a.g_scalar = __fmul_rn(u, a.g_scalar);
        a.h_scalar = __fmul_rn(u, a.h_scalar);
    }
    const int sq = a.q1 - a.q0, sr = a.r1 - a.r0;
    const int per_b = sq + sr;
    const int64_t total = (int64_t)a.B * per_b;
    // batch-major order: batch b's X outputs, then its Y outputs, so the one resident wave works on
    // one batch element's two clouds at a time and the second direction's reads (the clouds the
    // first direction gathered or streamed) hit L2 (c5: DRAM reads ~300 -> ~200 MB)
    // total = B (|q| + |r|) < 2^31 (cd_backward's size limit): 32-bit index arithmetic
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < (int)total; t += gridDim.x * blockDim.x) {
        double acc[3] = {0.0, 0.0, 0.0};
        const int64_t b = t / per_b;
        const int u = t - (int)b * per_b;
        if (u < sq) {
            const int i = a.q0 + u;
            const int64_t xi = b * a.N + i;
            double p[3];
            load_point64(a.x + xi * 3, p);
            const int part = min(max(a.idx_xy[xi], 0), a.M - 1);
            const double gi = a.g ? (double)a.g[xi] : (double)a.g_scalar;
            // own term, then: every term has the form 2 w (p - s) with p = this point
            {
                double own[3] = {0.0, 0.0, 0.0};
                const float* s = a.y + (b * a.M + part) * 3;
                const double w2 = __dmul_rn(2.0, gi);
#pragma unroll
                for (int c = 0; c < 3; ++c) own[c] = __dmul_rn(w2, __dsub_rn(p[c], (double)s[c]));
                acc[0] = own[0];
                acc[1] = own[1];
                acc[2] = own[2];
            }
            const int64_t key = (int64_t)a.B * a.M + b * a.N + i;
            const uint32_t e0 = a.off[key], e1 = a.off[key + 1];
            CD_CHECK(e0 <= e1 && e1 <= (uint32_t)((int64_t)a.B * (a.N + a.M)));
            for (uint32_t e = e0; e < e1; ++e) {
                const uint32_t src = a.vals[e];  // y row b*M + j
                CD_CHECK(src < (uint32_t)((int64_t)a.B * a.M));
                const double hj = a.h ? (double)a.h[src] : (double)a.h_scalar;
                acc_term(acc, p, a.y + (int64_t)src * 3, hj);
            }
            float* o = a.grad_x + (b * sq + (i - a.q0)) * 3;
            o[0] = (float)acc[0];
            o[1] = (float)acc[1];
            o[2] = (float)acc[2];
        } else {
            const int j = a.r0 + (u - sq);
            const int64_t yj = b * a.M + j;
            double p[3];
            load_point64(a.y + yj * 3, p);
            const int part = min(max(a.idx_yx[yj], 0), a.N - 1);
            const double hj = a.h ? (double)a.h[yj] : (double)a.h_scalar;
            {
                const float* s = a.x + (b * a.N + part) * 3;
                const double w2 = __dmul_rn(2.0, hj);
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[c] = __dmul_rn(w2, __dsub_rn(p[c], (double)s[c]));
            }
            const int64_t key = b * a.M + j;
            const uint32_t e0 = a.off[key], e1 = a.off[key + 1];
            CD_CHECK(e0 <= e1 && e1 <= (uint32_t)((int64_t)a.B * (a.N + a.M)));
            for (uint32_t e = e0; e < e1; ++e) {
                const uint32_t src = a.vals[e];  // x row b*N + i
                CD_CHECK(src < (uint32_t)((int64_t)a.B * a.N));
                const double gi = a.g ? (double)a.g[src] : (double)a.g_scalar;
                acc_term(acc, p, a.x + (int64_t)src * 3, gi);
            }
            float* o = a.grad_y + (b * sr + (j - a.r0)) * 3;
            o[0] = (float)acc[0];
            o[1] = (float)acc[1];
            o[2] = (float)acc[2];
        }
    }
}

// ------------------------------------------------------------------------------------------------
static int sm_count() { return current_sm_count(); }

struct RadixPlan {
    int npasses, digit_bits, items;
    SortSegs g;
};

// Digits per pass: the fewest passes of <= 11-bit digits, or (narrow = true, the backward) the pass
// count minimising passes x relative pass cost, measured per digit width on the c5 / c4 backward
// (one 8.4M-element pass: 8-bit digits ~98 us, 10-bit ~170 us, the ballot multisplit and the
// per-warp counter tables growing with the digit): <= 8 bits 1.0, 9 bits 1.3, 10-11 bits 1.75.
static RadixPlan radix_plan(const SegSpec& sp, int nbits, bool narrow = false) {
    RadixPlan r;
    nbits = std::max(nbits, 1);
    r.npasses = (nbits + kMaxDigitBits - 1) / kMaxDigitBits;
    if (narrow) {
        auto cost = [](int db) { return db <= 8 ? 1.0 : db == 9 ? 1.3 : 1.75; };
        double best = 1e30;
        for (int np = r.npasses; np <= r.npasses + 2; ++np) {
            const int db = (nbits + np - 1) / np;
            const double c = np * cost(db);
            if (c < best - 1e-9) {
                best = c;
                r.npasses = np;
            }
        }
    }
    r.digit_bits = (nbits + r.npasses - 1) / r.npasses;
    r.items = sort_items(r.digit_bits);
    r.g = make_segs(sp, kSortThreads * r.items);
    return r;
}

static SegSpec one_segment(int64_t L) { return SegSpec{1, L, 0, 0}; }

size_t radix_sort_counts_words(const SegSpec& sp, int nbits, bool narrow) {
    const RadixPlan r = radix_plan(sp, nbits, narrow);
    return (size_t)(1 << r.digit_bits) * r.g.ntiles();
}
size_t radix_sort_totals_words(const SegSpec& sp, int nbits, bool narrow) {
    const RadixPlan r = radix_plan(sp, nbits, narrow);
    return (size_t)(1 << r.digit_bits) * r.g.nsegs();
}
size_t radix_sort_counts_words(int64_t L, int nbits) { return radix_sort_counts_words(one_segment(L), nbits, false); }

// Stable LSD radix sort of (key, value) u32 pairs by the low `nbits` key bits, every segment of `sp`
// on its own.  keys[0]/vals[0] hold the input; returns the index (0 or 1) of the buffers holding the
// sorted output.  counts: radix_sort_counts_words words; totals: radix_sort_totals_words words.
int radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], const SegSpec& sp, int nbits, uint32_t* counts,
                     uint32_t* totals, cudaStream_t st, bool first_hist_done, bool narrow) {
    const RadixPlan r = radix_plan(sp, nbits, narrow);
    const int D = 1 << r.digit_bits;
    const int ntiles = r.g.ntiles();
    const size_t scatter_smem = ((size_t)(kSortWarps + 2) * D + 2 * kSortThreads * r.items) * 4;
    ensure_smem_attr((const void*)radix_scatter_kernel<kSortItems>,
                     ((kSortWarps + 2) * (1 << kMaxDigitBits) + 2 * kSortThreads * kSortItems) * 4);
    ensure_smem_attr((const void*)radix_scatter_kernel<kSortItemsWide>,
                     ((kSortWarps + 2) * (1 << kMaxDigitBits) + 2 * kSortThreads * kSortItemsWide) * 4);
    int cur = 0;
    if (ntiles == 0) return cur;
    for (int pass = 0; pass < r.npasses; ++pass) {
        const int shift = pass * r.digit_bits;
        if (!(pass == 0 && first_hist_done)) {
            if (r.items == kSortItemsWide)
                radix_hist_kernel<kSortItemsWide><<<ntiles, kSortThreads, (size_t)D * 4, st>>>(keys[cur], r.g, shift, D,
                                                                                              counts);
            else
                radix_hist_kernel<kSortItems><<<ntiles, kSortThreads, (size_t)D * 4, st>>>(keys[cur], r.g, shift, D,
                                                                                          counts);
        }
        radix_rowscan_kernel<<<(unsigned)(((int64_t)r.g.nsegs() * D + kSortWarps - 1) / kSortWarps), kSortThreads, 0,
                               st>>>(counts, r.g, D, totals);
        if (r.items == kSortItemsWide)
            radix_scatter_kernel<kSortItemsWide><<<ntiles, kSortThreads, scatter_smem, st>>>(
                keys[cur], vals[cur], r.g, shift, D, counts, totals, keys[1 - cur], vals[1 - cur]);
        else
            radix_scatter_kernel<kSortItems><<<ntiles, kSortThreads, scatter_smem, st>>>(
                keys[cur], vals[cur], r.g, shift, D, counts, totals, keys[1 - cur], vals[1 - cur]);
        cur = 1 - cur;
    }
    return cur;
}

int radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t L, int nbits, uint32_t* counts, uint32_t* totals,
                     cudaStream_t st, bool first_hist_done) {
    return radix_sort_pairs(keys, vals, one_segment(L), nbits, counts, totals, st, first_hist_done, false);
}

int radix_sort_launches(int64_t L, int nbits) { return 3 * radix_plan(one_segment(L), nbits).npasses; }
int radix_sort_launches(const SegSpec& sp, int nbits, bool narrow) { return 3 * radix_plan(sp, nbits, narrow).npasses; }

int radix_digit_bits(int64_t L, int nbits) { return radix_plan(one_segment(L), nbits).digit_bits; }

#ifndef CD_SEGSORT
#define CD_SEGSORT 1
#endif

void plan_backward(BwdPlan& p, int B, int N, int M, int q0, int q1, int r0, int r1) {
    p.B = B;
    p.N = N;
    p.M = M;
    p.q0 = q0;
    p.q1 = q1;
    p.r0 = r0;
    p.r1 = r1;
    p.L = (int64_t)B * (N + M);
    p.kmax = p.L;  // B*M keys for the xy edges + B*N keys for the yx edges
    // 2B segments sorted on their own: B of N xy edges keyed in [0, M), B of M yx edges keyed in [0, N)
    p.segs = SegSpec{B, N, B, M};
    int bits = 0;
    while (bits < 31 && (1 << bits) < std::max(N, M)) ++bits;
    p.nbits = std::max(bits, 1);
    const RadixPlan r = radix_plan(p.segs, p.nbits, true);
    p.npasses = r.npasses;
    p.digit_bits = r.digit_bits;
    p.ntiles = r.g.ntiles();
    p.segsort = CD_SEGSORT != 0 && std::max(N, M) <= kSegMax;
    size_t off = 0;
    for (int i = 0; i < 2; ++i) {
        p.off_keys[i] = off;
        off = align_up(off + (size_t)p.L * 4, 256);
        p.off_vals[i] = off;
        off = align_up(off + (size_t)p.L * 4, 256);
    }
    p.off_counts = off;
    off = align_up(off + radix_sort_counts_words(p.segs, p.nbits, true) * 4, 256);
    p.off_totals = off;
    off = align_up(off + radix_sort_totals_words(p.segs, p.nbits, true) * 4, 256);
    p.off_offsets = off;
    off = align_up(off + (size_t)(p.kmax + 1) * 4, 256);
    p.bytes = off;
}

int backward_launches(const BwdPlan& p) {
    return p.segsort ? 1 : 3 * p.npasses + 2;   // keys fused with the pass-0 histogram
}

cudaError_t launch_backward(const BwdPlan& p, const float* x, const float* y, const int32_t* idx_xy,
                            const int32_t* idx_yx, const float* g, const float* h, float g_scalar, float h_scalar,
                            const float* upstream, float* grad_x, float* grad_y, void* ws, cudaStream_t st) {
    char* w = static_cast<char*>(ws);
    uint32_t* keys[2] = {reinterpret_cast<uint32_t*>(w + p.off_keys[0]), reinterpret_cast<uint32_t*>(w + p.off_keys[1])};
    uint32_t* vals[2] = {reinterpret_cast<uint32_t*>(w + p.off_vals[0]), reinterpret_cast<uint32_t*>(w + p.off_vals[1])};
    uint32_t* counts = reinterpret_cast<uint32_t*>(w + p.off_counts);
    uint32_t* totals = reinterpret_cast<uint32_t*>(w + p.off_totals);
    uint32_t* off = reinterpret_cast<uint32_t*>(w + p.off_offsets);
    GradArgs a;
    a.x = x;
    a.y = y;
    a.B = p.B;
    a.N = p.N;
    a.M = p.M;
    a.q0 = p.q0;
    a.q1 = p.q1;
    a.r0 = p.r0;
    a.r1 = p.r1;
    a.idx_xy = idx_xy;
    a.idx_yx = idx_yx;
    a.g = g;
    a.h = h;
    a.g_scalar = g_scalar;
    a.h_scalar = h_scalar;
    a.upstream = upstream;
    a.grad_x = grad_x;
    a.grad_y = grad_y;
    if (p.segsort) {
        // one launch: each CTA sorts its (direction, batch) segment part on chip and writes the
        // gradients of that part's targets
        const int nmax = std::max(p.N, p.M);
        const size_t smem = seg_sort_smem(nmax);
        ensure_smem_attr((const void*)seg_sort_grad_kernel, (int)seg_sort_smem(kSegMax));
        // 2^lparts CTAs per segment (split by the keys' top bits) while the segments alone leave SMs idle
        int lparts = 0;
        while (lparts < CD_SEG_MAXPARTS && (int64_t)2 * p.B << (lparts + 1) <= sm_count()) ++lparts;
        a.vals = nullptr;
        a.off = nullptr;
        launch_pdl(seg_sort_grad_kernel, dim3((unsigned)((int64_t)2 * p.B << lparts)), dim3(kSegThreads), smem, st, a,
                   nmax, lparts);
        return cudaGetLastError();
    }
    const RadixPlan r = radix_plan(p.segs, p.nbits, true);
    const int D = 1 << r.digit_bits;
    if (r.items == kSortItemsWide)
        keys_hist_kernel<kSortItemsWide><<<p.ntiles, kSortThreads, (size_t)D * 4, st>>>(
            idx_xy, idx_yx, p.B, p.N, p.M, D, r.g, keys[0], vals[0], counts);
    else
        keys_hist_kernel<kSortItems><<<p.ntiles, kSortThreads, (size_t)D * 4, st>>>(
            idx_xy, idx_yx, p.B, p.N, p.M, D, r.g, keys[0], vals[0], counts);
    const int cur = radix_sort_pairs(keys, vals, p.segs, p.nbits, counts, totals, st, /*first_hist_done=*/true,
                                     /*narrow=*/true);
    const int grid_o = (int)std::min<int64_t>((p.L / kOffRun + 1 + 255) / 256, (int64_t)sm_count() * 16);
    offsets_kernel<<<grid_o, 256, 0, st>>>(keys[cur], r.g, p.M, p.N, p.kmax, off);
    a.vals = vals[cur];
    a.off = off;
    const int64_t total = (int64_t)p.B * ((p.q1 - p.q0) + (p.r1 - p.r0));
    if (total > 0) {
        // exactly one wave of resident CTAs striding over the points (measured: c5 backward 0.546 ->
        // 0.487 ms against 32 CTAs per SM; a second, partial wave costs more than it hides)
        static std::atomic<int> occ_table[kMaxDevices];
        const int occ = occupancy_of(occ_table, grad_kernel, 256, 0, 4);
        const int grid_g = (int)std::min<int64_t>((total + 255) / 256,
                                                  (int64_t)sm_count() * (CD_GRAD_CTAS_PER_SM > 0 ? CD_GRAD_CTAS_PER_SM : occ));
        launch_pdl(grad_kernel, dim3(grid_g), dim3(256), 0, st, a);
    }
    return cudaGetLastError();
}

}  // namespace cdk
