// seg_sort.cuh — on-chip stable LSD radix sort of one segment (<= kSegMax 16-bit keys with 16-bit
// values) by one CTA of kSegThreads threads, shared by the backward's segment sort (nn_backward.cu)
// and the pruned path's Hilbert sort (nn_pruned.cu).  Warp w owns a contiguous range of the segment
// (R rounds of 32); ranks come from a warp ballot multisplit (VOTE at ALU rate) and per-warp digit
// counters; the next pass's per-warp counts are integer shared-memory adds made while placing.
#pragma once
#include "cd_device.cuh"

namespace cdk {

#ifndef CD_SEG_THREADS
#define CD_SEG_THREADS 1024
#endif
constexpr int kSegThreads = CD_SEG_THREADS;
constexpr int kSegWarps = kSegThreads / 32;
constexpr int kSegMax = 24576;   // 8 B per edge + 32 KB of counters <= 227 KB of shared memory
constexpr int kSegDigitBits = 7;
constexpr int kSegD = 1 << kSegDigitBits;

inline size_t seg_sort_smem(int nmax) { return (size_t)nmax * 8 + 2 * (size_t)kSegWarps * kSegD * 4 + 1024; }

// One placement sweep of seg_sort_kernel with DB-bit digits (compile-time: unrolled ballots).
template <int DB>
__device__ __forceinline__ void seg_place(const uint16_t* kA, const uint16_t* vA, uint16_t* kB, uint16_t* vB,
                                          uint32_t* wcur, uint32_t* wnext, int n, int R, int lspan, int shift,
                                          bool last) {
    constexpr uint32_t D = 1u << DB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t* my = wcur + warp * D;
    for (int t = 0; t < R; ++t) {
        const int e0 = (warp * R + t) * 32;
        if (e0 >= n) break;   // warp-uniform
        const int e = e0 + lane;
        const bool valid = e < n;
        const uint16_t key = valid ? kA[e] : (uint16_t)0;
        const uint32_t digit = ((uint32_t)key >> shift) & (D - 1);
        uint32_t peers = __ballot_sync(0xffffffffu, valid);
        if (!valid) peers = ~peers;
#pragma unroll
        for (int bt = 0; bt < DB; ++bt) {
            const bool bit = (digit >> bt) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
        const uint32_t before = valid ? my[digit] : 0u;
        if (valid) {
            const uint32_t pos = before + __popc(peers & lt_mask);
            CD_CHECK(pos < (uint32_t)n);
            kB[pos] = key;
            vB[pos] = vA[e];
            if (!last) atomicAdd(&wnext[(pos >> lspan) * D + (((uint32_t)key >> (shift + DB)) & (D - 1))], 1u);
        }
        __syncwarp();
        if (valid && (peers & lt_mask) == 0u) my[digit] = before + __popc(peers);
        __syncwarp();
    }
}

// The passes of the sort: on entry wcur holds the first pass's per-warp digit counts (zeroed wnext
// alongside); kA/vA hold the keys/values; on exit kA/vA point at the sorted arrays.
__device__ __forceinline__ void seg_lsd_passes(uint16_t*& kA, uint16_t*& vA, uint16_t*& kB, uint16_t*& vB,
                                               uint32_t*& wcur, uint32_t*& wnext, uint32_t* dstart, int n,
                                               int passes, int db, int lspan, int R) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int D = 1 << db;
    for (int pass = 0; pass < passes; ++pass) {
        const int shift = pass * db;
        const bool last = pass + 1 == passes;
        __syncthreads();
        // digit starts, then per-warp starts inside each digit run
        if (threadIdx.x < D) {
            uint32_t tot = 0;
            for (int w = 0; w < kSegWarps; ++w) tot += wcur[w * D + threadIdx.x];
            dstart[threadIdx.x] = tot;
        }
        __syncthreads();
        if (warp == 0) {
            uint32_t c[kSegD / 32], loc = 0;
#pragma unroll
            for (int r = 0; r < kSegD / 32; ++r) {
                const int d = lane * (kSegD / 32) + r;
                c[r] = d < D ? dstart[d] : 0u;
                loc += c[r];
            }
            uint32_t incl = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            uint32_t run = incl - loc;
#pragma unroll
            for (int r = 0; r < kSegD / 32; ++r) {
                const int d = lane * (kSegD / 32) + r;
                if (d < D) dstart[d] = run;
                run += c[r];
            }
        }
        __syncthreads();
        if (threadIdx.x < D) {
            uint32_t run = dstart[threadIdx.x];
            for (int w = 0; w < kSegWarps; ++w) {
                const uint32_t c = wcur[w * D + threadIdx.x];
                wcur[w * D + threadIdx.x] = run;
                run += c;
            }
        }
        for (int i = threadIdx.x; i < kSegWarps * kSegD; i += kSegThreads) wnext[i] = 0;
        __syncthreads();
        // stable placement: each warp walks its range in order; ranks from a ballot multisplit
        switch (db) {
            case 1: seg_place<1>(kA, vA, kB, vB, wcur, wnext, n, R, lspan, shift, last); break;
            case 2: seg_place<2>(kA, vA, kB, vB, wcur, wnext, n, R, lspan, shift, last); break;
            case 3: seg_place<3>(kA, vA, kB, vB, wcur, wnext, n, R, lspan, shift, last); break;
            case 4: seg_place<4>(kA, vA, kB, vB, wcur, wnext, n, R, lspan, shift, last); break;
            case 5: seg_place<5>(kA, vA, kB, vB, wcur, wnext, n, R, lspan, shift, last); break;
            case 6: seg_place<6>(kA, vA, kB, vB, wcur, wnext, n, R, lspan, shift, last); break;
            default: seg_place<7>(kA, vA, kB, vB, wcur, wnext, n, R, lspan, shift, last); break;
        }
        uint16_t* tv = vA; vA = vB; vB = tv;
        uint16_t* tk = kA; kA = kB; kB = tk;
        uint32_t* tw = wcur; wcur = wnext; wnext = tw;
    }
}

}  // namespace cdk
