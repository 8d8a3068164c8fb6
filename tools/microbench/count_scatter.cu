// Round 2: would a counting sort (global atomics) beat the backward's segment-local radix passes at
// c5 (B = 4, N = M = 2^20: 8.4M NN edges, 8.4M distinct targets)?  Times, on uniformly random keys:
//   count   rank[p] = atomicAdd(&cnt[key[p]], 1)          (8.4M int atomics with return, L2-resident)
//   scan    exclusive scan of cnt (3 kernels: tile sums, scan of sums, tile scan)
//   place   vals[off[key[p]] + rank[p]] = p               (random gather + random scatter)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o count_scatter count_scatter.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void count_k(const uint32_t* __restrict__ key, uint32_t* cnt, uint32_t* rank, int L) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L; p += gridDim.x * blockDim.x)
        rank[p] = atomicAdd(&cnt[key[p]], 1u);
}
__global__ void count_norank_k(const uint32_t* __restrict__ key, uint32_t* cnt, int L) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L; p += gridDim.x * blockDim.x)
        atomicAdd(&cnt[key[p]], 1u);
}
constexpr int kT = 4096;
__global__ void tile_sum_k(const uint32_t* __restrict__ cnt, uint32_t* sums, int K) {
    __shared__ uint32_t s[32];
    uint32_t v = 0;
    for (int i = blockIdx.x * kT + threadIdx.x; i < min(K, (blockIdx.x + 1) * kT); i += blockDim.x) v += cnt[i];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < (int)blockDim.x / 32; ++w) t += s[w];
        sums[blockIdx.x] = t;
    }
}
__global__ void scan_sums_k(uint32_t* sums, int n) {
    if (threadIdx.x == 0) {
        uint32_t r = 0;
        for (int i = 0; i < n; ++i) {
            const uint32_t c = sums[i];
            sums[i] = r;
            r += c;
        }
    }
}
__global__ void tile_scan_k(const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ sums, uint32_t* off, int K) {
    // 1024 threads, 4 items each
    __shared__ uint32_t ws[32];
    const int base = blockIdx.x * kT + threadIdx.x * 4;
    uint32_t v[4], t = 0;
    for (int u = 0; u < 4; ++u) {
        v[u] = base + u < K ? cnt[base + u] : 0;
        t += v[u];
    }
    uint32_t incl = t;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint32_t x = ws[lane], ix = x;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(~0u, ix, o);
            if (lane >= o) ix += y;
        }
        ws[lane] = ix - x;
    }
    __syncthreads();
    uint32_t r = sums[blockIdx.x] + ws[w] + incl - t;
    for (int u = 0; u < 4; ++u) {
        if (base + u < K) off[base + u] = r;
        r += v[u];
    }
}
__global__ void place_k(const uint32_t* __restrict__ key, const uint32_t* __restrict__ rank,
                        const uint32_t* __restrict__ off, uint32_t* vals, int L) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L; p += gridDim.x * blockDim.x)
        vals[off[key[p]] + rank[p]] = (uint32_t)p;
}

int main() {
    const int L = 8 << 20, K = 8 << 20;
    std::vector<uint32_t> hk(L);
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < L; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        // segment-local NN targets: edge i of segment i / 2^20 -> a key in the same segment
        hk[i] = (uint32_t)((i >> 20) << 20) + (uint32_t)(s % (1u << 20));
    }
    uint32_t *key, *cnt, *rank, *off, *vals, *sums;
    cudaMalloc(&key, L * 4); cudaMalloc(&cnt, K * 4); cudaMalloc(&rank, L * 4); cudaMalloc(&off, K * 4);
    cudaMalloc(&vals, L * 4); cudaMalloc(&sums, (K / kT + 1) * 4);
    cudaMemcpy(key, hk.data(), L * 4, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e[8];
    for (auto& x : e) cudaEventCreate(&x);
    const int nt = (K + kT - 1) / kT;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemsetAsync(cnt, 0, K * 4);
        cudaEventRecord(e[0]);
        count_k<<<sms * 8, 256>>>(key, cnt, rank, L);
        cudaEventRecord(e[1]);
        tile_sum_k<<<nt, 1024>>>(cnt, sums, K);
        scan_sums_k<<<1, 32>>>(sums, nt);
        tile_scan_k<<<nt, 1024>>>(cnt, sums, off, K);
        cudaEventRecord(e[2]);
        place_k<<<sms * 8, 256>>>(key, rank, off, vals, L);
        cudaEventRecord(e[3]);
        cudaMemsetAsync(cnt, 0, K * 4);
        cudaEventRecord(e[4]);
        count_norank_k<<<sms * 8, 256>>>(key, cnt, L);
        cudaEventRecord(e[5]);
        cudaDeviceSynchronize();
        float a, b, c, d;
        cudaEventElapsedTime(&a, e[0], e[1]);
        cudaEventElapsedTime(&b, e[1], e[2]);
        cudaEventElapsedTime(&c, e[2], e[3]);
        cudaEventElapsedTime(&d, e[4], e[5]);
        printf("count+rank %.1f us  scan %.1f us  place %.1f us  (count without rank %.1f us)  err=%s\n", a * 1e3,
               b * 1e3, c * 1e3, d * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    // check: every position written once, runs hold their key
    std::vector<uint32_t> hv(L), ho(K);
    cudaMemcpy(hv.data(), vals, L * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ho.data(), off, K * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int q = 0; q < L; ++q) {
        const uint32_t p = hv[q], k = hk[p];
        const uint32_t lo = ho[k], hi = k + 1 < (uint32_t)K ? ho[k + 1] : (uint32_t)L;
        bad += !(q >= (int)lo && q < (int)hi);
    }
    printf("placement check: %ld bad\n", bad);
    return 0;
}
