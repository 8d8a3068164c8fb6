// cd_internal.h — host-side launch plumbing shared by the libcd translation units (not public).
#pragma once
#include <atomic>
#include <utility>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace cdk {

// Forward modes: the unfused kernel searches each direction separately (any query slices); the
// fused kernel evaluates every distance once for both directions.
enum FwdMode { kUnfused = 0, kFusedFull = 1, kFusedRows = 2, kFusedCols = 3, kTensor = 4 };
// identity of the column-key min: larger than every key (keys are non-negative int64)
constexpr long long kColKeyEmpty = 0x7fffffffffffffffLL;

// Forward problem description (one direction = "dir": 0 = X queries vs Y targets, 1 = Y vs X).
constexpr int kMaxPeers = 16;   // cd_forward_cols_peers: key arrays reduced on read (CD_MAX_PEERS)

struct FwdPlan {
    int mode;
    int B;
    int npts[2];        // points per batch element of cloud 0 (X: N) and cloud 1 (Y: M)
    int ppad[2];        // padded stride of the packed clouds
    int qlo[2], qhi[2]; // query slice per dir (dir 0 queries X, dir 1 queries Y)
    int qtiles[2];      // query tiles per (dir, b)
    int splits[2];      // target splits per dir
    int ttiles[2];      // target tiles (kTile points) per dir; split s covers [s*T/S, (s+1)*T/S)
    int64_t slice_off[2];  // offset of dir's rows inside the [B*sq + B*sr] per-split arrays
    int64_t slice_total;   // B*sq + B*sr
    int nchunks[2];     // merge chunks (kMergeThreads queries) per (dir, b)
    int64_t chunk_off[2];
    int64_t chunk_total;
    // workspace carve (byte offsets)
    size_t off_pack[2], off_rowkey, off_chunk_sum, off_chunk_hits, off_colkey, bytes;
    int forced_splits;   // 0: automatic
    int split_unit;      // fused kernel: targets per split unit (kTile, or kBlockK for small M)
    int fused_rows;      // fused kernel: rows per thread (kR = 16, or kRSmall = 8 for small clouds)
};

struct FwdOutputs {
    float* d[2];
    int32_t* idx[2];
    double* partials;   // B x 4 or nullptr
    float tau;          // < 0: no hits
    long long* colkey;  // fused rows/cols modes: caller's B x M column keys (out / in)
    // cols mode, peer reads (cd_forward_cols_peers): the column keys are the element-wise MIN of
    // npeers B x M arrays (this rank's and its peers', read over NVLink), reduced as they are read
    const long long* colkey_peers[kMaxPeers];
    int npeers = 0;
};

// Tensor-core forward (nn_tc.cu, R27): full problems only.
struct TcPlan {
    int B, npts[2], ppad[2], qblocks, ttiles, splits, nchunks[2];
    int64_t chunk_off[2];
    size_t off_box, off_pack[2], off_op[2], off_rowsum, off_colsum, off_fb, off_chunk_sum, off_chunk_hits, bytes;
};
void plan_tc(TcPlan& p, int B, int N, int M, int forced_splits);
int tc_launches(const TcPlan& p);
struct FwdOutputs;
cudaError_t launch_tc(const TcPlan& p, const float* x, const float* y, const FwdOutputs& o, void* ws, cudaStream_t st);

void plan_forward(FwdPlan& p, int mode, int B, int N, int M, int q0, int q1, int r0, int r1, int forced_splits);
cudaError_t launch_forward(const FwdPlan& p, const float* x, const float* y, const FwdOutputs& o, void* ws,
                           cudaStream_t st);
int forward_launches(const FwdPlan& p);
int fused_ctas_per_sm(int rows);
int unfused_ctas_per_sm();
// fused kernels (nn_fused.cu)
cudaError_t launch_fused_rows(const FwdPlan& p, const float4* xp, const float4* yp, long long* colkey,
                              long long* rowkey, cudaStream_t st);


// Exact pruned forward (nn_pruned.cu, NEXT-2): Hilbert-sorted tiles + box lower-bound culling.
// A sequence sorted as independent segments: nA segments of szA elements, then nB of szB.
struct SegSpec {
    int nA;
    int64_t szA;
    int nB;
    int64_t szB;
};

struct PrunedPlan {
    int B, npts[2], ppad[2], qtiles[2], cqtiles[2], ttiles[2];
    int kbits, nbits;          // nbits = 3*kbits: segment-local Hilbert keys
    SegSpec segs;              // the 2B (cloud, batch) segments the radix passes sort on their own
    int64_t L, cand_off[2];
    int nchunks[2];
    int64_t chunk_off[2];
    bool supported;
    bool hier;                 // two-level (super-tile) candidate search
    size_t off_bbox, off_keys[2], off_vals[2], off_counts, off_totals, off_sorted[2], off_perm[2], off_box[2], off_box32[2],
        off_best_d[2], off_best_blk[2], off_sbox[2], off_cand, off_ccount, off_chunk_sum, off_chunk_hits, off_fb, bytes;
};
void plan_pruned(PrunedPlan& p, int B, int N, int M);
cudaError_t launch_pruned(const PrunedPlan& p, const float* x, const float* y, const FwdOutputs& o, void* ws,
                          cudaStream_t st);
int pruned_launches(const PrunedPlan& p);
cudaError_t launch_partials(const double* chunk_sum, const int* chunk_hits, const int nchunks[2],
                            const int64_t chunk_off[2], int B, double* partials, int dirmask, cudaStream_t st);

// Differentiable mesh surface sampling (mesh_sample.cu, NEXT-4).
size_t sample_workspace(int B, int Nv, int Nf, int N);
cudaError_t launch_sample(const float* verts, const int* faces, int B, int Nv, int Nf, int N, const unsigned* r_face,
                          const float* r_bary, float* points, int* face_idx, float* bary, void* ws, cudaStream_t st);
size_t sample_backward_workspace(int B, int Nv, int Nf, int N);
int sample_backward_launches(int B, int Nv, int Nf, int N);
cudaError_t launch_sample_backward(const int* faces, const int* face_idx, const float* bary, int B, int Nv, int Nf,
                                   int N, const float* grad_points, float* grad_verts, void* ws, cudaStream_t st);

// Point-to-surface loss (p2s.cu, NEXT-3).
size_t p2s_workspace(int B, int N, int Nv, int Nf);
size_t p2s_backward_workspace(int B, int N, int Nv, int Nf);
cudaError_t launch_p2s(const float* points, const float* verts, const int* faces, int B, int N, int Nv, int Nf,
                       float* d, int* face, float* closest, float* bary, float* per_batch, float* loss, void* ws,
                       cudaStream_t st);
cudaError_t launch_p2s_backward(const float* points, const float* closest, const int* face, const float* bary,
                                const int* faces, int B, int N, int Nv, int Nf, const float* g, float g_scalar,
                                const float* upstream, float* grad_points, float* grad_verts, void* ws, cudaStream_t st);
int p2s_launches();
void launch_p2s_finalize(const double* chunk_sum, int B, int N, int nchunks, float* per_batch, float* loss,
                         cudaStream_t st);
// Culled point-to-surface forward (p2s_pruned.cu, R26); workspace 0 = unsupported size.
size_t p2s_pruned_workspace(int B, int N, int Nv, int Nf);
int p2s_pruned_launches(int B, int N, int Nv, int Nf);
cudaError_t launch_p2s_pruned(const float* points, const float* verts, const int* faces, int B, int N, int Nv, int Nf,
                              float* d, int* face, float* closest, float* bary, float* per_batch, float* loss,
                              void* ws, cudaStream_t st);
// Per-(cloud, batch) sample bounding boxes [2][B][6] (nn_pruned.cu).
int hilbert_bits(int nmax);
void launch_bbox(const float* src0, int n0, const float* src1, int n1, int B, float* bbox, cudaStream_t st);

// Stats of given distances (for cd_fscore): per-chunk sums + hits, then partials.
size_t fscore_workspace(int B, int N, int M);
cudaError_t launch_fscore(const float* d_xy, const float* d_yx, int B, int N, int M, float tau, float* fscore,
                          float* precision, float* recall, void* ws, cudaStream_t st);
constexpr int kFscoreLaunches = 3;

cudaError_t launch_finalize(const double* partials, int B, int N, int M, float w1, float w2, float* cd,
                            float* loss, float* fscore, float* precision, float* recall, cudaStream_t st);

// Backward.
struct BwdPlan {
    int B, N, M;
    int q0, q1, r0, r1;
    int64_t L;          // B*(N+M) key/value pairs
    int64_t kmax;       // number of distinct keys B*(M+N)
    int nbits, npasses, digit_bits, ntiles;
    bool segsort;       // max(N, M) <= 24576: one CTA per (direction, batch) segment sorts on chip
    SegSpec segs;       // else: the global radix passes sort the 2B (direction, batch) segments on their own
    size_t off_keys[2], off_vals[2], off_counts, off_totals, off_offsets, bytes;
};
void plan_backward(BwdPlan& p, int B, int N, int M, int q0, int q1, int r0, int r1);
cudaError_t launch_backward(const BwdPlan& p, const float* x, const float* y, const int32_t* idx_xy,
                            const int32_t* idx_yx, const float* g, const float* h, float g_scalar, float h_scalar,
                            const float* upstream, float* grad_x, float* grad_y, void* ws, cudaStream_t st);
int backward_launches(const BwdPlan& p);

// Reusable stable LSD radix sort of u32 (key, value) pairs (nn_backward.cu).
int radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t L, int nbits, uint32_t* counts, uint32_t* totals,
                     cudaStream_t st, bool first_hist_done = false);
int radix_digit_bits(int64_t L, int nbits);
size_t radix_sort_counts_words(int64_t L, int nbits);
int radix_sort_launches(int64_t L, int nbits);
// Segmented form: every segment of `sp` sorted on its own by the low `nbits` bits of segment-local
// keys; narrow = true picks the digit width by the measured pass-cost model (nn_backward.cu).
int radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], const SegSpec& sp, int nbits, uint32_t* counts,
                     uint32_t* totals, cudaStream_t st, bool first_hist_done, bool narrow);
size_t radix_sort_counts_words(const SegSpec& sp, int nbits, bool narrow);
size_t radix_sort_totals_words(const SegSpec& sp, int nbits, bool narrow);
int radix_sort_launches(const SegSpec& sp, int nbits, bool narrow);
constexpr int kSortTotalsWords = 1 << 12;   // >= 2^kMaxDigitBits

// thread-local measurement hook (cd_set_profile_events)
extern thread_local cudaEvent_t g_prof_start;
extern thread_local cudaEvent_t g_prof_stop;

// Record a measurement event; inside stream capture it must be an external event-record node so a
// graph replay re-records it (a plain record during capture only expresses a dependency).
inline void record_profile_event(cudaEvent_t ev, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
    else
        cudaEventRecord(ev, st);
}

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Process-wide per-device caches of device attributes / occupancies: one slot per device ordinal,
// filled on first use by `f` (idempotent: racing threads store the same value), read by every
// thread — the library's only mutable global state besides the thread-local error string.
constexpr int kMaxDevices = 64;
template <class F>
inline int per_device_cached(std::atomic<int>* table, F f) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
        cudaGetLastError();
        return f();
    }
    int v = table[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        v = f();
        table[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

// SMs of the current device (148 on B200; the fallback if the query fails).
inline int current_sm_count() {
    static std::atomic<int> table[kMaxDevices];
    return per_device_cached(table, [] {
        int dev = 0, s = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || s <= 0) {
            cudaGetLastError();
            s = 148;
        }
        return s;
    });
}

// Resident CTAs per SM of `kernel` with `threads` threads and `smem` dynamic bytes on the current
// device (`fallback` if the query fails).
template <class K>
inline int occupancy_of(std::atomic<int>* table, K kernel, int threads, size_t smem, int fallback) {
    return per_device_cached(table, [&] {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, threads, smem) != cudaSuccess || o <= 0) {
            cudaGetLastError();
            o = fallback;
        }
        return o;
    });
}

// Opt a kernel into more than 48 KB of dynamic shared memory, once per (device, kernel) on the
// calling thread (the attribute is per device: a thread that switches devices sets it again).
inline void ensure_smem_attr(const void* func, int bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    static thread_local const void* done_fn[32];
    static thread_local int done_dev[32];
    static thread_local int ndone = 0;
    for (int i = 0; i < ndone; ++i)
        if (done_fn[i] == func && done_dev[i] == dev) return;
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (ndone < 32) {
        done_fn[ndone] = func;
        done_dev[ndone] = dev;
        ++ndone;
    }
}


// Launch with programmatic stream serialisation when CD_PDL (see pdl_wait in cd_device.cuh).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
#if defined(CD_PDL) && CD_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
#else
    kernel<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
    return cudaSuccess;
#endif
}
void set_p2s_forced_splits(int s);   // p2s.cu (cd_set_forward_splits)

}  // namespace cdk
