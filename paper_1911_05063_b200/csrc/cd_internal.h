// cd_internal.h — host-side launch plumbing shared by the libcd translation units (not public).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace cdk {

// Forward problem description (one direction = "dir": 0 = X queries vs Y targets, 1 = Y vs X).
struct FwdPlan {
    int B;
    int npts[2];        // points per batch element of cloud 0 (X: N) and cloud 1 (Y: M)
    int ppad[2];        // padded stride of the packed clouds
    int qlo[2], qhi[2]; // query slice per dir (dir 0 queries X, dir 1 queries Y)
    int qtiles[2];      // query tiles per (dir, b)
    int splits[2];      // target splits per dir
    int split_len[2];   // targets per split (multiple of kTile)
    int64_t slice_off[2];  // offset of dir's rows inside the [B*sq + B*sr] per-split arrays
    int64_t slice_total;   // B*sq + B*sr
    int nchunks[2];     // merge chunks (kMergeThreads queries) per (dir, b)
    int64_t chunk_off[2];
    int64_t chunk_total;
    // workspace carve (byte offsets)
    size_t off_pack[2], off_best_d, off_best_blk, off_chunk_sum, off_chunk_hits, bytes;
};

struct FwdOutputs {
    float* d[2];
    int32_t* idx[2];
    double* partials;   // B x 4 or nullptr
    float tau;          // < 0: no hits
};

void plan_forward(FwdPlan& p, int B, int N, int M, int q0, int q1, int r0, int r1, int forced_splits);
cudaError_t launch_forward(const FwdPlan& p, const float* x, const float* y, const FwdOutputs& o, void* ws,
                           cudaStream_t st);
constexpr int kForwardLaunches = 4;

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
    int nbits, npasses, ntiles;
    size_t off_keys[2], off_vals[2], off_counts, off_offsets, bytes;
};
void plan_backward(BwdPlan& p, int B, int N, int M, int q0, int q1, int r0, int r1);
cudaError_t launch_backward(const BwdPlan& p, const float* x, const float* y, const int32_t* idx_xy,
                            const int32_t* idx_yx, const float* g, const float* h, float g_scalar, float h_scalar,
                            float* grad_x, float* grad_y, void* ws, cudaStream_t st);
int backward_launches(const BwdPlan& p);

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace cdk
