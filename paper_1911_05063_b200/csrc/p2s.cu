// p2s.cu — point-to-surface loss ("the point-to-surface loss
// [GEOMetrics] for Meshes"): for every point the squared distance to the closest
// triangle of its batch element's mesh, loss = mean_b mean_i d, VJP with the closest point fixed.
// Readings R23-R25.  Same tile engine as the Chamfer forward:
//
//   p2s_prep_kernel   per (b, face): the face's fixed-order fp32 data (a, e0 = b-a, e1 = c-a,
//                     e2 = c-b, unit normal, 1/|e|^2, inverse Gram matrix) packed as 24 floats; the
//                     face list is padded to the tile size by repeating the last face (same distance,
//                     higher index: never the argmin).
//   p2s_kernel        CTA = 1024 points (8 per thread as 4 packed f32x2 pairs) x a split of the faces,
//                     face tiles staged by 1-D TMA bulk copies; per (point, face)
//                       d = min( inside ? (ap.n)^2 : +inf, |ap - sat(ap.e0/|e0|^2) e0|^2,
//                                |ap - sat(ap.e1/|e1|^2) e1|^2, |bp - sat(bp.e2/|e2|^2) e2|^2 )
//                     (R24: the distance to the triangle = the plane distance when the projection is
//                     inside, else the nearest edge); value-only running minimum + 32-face block
//                     argmin tracking exactly as nn_fwd_kernel.
//   p2s_merge_kernel  merges the splits, re-scans the winning block with the same fp32 ops (lowest
//                     face with the minimum), then evaluates the closest point on that face in fp64 with
//                     the region decomposition (d, closest point, barycentrics), fp64 chunk sums.
//   p2s_finalize_kernel  loss = (1/B) sum_b (1/N) sum_i d.
//   backward          grad_p = 2 g (p - c); grad_verts through the barycentrics of c with the
//                     deterministic vertex scatter of mesh_sample.cu (R25).
#include "cd_internal.h"
#include "p2s_common.cuh"

#include <algorithm>

namespace cdk {

struct PrepArgs {
    const float* verts;
    const int* faces;
    int B, Nv, Nf, Nfpad;
    float* fd;   // [B][Nfpad][24]
};

__global__ void __launch_bounds__(256) p2s_prep_kernel(PrepArgs a) {
    const int64_t total = (int64_t)a.B * a.Nfpad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(e / a.Nfpad);
        const int f = min((int)(e - (int64_t)b * a.Nfpad), a.Nf - 1);
        write_face_record(a.verts + (int64_t)b * a.Nv * 3, a.Nv, a.faces, f, a.fd + e * kFaceFloats);
    }
}

struct P2sArgs {
    const float4* pts;      // packed points [B][Ppad]
    const float* fd;        // [B][Nfpad][24]
    int N, Ppad, Nf, Nfpad;
    int qtiles, splits, ftiles;
    int64_t total;          // B * N
    float* best_d;          // [splits][B*N]
    int* best_blk;
};

__global__ void __launch_bounds__(kFwdThreads, 3) p2s_kernel(P2sArgs a) {
    __shared__ __align__(128) float sm[kP2sStages][kFaceTile * kFaceFloats];
    __shared__ __align__(8) u64 full_bar[kP2sStages];
    const int b = blockIdx.y;
    const int tile = blockIdx.x / a.splits;
    const int split = blockIdx.x - tile * a.splits;
    const int t0 = (int)((int64_t)split * a.ftiles / a.splits), t1 = (int)((int64_t)(split + 1) * a.ftiles / a.splits);
    const int ntiles = t1 - t0;
    const float* FD = a.fd + (int64_t)b * a.Nfpad * kFaceFloats;
    const uint32_t bytes = kFaceTile * kFaceFloats * 4;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kP2sStages; ++s) mbar_init(&full_bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int k = 0; k < min(kP2sStages, ntiles); ++k) {
            mbar_arrive_expect_tx(&full_bar[k], bytes);
            tma_load_1d(sm[k], FD + (int64_t)(t0 + k) * kFaceTile * kFaceFloats, bytes, &full_bar[k]);
        }
    const float4* P = a.pts + (int64_t)b * a.Ppad;
    const int qbase = tile * kP2sQ + threadIdx.x * kP2sR;
    u64 qx[kP2sR / 2], qy[kP2sR / 2], qz[kP2sR / 2];
#pragma unroll
    for (int r = 0; r < kP2sR / 2; ++r) {
        const float4 p0 = P[min(qbase + 2 * r, a.N - 1)], p1 = P[min(qbase + 2 * r + 1, a.N - 1)];
        qx[r] = pk2(p0.x, p1.x);
        qy[r] = pk2(p0.y, p1.y);
        qz[r] = pk2(p0.z, p1.z);
    }
    float best[kP2sR];
    int blk[kP2sR];
#pragma unroll
    for (int r = 0; r < kP2sR; ++r) {
        best[r] = INFINITY;
        blk[r] = -1;
    }
    for (int k = 0; k < ntiles; ++k) {
        const int s = k % kP2sStages;
        mbar_wait(&full_bar[s], (k / kP2sStages) & 1);
        const float* tb = sm[s];
        const int ft = (t0 + k) * kFaceTile;
        for (int kb = 0; kb < kFaceTile; kb += kBlockK) {
            float old[kP2sR];
#pragma unroll
            for (int r = 0; r < kP2sR; ++r) old[r] = best[r];
#pragma unroll 1
            for (int j = 0; j < kBlockK; ++j) {
                const float* f = tb + (kb + j) * kFaceFloats;
#pragma unroll
                for (int r = 0; r < kP2sR / 2; ++r) {
                    float d0, d1;
                    face_dist2(f, qx[r], qy[r], qz[r], d0, d1);
                    best[2 * r] = fminf(best[2 * r], d0);
                    best[2 * r + 1] = fminf(best[2 * r + 1], d1);
                }
            }
#pragma unroll
            for (int r = 0; r < kP2sR; ++r) blk[r] = best[r] < old[r] ? ft + kb : blk[r];
        }
        __syncthreads();
        if (threadIdx.x == 0 && k + kP2sStages < ntiles) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[s], bytes);
            tma_load_1d(sm[s], FD + (int64_t)(t0 + k + kP2sStages) * kFaceTile * kFaceFloats, bytes, &full_bar[s]);
        }
    }
    const int64_t rowbase = (int64_t)split * a.total + (int64_t)b * a.N;
#pragma unroll
    for (int r = 0; r < kP2sR; ++r) {
        const int q = qbase + r;
        if (q < a.N) {
            a.best_d[rowbase + q] = best[r];
            a.best_blk[rowbase + q] = blk[r];
        }
    }
}

struct P2sMergeArgs {
    const float4* pts;
    const float* fd;
    const float* verts;
    const int* faces;
    int B, N, Ppad, Nv, Nf, Nfpad, splits, nchunks;
    int64_t total;
    const float* best_d;
    const int* best_blk;
    float* d_out;       // [B][N]
    int* face_out;      // [B][N]
    float* closest;     // [B][N][3] (may be null)
    float* bary;        // [B][N][3] (may be null)
    double* chunk_sum;  // [B][nchunks]
};

__global__ void __launch_bounds__(kMergeThreads) p2s_merge_kernel(P2sMergeArgs a) {
    const int b = blockIdx.x / a.nchunks;
    const int chunk = blockIdx.x - b * a.nchunks;
    const int i = chunk * kMergeThreads + threadIdx.x;
    double v = 0.0;
    if (i < a.N) {
        const int64_t row = (int64_t)b * a.N + i;
        float best = INFINITY;
        int bb = -1;
        for (int s = 0; s < a.splits; ++s) {
            const float d = a.best_d[(int64_t)s * a.total + row];
            if (d < best) {
                best = d;
                bb = a.best_blk[(int64_t)s * a.total + row];
            }
        }
        const float4 pp = a.pts[(int64_t)b * a.Ppad + i];
        int face = 0;
        if (bb >= 0) {
            const u64 qx = pk2(pp.x, pp.x), qy = pk2(pp.y, pp.y), qz = pk2(pp.z, pp.z);
            const float* FD = a.fd + (int64_t)b * a.Nfpad * kFaceFloats;
            const int fend = min(bb + kBlockK, a.Nf);
            face = -1;
            for (int f = bb; f < fend; ++f) {
                float d0, d1;
                face_dist2(FD + (int64_t)f * kFaceFloats, qx, qy, qz, d0, d1);
                if (d0 == best) {
                    face = f;
                    break;
                }
            }
            if (face < 0) face = bb;
        }
        // fp64 closest point on the chosen face; no finite candidate (a non-finite point, R6):
        // (+inf, face -1, closest 0, bary 0), the oracle's values
        const float* vv = a.verts + (int64_t)b * a.Nv * 3;
        double A[3], Bv[3], C[3], p[3] = {pp.x, pp.y, pp.z}, c[3] = {0.0, 0.0, 0.0}, lam[3] = {0.0, 0.0, 0.0};
        double dd = INFINITY;
        if (bb >= 0) {
            const int ia = min(max(a.faces[3 * face], 0), a.Nv - 1), ib = min(max(a.faces[3 * face + 1], 0), a.Nv - 1),
                      ic = min(max(a.faces[3 * face + 2], 0), a.Nv - 1);
            for (int k = 0; k < 3; ++k) {
                A[k] = vv[3 * ia + k];
                Bv[k] = vv[3 * ib + k];
                C[k] = vv[3 * ic + k];
            }
            dd = face_foot64(p, A, Bv, C, c, lam);
        } else {
            face = -1;
        }
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

__global__ void __launch_bounds__(256) p2s_finalize_kernel(const double* chunk_sum, int B, int N, int nchunks,
                                                           float* per_batch, float* loss) {
    __shared__ double sl[256];
    double acc = 0.0;
    for (int b = threadIdx.x; b < B; b += 256) {
        double s = 0.0;
        for (int c = 0; c < nchunks; ++c) s += chunk_sum[(int64_t)b * nchunks + c];
        const double m = s / N;
        if (per_batch) per_batch[b] = (float)m;
        acc += m;
    }
    sl[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sl[threadIdx.x] += sl[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0 && loss) loss[0] = (float)(sl[0] / B);
}

void launch_p2s_finalize(const double* chunk_sum, int B, int N, int nchunks, float* per_batch, float* loss,
                         cudaStream_t st) {
    p2s_finalize_kernel<<<1, 256, 0, st>>>(chunk_sum, B, N, nchunks, per_batch, loss);
}

struct P2sPackArgs {
    const float* src;
    float4* dst;
    int N, Ppad, B;
};

__global__ void __launch_bounds__(256) p2s_pack_kernel(P2sPackArgs a) {
    const int64_t total = (int64_t)a.B * a.Ppad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / a.Ppad;
        const int i = (int)(e - b * a.Ppad);
        const int j = min(i, a.N - 1);
        const float* s = a.src + (b * a.N + j) * 3;
        a.dst[e] = make_float4(s[0], s[1], s[2], 0.f);
    }
}

__global__ void __launch_bounds__(256) p2s_grad_points_kernel(const float* pts, const float* closest, const float* g,
                                                              float g_scalar, const float* upstream, int64_t total,
                                                              float* grad_points, float* upstream_verts) {
    if (upstream) g_scalar = __fmul_rn(*upstream, g_scalar);   // loss backward: the fill RN(u * 1/(B N))
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const double gi = g ? (double)g[e] : (double)g_scalar;
        for (int k = 0; k < 3; ++k) {
            const double t = __dmul_rn(__dmul_rn(2.0, gi), __dsub_rn((double)pts[3 * e + k], (double)closest[3 * e + k]));
            if (grad_points) grad_points[3 * e + k] = (float)t;
            upstream_verts[3 * e + k] = (float)(-t);   // d/dc of |p - c|^2 = -2 (p - c)
        }
    }
}

// ------------------------------------------------------------------------------------------ host
static int cdiv(int64_t x, int64_t y) { return (int)((x + y - 1) / y); }

struct P2sPlan {
    int B, N, Nv, Nf, Ppad, Nfpad, qtiles, ftiles, splits, nchunks;
    size_t off_pts, off_fd, off_best_d, off_best_blk, off_chunk, bytes;
};

// cd_set_forward_splits also forces the point-to-surface split count (design sweeps)
static thread_local int g_p2s_forced_splits = 0;
void set_p2s_forced_splits(int s) { g_p2s_forced_splits = s > 0 ? s : 0; }

static void plan_p2s(P2sPlan& p, int B, int N, int Nv, int Nf) {
    p.B = B;
    p.N = N;
    p.Nv = Nv;
    p.Nf = Nf;
    p.Ppad = cdiv(N, kP2sQ) * kP2sQ;
    p.Nfpad = cdiv(Nf, kFaceTile) * kFaceTile;
    p.qtiles = p.Ppad / kP2sQ;
    p.ftiles = p.Nfpad / kFaceTile;
    const int sms = current_sm_count();
    const int64_t units = (int64_t)B * p.qtiles, slots = (int64_t)sms * 3;
    // t(S) = U (T + S c0) / slots + (ceil(T/S) + c0) / 2, c0 = 0.1 face tile: the fused kernel's fitted
    // split model (nn_forward.cu); sweep (tools/sweep_p2s_splits.py, NEXT-3 workload): S = 32-40
    // 4.37-4.39 ms vs 4.54 ms at the ceil-wave model's choice
    int best = 1;
    double bt = 1e300;
    for (int s = 1; s <= std::min(64, p.ftiles); ++s) {
        const double t = (double)units * (p.ftiles + 0.1 * s) / (double)slots + 0.5 * ((double)cdiv(p.ftiles, s) + 0.1);
        if (t < bt * 0.999) {
            bt = t;
            best = s;
        }
    }
    p.splits = g_p2s_forced_splits > 0 ? std::min(g_p2s_forced_splits, p.ftiles) : best;
    p.nchunks = cdiv(N, kMergeThreads);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    p.off_pts = take((size_t)B * p.Ppad * 16);
    p.off_fd = take((size_t)B * p.Nfpad * kFaceFloats * 4);
    p.off_best_d = take((size_t)p.splits * B * N * 4);
    p.off_best_blk = take((size_t)p.splits * B * N * 4);
    p.off_chunk = take((size_t)B * p.nchunks * 8);
    p.bytes = off;
}

size_t p2s_workspace(int B, int N, int Nv, int Nf) {
    P2sPlan p;
    plan_p2s(p, B, N, Nv, Nf);
    return p.bytes;
}

size_t p2s_backward_workspace(int B, int N, int Nv, int Nf) {
    return align_up((size_t)B * N * 12, 256) + sample_backward_workspace(B, Nv, Nf, N);
}

cudaError_t launch_p2s(const float* points, const float* verts, const int* faces, int B, int N, int Nv, int Nf,
                       float* d, int* face, float* closest, float* bary, float* per_batch, float* loss, void* ws,
                       cudaStream_t st) {
    P2sPlan p;
    plan_p2s(p, B, N, Nv, Nf);
    char* w = static_cast<char*>(ws);
    float4* pts = reinterpret_cast<float4*>(w + p.off_pts);
    float* fd = reinterpret_cast<float*>(w + p.off_fd);
    float* best_d = reinterpret_cast<float*>(w + p.off_best_d);
    int* best_blk = reinterpret_cast<int*>(w + p.off_best_blk);
    double* chunk = reinterpret_cast<double*>(w + p.off_chunk);
    {
        P2sPackArgs a{points, pts, N, p.Ppad, B};
        p2s_pack_kernel<<<std::min(cdiv((int64_t)B * p.Ppad, 256), current_sm_count() * 16), 256, 0, st>>>(a);
    }
    {
        PrepArgs a{verts, faces, B, Nv, Nf, p.Nfpad, fd};
        p2s_prep_kernel<<<std::min(cdiv((int64_t)B * p.Nfpad, 256), current_sm_count() * 16), 256, 0, st>>>(a);
    }
    {
        P2sArgs a;
        a.pts = pts;
        a.fd = fd;
        a.N = N;
        a.Ppad = p.Ppad;
        a.Nf = Nf;
        a.Nfpad = p.Nfpad;
        a.qtiles = p.qtiles;
        a.splits = p.splits;
        a.ftiles = p.ftiles;
        a.total = (int64_t)B * N;
        a.best_d = best_d;
        a.best_blk = best_blk;
        if (g_prof_start) record_profile_event(g_prof_start, st);
        p2s_kernel<<<dim3(p.qtiles * p.splits, B), kFwdThreads, 0, st>>>(a);
        if (g_prof_stop) record_profile_event(g_prof_stop, st);
    }
    {
        P2sMergeArgs a;
        a.pts = pts;
        a.fd = fd;
        a.verts = verts;
        a.faces = faces;
        a.B = B;
        a.N = N;
        a.Ppad = p.Ppad;
        a.Nv = Nv;
        a.Nf = Nf;
        a.Nfpad = p.Nfpad;
        a.splits = p.splits;
        a.nchunks = p.nchunks;
        a.total = (int64_t)B * N;
        a.best_d = best_d;
        a.best_blk = best_blk;
        a.d_out = d;
        a.face_out = face;
        a.closest = closest;
        a.bary = bary;
        a.chunk_sum = chunk;
        p2s_merge_kernel<<<B * p.nchunks, kMergeThreads, 0, st>>>(a);
    }
    if (per_batch || loss) p2s_finalize_kernel<<<1, 256, 0, st>>>(chunk, B, N, p.nchunks, per_batch, loss);
    return cudaGetLastError();
}

cudaError_t launch_p2s_backward(const float* points, const float* closest, const int* face, const float* bary,
                                const int* faces, int B, int N, int Nv, int Nf, const float* g, float g_scalar,
                                const float* upstream, float* grad_points, float* grad_verts, void* ws, cudaStream_t st) {
    char* w = static_cast<char*>(ws);
    float* up = reinterpret_cast<float*>(w);
    const int64_t total = (int64_t)B * N;
    p2s_grad_points_kernel<<<std::min(cdiv(total, 256), current_sm_count() * 16), 256, 0, st>>>(points, closest, g, g_scalar, upstream,
                                                                                 total, grad_points, up);
    if (grad_verts)
        return launch_sample_backward(faces, face, bary, B, Nv, Nf, N, up, grad_verts,
                                      w + align_up((size_t)B * N * 12, 256), st);
    return cudaGetLastError();
}

int p2s_launches() { return 5; }

}  // namespace cdk
