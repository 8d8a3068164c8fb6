// cd_api.cu — the C ABI of libcd.so (declared in include/cd.h): validation, workspace carving and
// launch sequencing.  No allocation, no synchronisation; everything is asynchronous on `stream`.
#include "../../include/cd.h"
#include "cd_internal.h"

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

namespace {

thread_local std::string g_err;
thread_local int g_forced_splits = 0;
thread_local int g_forward_mode = 0;  // 0 auto, 1 unfused, 2 fused (FP32 pipe), 3 tensor-core filter

int auto_mode(int N, int M, int q0, int q1, int r0, int r1) {
    const bool full = q0 == 0 && q1 == N && r0 == 0 && r1 == M;
    if (g_forward_mode == 1 || !full) return cdk::kUnfused;
    if (g_forward_mode == 3) return cdk::kTensor;
    return cdk::kFusedFull;
}

cd_status fail(cd_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
cd_status fail(cd_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

cd_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return CD_OK;
    return fail(CD_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

constexpr int kMaxBatch = 65535;   // batch elements map to gridDim.y

cd_status check_sizes(int B, int N, int M) {
    if (B < 1 || N < 1 || M < 1)
        return fail(CD_ERR_INVALID_VALUE, "B, N, M must be >= 1 (empty cloud, SPEC.md:440-442): B=%d N=%d M=%d", B,
                    N, M);
    const long long L = (long long)B * ((long long)N + (long long)M);
    if (L > 0x7fffffffLL) return fail(CD_ERR_TOO_LARGE, "B*(N+M) = %lld exceeds 2^31-1", L);
    if (B > kMaxBatch) return fail(CD_ERR_TOO_LARGE, "B = %d exceeds %d (one grid row per batch element)", B, kMaxBatch);
    return CD_OK;
}

cd_status check_device() {
    int dev = 0, major = 0, minor = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return fail(CD_ERR_UNSUPPORTED_DEVICE, "device %d is sm_%d%d; libcd is built for sm_100a only", dev, major,
                    minor);
    return CD_OK;
}

size_t forward_ws(int B, int N, int M, int q0, int q1, int r0, int r1) {
    // large enough for either FP32-pipe forward kernel (the mode is chosen per call); the tensor-core
    // filter's per-(query block, column) summaries grow as N*M/128, so its workspace is only
    // included while forward mode 3 is selected on this thread (a call in mode 3 with a smaller
    // workspace fails with CD_ERR_TOO_LARGE before any launch)
    cdk::FwdPlan p, u;
    cdk::plan_forward(p, cdk::kFusedFull, B, N, M, q0, q1, r0, r1, g_forced_splits);
    cdk::plan_forward(u, cdk::kUnfused, B, N, M, q0, q1, r0, r1, g_forced_splits);
    size_t bytes = std::max(p.bytes, u.bytes);
    if (g_forward_mode == 3 && q0 == 0 && q1 == N && r0 == 0 && r1 == M) {
        cdk::FwdPlan t;
        cdk::plan_forward(t, cdk::kTensor, B, N, M, q0, q1, r0, r1, g_forced_splits);
        bytes = std::max(bytes, t.bytes);
    }
    return bytes;
}

int fwd_launches(int B, int N, int M) {
    cdk::FwdPlan p;
    cdk::plan_forward(p, auto_mode(N, M, 0, N, 0, M), B, N, M, 0, N, 0, M, g_forced_splits);
    return cdk::forward_launches(p);
}

// cd_step_host workspace: staging of x, y, outputs of forward, partials/loss/fscore, grads, plus
// the larger of the forward and backward workspaces.
struct StepLayout {
    size_t x, y, dxy, ixy, dyx, iyx, part, loss, fs, gx, gy, inner, inner2, inner_bytes, bytes;
};
StepLayout step_layout(int B, int N, int M) {
    StepLayout s;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = cdk::align_up(off + bytes, 256);
        return o;
    };
    s.x = take((size_t)B * N * 12);
    s.y = take((size_t)B * M * 12);
    s.dxy = take((size_t)B * N * 4);
    s.ixy = take((size_t)B * N * 4);
    s.dyx = take((size_t)B * M * 4);
    s.iyx = take((size_t)B * M * 4);
    s.part = take((size_t)B * 32);
    s.loss = take(4);
    s.fs = take((size_t)B * 4);
    s.gx = take((size_t)B * N * 12);
    s.gy = take((size_t)B * M * 12);
    cdk::BwdPlan bp;
    cdk::plan_backward(bp, B, N, M, 0, N, 0, M);
    s.inner_bytes = std::max(forward_ws(B, N, M, 0, N, 0, M), bp.bytes);
    s.inner = take(s.inner_bytes);
    s.inner2 = take(s.inner_bytes);   // cd_step_host_overlapped's second compute stream
    s.bytes = off;
    return s;
}

}  // namespace

extern "C" {

int cd_abi_version(void) { return CD_ABI_VERSION; }

const char* cd_status_string(cd_status s) {
    switch (s) {
        case CD_OK: return "CD_OK";
        case CD_ERR_INVALID_VALUE: return "CD_ERR_INVALID_VALUE";
        case CD_ERR_MISALIGNED: return "CD_ERR_MISALIGNED";
        case CD_ERR_TOO_LARGE: return "CD_ERR_TOO_LARGE";
        case CD_ERR_UNSUPPORTED_DEVICE: return "CD_ERR_UNSUPPORTED_DEVICE";
        case CD_ERR_CUDA: return "CD_ERR_CUDA";
    }
    return "CD_ERR_UNKNOWN";
}

// The loss's fills (R8): RN32(w / (B P)) in fp64 then rounded once.
static float loss_fill(float w, int B, int P) { return (float)((double)w / ((double)B * P)); }

const char* cd_last_error_string(void) { return g_err.c_str(); }

void cd_set_profile_events(void* start, void* stop) {
    cdk::g_prof_start = static_cast<cudaEvent_t>(start);
    cdk::g_prof_stop = static_cast<cudaEvent_t>(stop);
}

int cd_set_forward_splits(int splits) {
    int old = g_forced_splits;
    g_forced_splits = splits > 0 ? splits : 0;
    cdk::set_p2s_forced_splits(g_forced_splits);
    return old;
}

size_t cd_workspace_size(int op, int B, int N, int M) {
    if (B < 1 || N < 1 || M < 1) return 0;
    if ((long long)B * ((long long)N + M) > 0x7fffffffLL) return 0;
    switch (op) {
        case CD_OP_FORWARD: return forward_ws(B, N, M, 0, N, 0, M);
        case CD_OP_FSCORE: return cdk::fscore_workspace(B, N, M);
        case CD_OP_BACKWARD: {
            cdk::BwdPlan p;
            cdk::plan_backward(p, B, N, M, 0, N, 0, M);
            return p.bytes;
        }
        case CD_OP_STEP: return step_layout(B, N, M).bytes;
        case CD_OP_FORWARD_PRUNED: {
            cdk::PrunedPlan p;
            cdk::plan_pruned(p, B, N, M);
            return p.bytes;
        }
    }
    return 0;
}

int cd_launch_count(int op, int B, int N, int M) {
    if (B < 1 || N < 1 || M < 1) return 0;
    cdk::BwdPlan bp;
    cdk::plan_backward(bp, B, N, M, 0, N, 0, M);
    switch (op) {
        case CD_OP_FORWARD: return fwd_launches(B, N, M);
        case CD_OP_FSCORE: return cdk::kFscoreLaunches;
        case CD_OP_BACKWARD: return cdk::backward_launches(bp);
        case CD_OP_STEP: return fwd_launches(B, N, M) + 1 + cdk::backward_launches(bp);
        case CD_OP_FORWARD_PRUNED: {
            cdk::PrunedPlan p;
            cdk::plan_pruned(p, B, N, M);
            return cdk::pruned_launches(p);
        }
    }
    return 0;
}

cd_status cd_forward(const float* x, const float* y, int B, int N, int M, int q0, int q1, int r0, int r1,
                     float* d_xy, int32_t* idx_xy, float* d_yx, int32_t* idx_yx, double* partials, float tau,
                     void* workspace, size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!x || !y || !workspace) return fail(CD_ERR_INVALID_VALUE, "null x, y or workspace pointer");
    if (q0 < 0 || q1 < q0 || q1 > N || r0 < 0 || r1 < r0 || r1 > M)
        return fail(CD_ERR_INVALID_VALUE, "bad query slices [%d,%d) of N=%d, [%d,%d) of M=%d", q0, q1, N, r0, r1, M);
    if (q1 > q0 && (!d_xy || !idx_xy)) return fail(CD_ERR_INVALID_VALUE, "null d_xy / idx_xy");
    if (r1 > r0 && (!d_yx || !idx_yx)) return fail(CD_ERR_INVALID_VALUE, "null d_yx / idx_yx");
    if (tau != tau) return fail(CD_ERR_INVALID_VALUE, "tau is NaN");
    if (!aligned(x, 4) || !aligned(y, 4)) return fail(CD_ERR_MISALIGNED, "cloud pointers must be 4-byte aligned");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    cdk::FwdPlan p;
    cdk::plan_forward(p, auto_mode(N, M, q0, q1, r0, r1), B, N, M, q0, q1, r0, r1, g_forced_splits);
    if (workspace_bytes < p.bytes)
        return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu bytes", workspace_bytes, p.bytes);
    s = check_device();
    if (s != CD_OK) return s;
    cdk::FwdOutputs o;
    o.d[0] = d_xy;
    o.d[1] = d_yx;
    o.idx[0] = idx_xy;
    o.idx[1] = idx_yx;
    o.partials = partials;
    o.tau = tau;
    o.colkey = nullptr;
    return cuda_status(cdk::launch_forward(p, x, y, o, workspace, static_cast<cudaStream_t>(stream)), "cd_forward");
}

cd_status cd_forward_rows(const float* x, const float* y, int B, int N, int M, int q0, int q1, float* d_xy,
                          int32_t* idx_xy, int64_t* colkeys, double* partials, float tau, void* workspace,
                          size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!x || !y || !workspace || !colkeys) return fail(CD_ERR_INVALID_VALUE, "null x, y, colkeys or workspace");
    if (q0 < 0 || q1 < q0 || q1 > N) return fail(CD_ERR_INVALID_VALUE, "bad row slice [%d,%d) of N=%d", q0, q1, N);
    if (q1 > q0 && (!d_xy || !idx_xy)) return fail(CD_ERR_INVALID_VALUE, "null d_xy / idx_xy");
    if (tau != tau) return fail(CD_ERR_INVALID_VALUE, "tau is NaN");
    if (!aligned(x, 4) || !aligned(y, 4) || !aligned(colkeys, 8))
        return fail(CD_ERR_MISALIGNED, "cloud pointers must be 4-byte and colkeys 8-byte aligned");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    cdk::FwdPlan p;
    cdk::plan_forward(p, cdk::kFusedRows, B, N, M, q0, q1, 0, 0, g_forced_splits);
    if (workspace_bytes < p.bytes)
        return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu bytes", workspace_bytes, p.bytes);
    s = check_device();
    if (s != CD_OK) return s;
    cdk::FwdOutputs o;
    o.d[0] = d_xy;
    o.d[1] = nullptr;
    o.idx[0] = idx_xy;
    o.idx[1] = nullptr;
    o.partials = partials;
    o.tau = tau;
    o.colkey = reinterpret_cast<long long*>(colkeys);
    return cuda_status(cdk::launch_forward(p, x, y, o, workspace, static_cast<cudaStream_t>(stream)),
                       "cd_forward_rows");
}

cd_status cd_forward_cols(const float* x, const float* y, int B, int N, int M, const int64_t* colkeys, int r0,
                          int r1, float* d_yx, int32_t* idx_yx, double* partials, float tau, void* workspace,
                          size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!x || !y || !workspace || !colkeys) return fail(CD_ERR_INVALID_VALUE, "null x, y, colkeys or workspace");
    if (r0 < 0 || r1 < r0 || r1 > M) return fail(CD_ERR_INVALID_VALUE, "bad column slice [%d,%d) of M=%d", r0, r1, M);
    if (r1 > r0 && (!d_yx || !idx_yx)) return fail(CD_ERR_INVALID_VALUE, "null d_yx / idx_yx");
    if (tau != tau) return fail(CD_ERR_INVALID_VALUE, "tau is NaN");
    if (!aligned(x, 4) || !aligned(y, 4) || !aligned(colkeys, 8))
        return fail(CD_ERR_MISALIGNED, "cloud pointers must be 4-byte and colkeys 8-byte aligned");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    cdk::FwdPlan p;
    cdk::plan_forward(p, cdk::kFusedCols, B, N, M, 0, 0, r0, r1, g_forced_splits);
    if (workspace_bytes < p.bytes)
        return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu bytes", workspace_bytes, p.bytes);
    s = check_device();
    if (s != CD_OK) return s;
    cdk::FwdOutputs o;
    o.d[0] = nullptr;
    o.d[1] = d_yx;
    o.idx[0] = nullptr;
    o.idx[1] = idx_yx;
    o.partials = partials;
    o.tau = tau;
    o.colkey = const_cast<long long*>(reinterpret_cast<const long long*>(colkeys));
    return cuda_status(cdk::launch_forward(p, x, y, o, workspace, static_cast<cudaStream_t>(stream)),
                       "cd_forward_cols");
}

cd_status cd_forward_cols_peers(const float* x, const float* y, int B, int N, int M, const int64_t* const* colkeys,
                                int npeers, int r0, int r1, float* d_yx, int32_t* idx_yx, double* partials,
                                float tau, void* workspace, size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!x || !y || !workspace || !colkeys) return fail(CD_ERR_INVALID_VALUE, "null x, y, colkeys or workspace");
    if (npeers < 1 || npeers > CD_MAX_PEERS)
        return fail(CD_ERR_INVALID_VALUE, "npeers must be in [1, %d] (got %d)", CD_MAX_PEERS, npeers);
    for (int q = 0; q < npeers; ++q) {
        if (!colkeys[q]) return fail(CD_ERR_INVALID_VALUE, "colkeys[%d] is null", q);
        if (!aligned(colkeys[q], 8)) return fail(CD_ERR_MISALIGNED, "colkeys[%d] must be 8-byte aligned", q);
    }
    if (r0 < 0 || r1 < r0 || r1 > M) return fail(CD_ERR_INVALID_VALUE, "bad column slice [%d,%d) of M=%d", r0, r1, M);
    if (r1 > r0 && (!d_yx || !idx_yx)) return fail(CD_ERR_INVALID_VALUE, "null d_yx / idx_yx");
    if (tau != tau) return fail(CD_ERR_INVALID_VALUE, "tau is NaN");
    if (!aligned(x, 4) || !aligned(y, 4)) return fail(CD_ERR_MISALIGNED, "cloud pointers must be 4-byte aligned");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    cdk::FwdPlan p;
    cdk::plan_forward(p, cdk::kFusedCols, B, N, M, 0, 0, r0, r1, g_forced_splits);
    if (workspace_bytes < p.bytes)
        return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu bytes", workspace_bytes, p.bytes);
    s = check_device();
    if (s != CD_OK) return s;
    cdk::FwdOutputs o;
    o.d[0] = nullptr;
    o.d[1] = d_yx;
    o.idx[0] = nullptr;
    o.idx[1] = idx_yx;
    o.partials = partials;
    o.tau = tau;
    o.colkey = const_cast<long long*>(reinterpret_cast<const long long*>(colkeys[0]));
    o.npeers = npeers;
    for (int q = 0; q < npeers; ++q) o.colkey_peers[q] = reinterpret_cast<const long long*>(colkeys[q]);
    return cuda_status(cdk::launch_forward(p, x, y, o, workspace, static_cast<cudaStream_t>(stream)),
                       "cd_forward_cols_peers");
}

cd_status cd_forward_pruned(const float* x, const float* y, int B, int N, int M, float* d_xy, int32_t* idx_xy,
                            float* d_yx, int32_t* idx_yx, double* partials, float tau, void* workspace,
                            size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!x || !y || !workspace || !d_xy || !idx_xy || !d_yx || !idx_yx)
        return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (tau != tau) return fail(CD_ERR_INVALID_VALUE, "tau is NaN");
    if (!aligned(x, 4) || !aligned(y, 4)) return fail(CD_ERR_MISALIGNED, "cloud pointers must be 4-byte aligned");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    cdk::PrunedPlan p;
    cdk::plan_pruned(p, B, N, M);
    if (!p.supported) return fail(CD_ERR_TOO_LARGE, "pruned path supports at most 8192 tiles (4,194,304 points) per cloud");
    if (workspace_bytes < p.bytes)
        return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu bytes", workspace_bytes, p.bytes);
    s = check_device();
    if (s != CD_OK) return s;
    cdk::FwdOutputs o;
    o.d[0] = d_xy;
    o.d[1] = d_yx;
    o.idx[0] = idx_xy;
    o.idx[1] = idx_yx;
    o.partials = partials;
    o.tau = tau;
    o.colkey = nullptr;
    return cuda_status(cdk::launch_pruned(p, x, y, o, workspace, static_cast<cudaStream_t>(stream)),
                       "cd_forward_pruned");
}

cd_status cd_sample_mesh(const float* verts, const int32_t* faces, int B, int Nv, int Nf, int N,
                         const uint32_t* r_face, const float* r_bary, float* points, int32_t* face_idx, float* bary,
                         void* workspace, size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    if (B < 1 || Nv < 3 || Nf < 1 || N < 1)
        return fail(CD_ERR_INVALID_VALUE, "need B >= 1, Nv >= 3, Nf >= 1, N >= 1 (got %d %d %d %d)", B, Nv, Nf, N);
    if ((long long)B * N * 3 > 0x7fffffffLL || (long long)B * Nv > 0x7fffffffLL)
        return fail(CD_ERR_TOO_LARGE, "B*N*3 or B*Nv exceeds 2^31-1");
    if (B > kMaxBatch) return fail(CD_ERR_TOO_LARGE, "B = %d exceeds %d (one grid row per batch element)", B, kMaxBatch);
    if (!verts || !faces || !r_face || !r_bary || !points || !face_idx || !workspace)
        return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    const size_t need = cdk::sample_workspace(B, Nv, Nf, N);
    if (workspace_bytes < need) return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu", workspace_bytes, need);
    cd_status s = check_device();
    if (s != CD_OK) return s;
    return cuda_status(cdk::launch_sample(verts, faces, B, Nv, Nf, N, r_face, r_bary, points, face_idx, bary, workspace,
                                          static_cast<cudaStream_t>(stream)),
                       "cd_sample_mesh");
}

cd_status cd_sample_mesh_backward(const int32_t* faces, const int32_t* face_idx, const float* bary, int B, int Nv,
                                  int Nf, int N, const float* grad_points, float* grad_verts, void* workspace,
                                  size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    if (B < 1 || Nv < 3 || Nf < 1 || N < 1)
        return fail(CD_ERR_INVALID_VALUE, "need B >= 1, Nv >= 3, Nf >= 1, N >= 1 (got %d %d %d %d)", B, Nv, Nf, N);
    if ((long long)B * N * 3 > 0x7fffffffLL || (long long)B * Nv > 0x7fffffffLL)
        return fail(CD_ERR_TOO_LARGE, "B*N*3 or B*Nv exceeds 2^31-1");
    if (!faces || !face_idx || !bary || !grad_points || !grad_verts || !workspace)
        return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    const size_t need = cdk::sample_backward_workspace(B, Nv, Nf, N);
    if (workspace_bytes < need) return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu", workspace_bytes, need);
    cd_status s = check_device();
    if (s != CD_OK) return s;
    return cuda_status(cdk::launch_sample_backward(faces, face_idx, bary, B, Nv, Nf, N, grad_points, grad_verts,
                                                   workspace, static_cast<cudaStream_t>(stream)),
                       "cd_sample_mesh_backward");
}

size_t cd_sample_workspace_size(int op, int B, int Nv, int Nf, int N) {
    if (B < 1 || Nv < 3 || Nf < 1 || N < 1) return 0;
    if (op == CD_OP_SAMPLE) return cdk::sample_workspace(B, Nv, Nf, N);
    if (op == CD_OP_SAMPLE_BACKWARD) return cdk::sample_backward_workspace(B, Nv, Nf, N);
    return 0;
}

int cd_sample_launch_count(int op, int B, int Nv, int Nf, int N) {
    if (B < 1 || Nv < 3 || Nf < 1 || N < 1) return 0;
    if (op == CD_OP_SAMPLE) return 3;
    if (op == CD_OP_SAMPLE_BACKWARD) return cdk::sample_backward_launches(B, Nv, Nf, N);
    return 0;
}

static cd_status check_p2s_sizes(int B, int N, int Nv, int Nf) {
    if (B < 1 || N < 1 || Nv < 3 || Nf < 1)
        return fail(CD_ERR_INVALID_VALUE, "need B, N, Nf >= 1 and Nv >= 3 (got %d %d %d %d)", B, N, Nv, Nf);
    if ((long long)B * N * 3 > 0x7fffffffLL || (long long)B * Nv > 0x7fffffffLL || (long long)B * Nf * 24 > 0x7fffffffLL)
        return fail(CD_ERR_TOO_LARGE, "problem too large for 32-bit indexing");
    if (B > kMaxBatch) return fail(CD_ERR_TOO_LARGE, "B = %d exceeds %d (one grid row per batch element)", B, kMaxBatch);
    return CD_OK;
}

cd_status cd_p2s_forward(const float* points, const float* verts, const int32_t* faces, int B, int N, int Nv, int Nf,
                         float* d, int32_t* face, float* closest, float* bary, float* per_batch, float* loss,
                         void* workspace, size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_p2s_sizes(B, N, Nv, Nf);
    if (s != CD_OK) return s;
    if (!points || !verts || !faces || !d || !face || !workspace) return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    const size_t need = cdk::p2s_workspace(B, N, Nv, Nf);
    if (workspace_bytes < need) return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu", workspace_bytes, need);
    s = check_device();
    if (s != CD_OK) return s;
    return cuda_status(cdk::launch_p2s(points, verts, faces, B, N, Nv, Nf, d, face, closest, bary, per_batch, loss,
                                       workspace, static_cast<cudaStream_t>(stream)),
                       "cd_p2s_forward");
}

static cd_status p2s_backward_common(const char* who, const float* points, const float* closest,
                                     const int32_t* face, const float* bary, const int32_t* faces, int B, int N,
                                     int Nv, int Nf, const float* g, float g_scalar, const float* upstream,
                                     float* grad_points, float* grad_verts, void* workspace, size_t workspace_bytes,
                                     cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_p2s_sizes(B, N, Nv, Nf);
    if (s != CD_OK) return s;
    if (!points || !closest || !face || !faces || !workspace || (grad_verts && !bary))
        return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    const size_t need = cdk::p2s_backward_workspace(B, N, Nv, Nf);
    if (workspace_bytes < need) return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu", workspace_bytes, need);
    s = check_device();
    if (s != CD_OK) return s;
    return cuda_status(cdk::launch_p2s_backward(points, closest, face, bary, faces, B, N, Nv, Nf, g, g_scalar, upstream,
                                                grad_points, grad_verts, workspace, static_cast<cudaStream_t>(stream)),
                       who);
}

cd_status cd_p2s_backward(const float* points, const float* closest, const int32_t* face, const float* bary,
                          const int32_t* faces, int B, int N, int Nv, int Nf, const float* g, float g_scalar,
                          float* grad_points, float* grad_verts, void* workspace, size_t workspace_bytes,
                          cd_stream_t stream) {
    return p2s_backward_common("cd_p2s_backward", points, closest, face, bary, faces, B, N, Nv, Nf, g, g_scalar,
                               nullptr, grad_points, grad_verts, workspace, workspace_bytes, stream);
}

cd_status cd_p2s_loss_backward(const float* points, const float* closest, const int32_t* face, const float* bary,
                               const int32_t* faces, int B, int N, int Nv, int Nf, const float* grad_loss,
                               float* grad_points, float* grad_verts, void* workspace, size_t workspace_bytes,
                               cd_stream_t stream) {
    if (!grad_loss || B < 1 || N < 1) {
        g_err.clear();
        return fail(CD_ERR_INVALID_VALUE, "null grad_loss or empty point set");
    }
    return p2s_backward_common("cd_p2s_loss_backward", points, closest, face, bary, faces, B, N, Nv, Nf, nullptr,
                               loss_fill(1.0f, B, N), grad_loss, grad_points, grad_verts, workspace, workspace_bytes,
                               stream);
}

size_t cd_p2s_workspace_size(int op, int B, int N, int Nv, int Nf) {
    if (B < 1 || N < 1 || Nv < 3 || Nf < 1) return 0;
    if (op == CD_OP_P2S) return cdk::p2s_workspace(B, N, Nv, Nf);
    if (op == CD_OP_P2S_BACKWARD) return cdk::p2s_backward_workspace(B, N, Nv, Nf);
    if (op == CD_OP_P2S_PRUNED) return cdk::p2s_pruned_workspace(B, N, Nv, Nf);
    return 0;
}

int cd_p2s_launch_count(int op, int B, int N, int Nv, int Nf) {
    if (B < 1 || N < 1 || Nv < 3 || Nf < 1) return 0;
    if (op == CD_OP_P2S) return cdk::p2s_launches();
    if (op == CD_OP_P2S_BACKWARD) return 1 + cdk::sample_backward_launches(B, Nv, Nf, N);
    if (op == CD_OP_P2S_PRUNED) return cdk::p2s_pruned_workspace(B, N, Nv, Nf) ? cdk::p2s_pruned_launches(B, N, Nv, Nf) : 0;
    return 0;
}

cd_status cd_p2s_forward_pruned(const float* points, const float* verts, const int32_t* faces, int B, int N, int Nv,
                                int Nf, float* d, int32_t* face, float* closest, float* bary, float* per_batch,
                                float* loss, void* workspace, size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_p2s_sizes(B, N, Nv, Nf);
    if (s != CD_OK) return s;
    if (!points || !verts || !faces || !d || !face || !workspace) return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    const size_t need = cdk::p2s_pruned_workspace(B, N, Nv, Nf);
    if (need == 0) return fail(CD_ERR_TOO_LARGE, "pruned point-to-surface: unsupported size (Nf %d, B %d, N %d)", Nf, B, N);
    if (workspace_bytes < need) return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu", workspace_bytes, need);
    s = check_device();
    if (s != CD_OK) return s;
    return cuda_status(cdk::launch_p2s_pruned(points, verts, faces, B, N, Nv, Nf, d, face, closest, bary, per_batch,
                                              loss, workspace, static_cast<cudaStream_t>(stream)),
                       "cd_p2s_forward_pruned");
}

int cd_set_forward_mode(int mode) {
    int old = g_forward_mode;
    g_forward_mode = (mode >= 1 && mode <= 3) ? mode : 0;
    return old;
}

cd_status cd_finalize(const double* partials, int B, int N, int M, float w1, float w2, float* cd_per_batch,
                      float* loss, float* fscore, float* precision, float* recall, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!partials || !loss) return fail(CD_ERR_INVALID_VALUE, "null partials or loss pointer");
    s = check_device();
    if (s != CD_OK) return s;
    return cuda_status(cdk::launch_finalize(partials, B, N, M, w1, w2, cd_per_batch, loss, fscore, precision, recall,
                                            static_cast<cudaStream_t>(stream)),
                       "cd_finalize");
}

cd_status cd_fscore(const float* d_xy, const float* d_yx, int B, int N, int M, float tau, float* fscore,
                    float* precision, float* recall, void* workspace, size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!d_xy || !d_yx || !fscore || !workspace) return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (!(tau >= 0.f)) return fail(CD_ERR_INVALID_VALUE, "tau must be >= 0 (got %g)", (double)tau);
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    const size_t need = cdk::fscore_workspace(B, N, M);
    if (workspace_bytes < need) return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu", workspace_bytes, need);
    s = check_device();
    if (s != CD_OK) return s;
    return cuda_status(cdk::launch_fscore(d_xy, d_yx, B, N, M, tau, fscore, precision, recall, workspace,
                                          static_cast<cudaStream_t>(stream)),
                       "cd_fscore");
}

static cd_status backward_common(const char* who, const float* x, const float* y, int B, int N, int M,
                                 const int32_t* idx_xy, const int32_t* idx_yx, const float* g, const float* h,
                                 float g_scalar, float h_scalar, const float* upstream, int q0, int q1, int r0, int r1,
                                 float* grad_x, float* grad_y, void* workspace, size_t workspace_bytes,
                                 cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!x || !y || !idx_xy || !idx_yx || !workspace) return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (q0 < 0 || q1 < q0 || q1 > N || r0 < 0 || r1 < r0 || r1 > M)
        return fail(CD_ERR_INVALID_VALUE, "bad slices [%d,%d) of N=%d, [%d,%d) of M=%d", q0, q1, N, r0, r1, M);
    if (q1 > q0 && !grad_x) return fail(CD_ERR_INVALID_VALUE, "null grad_x");
    if (r1 > r0 && !grad_y) return fail(CD_ERR_INVALID_VALUE, "null grad_y");
    if (!aligned(x, 4) || !aligned(y, 4)) return fail(CD_ERR_MISALIGNED, "cloud pointers must be 4-byte aligned");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    cdk::BwdPlan p;
    cdk::plan_backward(p, B, N, M, q0, q1, r0, r1);
    if (workspace_bytes < p.bytes)
        return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu bytes", workspace_bytes, p.bytes);
    s = check_device();
    if (s != CD_OK) return s;
    return cuda_status(cdk::launch_backward(p, x, y, idx_xy, idx_yx, g, h, g_scalar, h_scalar, upstream, grad_x,
                                            grad_y, workspace, static_cast<cudaStream_t>(stream)),
                       who);
}

cd_status cd_backward(const float* x, const float* y, int B, int N, int M, const int32_t* idx_xy,
                      const int32_t* idx_yx, const float* g, const float* h, float g_scalar, float h_scalar, int q0,
                      int q1, int r0, int r1, float* grad_x, float* grad_y, void* workspace, size_t workspace_bytes,
                      cd_stream_t stream) {
    return backward_common("cd_backward", x, y, B, N, M, idx_xy, idx_yx, g, h, g_scalar, h_scalar, nullptr, q0, q1,
                           r0, r1, grad_x, grad_y, workspace, workspace_bytes, stream);
}

cd_status cd_loss_backward(const float* x, const float* y, int B, int N, int M, const int32_t* idx_xy,
                           const int32_t* idx_yx, const float* grad_loss, float w1, float w2, int q0, int q1, int r0,
                           int r1, float* grad_x, float* grad_y, void* workspace, size_t workspace_bytes,
                           cd_stream_t stream) {
    if (!grad_loss) {
        g_err.clear();
        return fail(CD_ERR_INVALID_VALUE, "null grad_loss");
    }
    if (B < 1 || N < 1 || M < 1) {
        g_err.clear();
        return fail(CD_ERR_INVALID_VALUE, "empty cloud: B=%d N=%d M=%d", B, N, M);
    }
    return backward_common("cd_loss_backward", x, y, B, N, M, idx_xy, idx_yx, nullptr, nullptr, loss_fill(w1, B, N),
                           loss_fill(w2, B, M), grad_loss, q0, q1, r0, r1, grad_x, grad_y, workspace, workspace_bytes,
                           stream);
}

cd_status cd_step_host(const float* x_host, const float* y_host, int B, int N, int M, float tau, float w1, float w2,
                       float* loss_host, float* fscore_host, float* grad_x_host, float* grad_y_host, void* workspace,
                       size_t workspace_bytes, cd_stream_t stream) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!x_host || !y_host || !loss_host || !workspace) return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    const StepLayout L = step_layout(B, N, M);
    if (workspace_bytes < L.bytes)
        return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu bytes", workspace_bytes, L.bytes);
    s = check_device();
    if (s != CD_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* w = static_cast<char*>(workspace);
    float* x = reinterpret_cast<float*>(w + L.x);
    float* y = reinterpret_cast<float*>(w + L.y);
    cudaError_t e = cudaMemcpyAsync(x, x_host, (size_t)B * N * 12, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(y, y_host, (size_t)B * M * 12, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_status(e, "cd_step_host H2D");
    float* dxy = reinterpret_cast<float*>(w + L.dxy);
    int32_t* ixy = reinterpret_cast<int32_t*>(w + L.ixy);
    float* dyx = reinterpret_cast<float*>(w + L.dyx);
    int32_t* iyx = reinterpret_cast<int32_t*>(w + L.iyx);
    double* part = reinterpret_cast<double*>(w + L.part);
    float* loss = reinterpret_cast<float*>(w + L.loss);
    float* fs = reinterpret_cast<float*>(w + L.fs);
    float* gx = reinterpret_cast<float*>(w + L.gx);
    float* gy = reinterpret_cast<float*>(w + L.gy);
    void* inner = w + L.inner;
    s = cd_forward(x, y, B, N, M, 0, N, 0, M, dxy, ixy, dyx, iyx, part, tau, inner, L.inner_bytes, stream);
    if (s != CD_OK) return s;
    s = cd_finalize(part, B, N, M, w1, w2, nullptr, loss, tau >= 0.f ? fs : nullptr, nullptr, nullptr, stream);
    if (s != CD_OK) return s;
    const float gs = loss_fill(w1, B, N);
    const float hs = loss_fill(w2, B, M);
    s = cd_backward(x, y, B, N, M, ixy, iyx, nullptr, nullptr, gs, hs, 0, N, 0, M, gx, gy, inner, L.inner_bytes,
                    stream);
    if (s != CD_OK) return s;
    e = cudaMemcpyAsync(loss_host, loss, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && fscore_host && tau >= 0.f)
        e = cudaMemcpyAsync(fscore_host, fs, (size_t)B * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && grad_x_host)
        e = cudaMemcpyAsync(grad_x_host, gx, (size_t)B * N * 12, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && grad_y_host)
        e = cudaMemcpyAsync(grad_y_host, gy, (size_t)B * M * 12, cudaMemcpyDeviceToHost, st);
    return cuda_status(e, "cd_step_host D2H");
}

#ifndef CD_STEP_FIRST_DIV
#define CD_STEP_FIRST_DIV 2
#endif
cd_status cd_step_host_overlapped(const float* x_host, const float* y_host, int B, int N, int M, float tau, float w1,
                                  float w2, float* loss_host, float* fscore_host, float* grad_x_host,
                                  float* grad_y_host, int nchunks, void* workspace, size_t workspace_bytes,
                                  cd_stream_t stream, cd_stream_t copy_stream, cd_stream_t stream2,
                                  void* const* events) {
    g_err.clear();
    cd_status s = check_sizes(B, N, M);
    if (s != CD_OK) return s;
    if (!x_host || !y_host || !loss_host || !workspace || !events || !copy_stream)
        return fail(CD_ERR_INVALID_VALUE, "null pointer argument");
    if (nchunks < 1 || nchunks > B) return fail(CD_ERR_INVALID_VALUE, "nchunks must be in [1, B] (got %d)", nchunks);
    for (int c = 0; c <= nchunks; ++c)
        if (!events[c]) return fail(CD_ERR_INVALID_VALUE, "events[%d] is null", c);
    if (!aligned(workspace, 256)) return fail(CD_ERR_MISALIGNED, "workspace must be 256-byte aligned");
    const StepLayout L = step_layout(B, N, M);
    if (workspace_bytes < L.bytes)
        return fail(CD_ERR_TOO_LARGE, "workspace too small: %zu < %zu bytes", workspace_bytes, L.bytes);
    s = check_device();
    if (s != CD_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaStream_t cs = static_cast<cudaStream_t>(copy_stream);
    // ranges alternate between `stream` and `stream2` (when given): a range's fused forward then fills
    // the SMs the previous range's last wave leaves idle (measured on c3's [4, 12, 12, 4] ranges:
    // 2.124 ms on one stream, 2.047 ms alternating, 1.994 ms unchunked; tools/time_chunk_streams.py)
    const bool two = stream2 != nullptr && nchunks > 1;
    cudaStream_t sc2 = two ? static_cast<cudaStream_t>(stream2) : st;
    char* w = static_cast<char*>(workspace);
    float* x = reinterpret_cast<float*>(w + L.x);
    float* y = reinterpret_cast<float*>(w + L.y);
    float* dxy = reinterpret_cast<float*>(w + L.dxy);
    int32_t* ixy = reinterpret_cast<int32_t*>(w + L.ixy);
    float* dyx = reinterpret_cast<float*>(w + L.dyx);
    int32_t* iyx = reinterpret_cast<int32_t*>(w + L.iyx);
    double* part = reinterpret_cast<double*>(w + L.part);
    float* loss = reinterpret_cast<float*>(w + L.loss);
    float* fs = reinterpret_cast<float*>(w + L.fs);
    float* gx = reinterpret_cast<float*>(w + L.gx);
    float* gy = reinterpret_cast<float*>(w + L.gy);
    cudaEvent_t done = static_cast<cudaEvent_t>(events[nchunks]);
    // batch ranges: the first range is 1/CD_STEP_FIRST_DIV of an equal share (its copy is the only
    // exposed one); with 3 or more ranges the last one is as short as the first (only its backward
    // and gradient copy are exposed); the rest split equally
    auto bound = [&](int c) -> int {
        if (c <= 0) return 0;
        if (c >= nchunks) return B;
        const int first = std::max(1, (int)((int64_t)B / ((int64_t)nchunks * CD_STEP_FIRST_DIV)));
        const int last = nchunks >= 3 ? first : 0;
        const int mid = nchunks - 1 - (last > 0 ? 1 : 0);
        if (c == nchunks - 1 && last > 0) return B - last;
        return first + (int)((int64_t)(B - first - last) * (c - 1) / mid);
    };
    // fork: the copy stream (and the second compute stream) start after everything already queued on
    // `stream` (so the staging buffers of the previous step are free); the same pattern makes the call
    // capturable in a CUDA graph (both join `stream` again below)
    cudaError_t e = cudaEventRecord(done, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, done, 0);
    if (e == cudaSuccess && two) e = cudaStreamWaitEvent(sc2, done, 0);
    for (int c = 0; c < nchunks && e == cudaSuccess; ++c) {
        const int b0 = bound(c), b1 = bound(c + 1);
        e = cudaMemcpyAsync(x + (size_t)b0 * N * 3, x_host + (size_t)b0 * N * 3, (size_t)(b1 - b0) * N * 12,
                            cudaMemcpyHostToDevice, cs);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(y + (size_t)b0 * M * 3, y_host + (size_t)b0 * M * 3, (size_t)(b1 - b0) * M * 12,
                                cudaMemcpyHostToDevice, cs);
        if (e == cudaSuccess) e = cudaEventRecord(static_cast<cudaEvent_t>(events[c]), cs);
    }
    if (e != cudaSuccess) return cuda_status(e, "cd_step_host_overlapped H2D");
    // range c's forward starts as soon as its clouds have landed (later ranges copy meanwhile), and its
    // backward follows at once: the loss gradient's fills w/(B P) do not depend on the loss value, and
    // every batch element's gradient depends only on its own clouds and indices.  Range c's gradients
    // then return on the copy stream while the next range computes.
    const float gs = loss_fill(w1, B, N);
    const float hs = loss_fill(w2, B, M);
    for (int c = 0; c < nchunks; ++c) {
        const int b0 = bound(c), b1 = bound(c + 1);
        cudaStream_t sc = (c & 1) ? sc2 : st;
        void* inner = w + ((c & 1) && two ? L.inner2 : L.inner);
        cudaEvent_t ev = static_cast<cudaEvent_t>(events[c]);
        e = cudaStreamWaitEvent(sc, ev, 0);
        if (e != cudaSuccess) return cuda_status(e, "cd_step_host_overlapped wait");
        float* xr = x + (size_t)b0 * N * 3;
        float* yr = y + (size_t)b0 * M * 3;
        s = cd_forward(xr, yr, b1 - b0, N, M, 0, N, 0, M, dxy + (size_t)b0 * N, ixy + (size_t)b0 * N,
                       dyx + (size_t)b0 * M, iyx + (size_t)b0 * M, part + 4 * (size_t)b0, tau, inner, L.inner_bytes,
                       sc);
        if (s != CD_OK) return s;
        s = cd_backward(xr, yr, b1 - b0, N, M, ixy + (size_t)b0 * N, iyx + (size_t)b0 * M, nullptr, nullptr, gs, hs,
                        0, N, 0, M, gx + (size_t)b0 * N * 3, gy + (size_t)b0 * M * 3, inner, L.inner_bytes, sc);
        if (s != CD_OK) return s;
        if (grad_x_host || grad_y_host) {
            // the wait above already captured ev's H2D record, so it can be re-recorded here
            e = cudaEventRecord(ev, sc);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev, 0);
            if (e == cudaSuccess && grad_x_host)
                e = cudaMemcpyAsync(grad_x_host + (size_t)b0 * N * 3, gx + (size_t)b0 * N * 3,
                                    (size_t)(b1 - b0) * N * 12, cudaMemcpyDeviceToHost, cs);
            if (e == cudaSuccess && grad_y_host)
                e = cudaMemcpyAsync(grad_y_host + (size_t)b0 * M * 3, gy + (size_t)b0 * M * 3,
                                    (size_t)(b1 - b0) * M * 12, cudaMemcpyDeviceToHost, cs);
            if (e != cudaSuccess) return cuda_status(e, "cd_step_host_overlapped gradient D2H");
        }
    }
    if (two) {
        // join the second compute stream (all its waits above were enqueued before this re-record)
        e = cudaEventRecord(static_cast<cudaEvent_t>(events[1]), sc2);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(events[1]), 0);
        if (e != cudaSuccess) return cuda_status(e, "cd_step_host_overlapped join");
    }
    s = cd_finalize(part, B, N, M, w1, w2, nullptr, loss, tau >= 0.f ? fs : nullptr, nullptr, nullptr, stream);
    if (s != CD_OK) return s;
    e = cudaMemcpyAsync(loss_host, loss, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && fscore_host && tau >= 0.f)
        e = cudaMemcpyAsync(fscore_host, fs, (size_t)B * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) {
        // `stream` completes only after the copy stream's work (the caller synchronises `stream`)
        e = cudaEventRecord(static_cast<cudaEvent_t>(events[0]), cs);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(events[0]), 0);
    }
    if (e == cudaSuccess) e = cudaEventRecord(done, st);
    return cuda_status(e, "cd_step_host_overlapped D2H");
}

}  // extern "C"
