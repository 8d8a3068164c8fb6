// mesh_sample.cu — differentiable mesh surface sampling, the step before the Chamfer path
// ("differentiable surface sampling ... by
// application of the reparameterization trick").  Readings R19-R22:
//
//   mesh_area_kernel    fp64 face areas (fixed op order, no contraction) on every SM, per-CTA max.
//   mesh_cdf_kernel     one CTA per batch element: areas quantised to integers q_f = floor(area_f * 2^k)
//                       with k = 52 - e, Nf * max area = m 2^e; exact uint64 inclusive prefix
//                       (order-free integers), so the face choice is the same integer decision on
//                       every implementation.
//   mesh_sample_kernel  per sample: t = (r_face * S) >> 32 exactly, face = upper_bound(prefix, t),
//                       square-root barycentrics and the point, fp32 .rn ops.
//   backward            keys (b*Nv + corner vertex) for every (sample, corner), the stable radix sort
//                       of nn_backward.cu, segment offsets, one thread per vertex accumulating
//                       w * g in fp64 in ascending (sample, corner) order: deterministic, no atomics.
#include "cd_device.cuh"
#include "cd_internal.h"

#include <algorithm>

namespace cdk {

constexpr int kCdfThreads = 512;

__device__ __forceinline__ double face_area64(const float* v, int fa, int fb, int fc) {
    const float* a = v + 3 * (int64_t)fa;
    const float* b = v + 3 * (int64_t)fb;
    const float* c = v + 3 * (int64_t)fc;
    const double e1x = __dsub_rn(b[0], a[0]), e1y = __dsub_rn(b[1], a[1]), e1z = __dsub_rn(b[2], a[2]);
    const double e2x = __dsub_rn(c[0], a[0]), e2y = __dsub_rn(c[1], a[1]), e2z = __dsub_rn(c[2], a[2]);
    const double cx = __dsub_rn(__dmul_rn(e1y, e2z), __dmul_rn(e1z, e2y));
    const double cy = __dsub_rn(__dmul_rn(e1z, e2x), __dmul_rn(e1x, e2z));
    const double cz = __dsub_rn(__dmul_rn(e1x, e2y), __dmul_rn(e1y, e2x));
    return __dmul_rn(0.5, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz))));
}

struct CdfArgs {
    const float* verts;   // [B][Nv][3]
    const int* faces;     // [Nf][3]
    int Nv, Nf, nblk;
    double* areas;        // [B][Nf] scratch
    double* blkmax;       // [B][nblk] scratch
    unsigned long long* cdf;  // [B][Nf] inclusive prefix of the quantised areas
};

constexpr int kAreaThreads = 256;

// (1) fp64 areas of every face (all SMs), per-CTA maximum (fixed-order, no atomics)
__global__ void __launch_bounds__(kAreaThreads) mesh_area_kernel(CdfArgs a) {
    const int b = blockIdx.y;
    const float* v = a.verts + (int64_t)b * a.Nv * 3;
    const int f = blockIdx.x * kAreaThreads + threadIdx.x;
    double ar = 0.0;
    if (f < a.Nf) {
        const int ia = min(max(a.faces[3 * f], 0), a.Nv - 1), ib = min(max(a.faces[3 * f + 1], 0), a.Nv - 1),
                  ic = min(max(a.faces[3 * f + 2], 0), a.Nv - 1);
        ar = face_area64(v, ia, ib, ic);
        a.areas[(int64_t)b * a.Nf + f] = ar;
    }
    __shared__ double sm[kAreaThreads / 32];
    double m = ar;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = 0.0;
        for (int w = 0; w < kAreaThreads / 32; ++w) mm = fmax(mm, sm[w]);
        a.blkmax[(int64_t)b * a.nblk + blockIdx.x] = mm;
    }
}

// (2) one CTA per batch element: max -> exponent, quantise, exact uint64 inclusive prefix
// (each thread a contiguous run of faces, one block scan of the run totals)
__global__ void __launch_bounds__(kCdfThreads) mesh_cdf_kernel(CdfArgs a) {
    const int b = blockIdx.x;
    __shared__ double smax[kCdfThreads / 32];
    __shared__ unsigned long long wtot[kCdfThreads / 32];
    __shared__ int s_e;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double m = 0.0;
    for (int i = threadIdx.x; i < a.nblk; i += kCdfThreads) m = fmax(m, a.blkmax[(int64_t)b * a.nblk + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) smax[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = 0.0;
        for (int w = 0; w < kCdfThreads / 32; ++w) mm = fmax(mm, smax[w]);
        int e = 0;
        if (mm > 0.0) frexp(__dmul_rn(mm, (double)a.Nf), &e);
        s_e = mm > 0.0 ? e : 1000;   // 1000: every area is 0 -> all q_f = 0
    }
    __syncthreads();
    const int e = s_e;
    const double* ar = a.areas + (int64_t)b * a.Nf;
    const int per = (a.Nf + kCdfThreads - 1) / kCdfThreads;
    const int f0 = threadIdx.x * per, f1 = min(f0 + per, a.Nf);
    auto quant = [&](int f) -> unsigned long long {
        return e == 1000 ? 0ull : (unsigned long long)ldexp(ar[f], 52 - e);  // exact scaling, floor
    };
    unsigned long long loc = 0;
    for (int f = f0; f < f1; ++f) loc += quant(f);
    unsigned long long incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    unsigned long long run = incl - loc;
    for (int w = 0; w < warp; ++w) run += wtot[w];
    unsigned long long* out = a.cdf + (int64_t)b * a.Nf;
    for (int f = f0; f < f1; ++f) {
        run += quant(f);
        out[f] = run;
    }
}

struct SampleArgs {
    const float* verts;
    const int* faces;
    int B, Nv, Nf, N;
    const unsigned long long* cdf;
    const unsigned* r_face;   // [B][N]
    const float* r_bary;      // [B][N][2]
    float* points;            // [B][N][3]
    int* face_idx;            // [B][N]
    float* bary;              // [B][N][3] (may be null)
};

__global__ void __launch_bounds__(256) mesh_sample_kernel(SampleArgs a) {
    const int64_t total = (int64_t)a.B * a.N;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < total; s += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(s / a.N);
        const unsigned long long* P = a.cdf + (int64_t)b * a.Nf;
        const unsigned long long S = P[a.Nf - 1];
        int face = 0;
        if (S > 0) {
            const unsigned long long r = a.r_face[s];
            const unsigned long long t = (S >> 32) * r + (((S & 0xffffffffull) * r) >> 32);  // (r * S) >> 32
            int lo = 0, hi = a.Nf - 1;   // smallest f with P[f] > t (P[Nf-1] = S > t always)
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (P[mid] > t) hi = mid;
                else lo = mid + 1;
            }
            face = lo;
        }
        const float r1 = a.r_bary[2 * s], r2 = a.r_bary[2 * s + 1];
        const float sq = __fsqrt_rn(r1);
        const float w0 = __fsub_rn(1.0f, sq), w1 = __fmul_rn(sq, __fsub_rn(1.0f, r2)), w2 = __fmul_rn(sq, r2);
        const float* v = a.verts + (int64_t)b * a.Nv * 3;
        const int ia = min(max(a.faces[3 * face], 0), a.Nv - 1);
        const int ib = min(max(a.faces[3 * face + 1], 0), a.Nv - 1);
        const int ic = min(max(a.faces[3 * face + 2], 0), a.Nv - 1);
#pragma unroll
        for (int c = 0; c < 3; ++c)
            a.points[3 * s + c] = __fadd_rn(__fadd_rn(__fmul_rn(w0, v[3 * ia + c]), __fmul_rn(w1, v[3 * ib + c])),
                                            __fmul_rn(w2, v[3 * ic + c]));
        a.face_idx[s] = face;
        if (a.bary) {
            a.bary[3 * s] = w0;
            a.bary[3 * s + 1] = w1;
            a.bary[3 * s + 2] = w2;
        }
    }
}

// ------------------------------------------------------------------------------------------ backward
__global__ void __launch_bounds__(256) sample_keys_kernel(const int* __restrict__ faces,
                                                          const int* __restrict__ face_idx, int B, int Nv, int Nf,
                                                          int N, uint32_t* __restrict__ keys,
                                                          uint32_t* __restrict__ vals) {
    const int64_t L = (int64_t)B * N * 3;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < L; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / 3;
        const int k = (int)(e - s * 3);
        const int b = (int)(s / N);
        const int f = min(max(face_idx[s], 0), Nf - 1);
        const int v = min(max(faces[3 * f + k], 0), Nv - 1);
        keys[e] = (uint32_t)((int64_t)b * Nv + v);
        vals[e] = (uint32_t)e;   // = sample * 3 + corner: ascending (sample, corner) order
    }
}

__global__ void __launch_bounds__(256) vertex_offsets_kernel(const uint32_t* __restrict__ keys, int64_t L, int64_t kmax,
                                                             uint32_t* __restrict__ off) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= L; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = p == 0 ? 0 : (int64_t)keys[p - 1] + 1;
        const int64_t hi = p == L ? kmax : (int64_t)keys[p];
        for (int64_t k = lo; k <= hi; ++k) off[k] = (uint32_t)p;
    }
}

__global__ void __launch_bounds__(256) vertex_grad_kernel(const uint32_t* __restrict__ vals,
                                                          const uint32_t* __restrict__ off,
                                                          const float* __restrict__ bary,
                                                          const float* __restrict__ grad_points, int64_t nvert,
                                                          float* __restrict__ grad_verts) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvert; v += (int64_t)gridDim.x * blockDim.x) {
        double acc[3] = {0.0, 0.0, 0.0};
        for (uint32_t e = off[v]; e < off[v + 1]; ++e) {
            const uint32_t val = vals[e];
            const uint32_t s = val / 3;
            const double w = (double)bary[val];
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(w, (double)grad_points[3 * (int64_t)s + c]));
        }
        grad_verts[3 * v] = (float)acc[0];
        grad_verts[3 * v + 1] = (float)acc[1];
        grad_verts[3 * v + 2] = (float)acc[2];
    }
}

// ------------------------------------------------------------------------------------------ host
static int ceil_div64(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

static int area_blocks(int Nf) { return (Nf + kAreaThreads - 1) / kAreaThreads; }

size_t sample_workspace(int B, int Nv, int Nf, int N) {
    (void)Nv;
    (void)N;
    return align_up((size_t)B * Nf * 8, 256) * 2 + align_up((size_t)B * area_blocks(Nf) * 8, 256);
}

cudaError_t launch_sample(const float* verts, const int* faces, int B, int Nv, int Nf, int N, const unsigned* r_face,
                          const float* r_bary, float* points, int* face_idx, float* bary, void* ws, cudaStream_t st) {
    char* w = static_cast<char*>(ws);
    unsigned long long* cdf = reinterpret_cast<unsigned long long*>(w);
    CdfArgs c;
    c.verts = verts;
    c.faces = faces;
    c.Nv = Nv;
    c.Nf = Nf;
    c.nblk = area_blocks(Nf);
    c.cdf = cdf;
    c.areas = reinterpret_cast<double*>(w + align_up((size_t)B * Nf * 8, 256));
    c.blkmax = reinterpret_cast<double*>(w + 2 * align_up((size_t)B * Nf * 8, 256));
    mesh_area_kernel<<<dim3(c.nblk, B), kAreaThreads, 0, st>>>(c);
    mesh_cdf_kernel<<<B, kCdfThreads, 0, st>>>(c);
    SampleArgs s;
    s.verts = verts;
    s.faces = faces;
    s.B = B;
    s.Nv = Nv;
    s.Nf = Nf;
    s.N = N;
    s.cdf = cdf;
    s.r_face = r_face;
    s.r_bary = r_bary;
    s.points = points;
    s.face_idx = face_idx;
    s.bary = bary;
    const int64_t total = (int64_t)B * N;
    mesh_sample_kernel<<<std::min(ceil_div64(total, 256), current_sm_count() * 16), 256, 0, st>>>(s);
    return cudaGetLastError();
}

static int key_bits(int64_t kmax) {
    int bits = 0;
    while (bits < 32 && ((int64_t)1 << bits) < kmax) ++bits;
    return std::max(bits, 1);
}

size_t sample_backward_workspace(int B, int Nv, int Nf, int N) {
    (void)Nf;
    const int64_t L = (int64_t)B * N * 3;
    const int64_t kmax = (int64_t)B * Nv;
    size_t off = 0;
    off = align_up(off + (size_t)L * 4 * 4, 256);                          // keys[2], vals[2]
    off = align_up(off + radix_sort_counts_words(L, key_bits(kmax)) * 4, 256);
    off = align_up(off + (size_t)kSortTotalsWords * 4, 256);
    off = align_up(off + (size_t)(kmax + 1) * 4, 256);
    return off;
}

int sample_backward_launches(int B, int Nv, int Nf, int N) {
    (void)Nf;
    return 1 + radix_sort_launches((int64_t)B * N * 3, key_bits((int64_t)B * Nv)) + 2;
}

cudaError_t launch_sample_backward(const int* faces, const int* face_idx, const float* bary, int B, int Nv, int Nf,
                                   int N, const float* grad_points, float* grad_verts, void* ws, cudaStream_t st) {
    const int64_t L = (int64_t)B * N * 3;
    const int64_t kmax = (int64_t)B * Nv;
    char* w = static_cast<char*>(ws);
    uint32_t* keys[2] = {reinterpret_cast<uint32_t*>(w), reinterpret_cast<uint32_t*>(w + L * 4)};
    uint32_t* vals[2] = {reinterpret_cast<uint32_t*>(w + L * 8), reinterpret_cast<uint32_t*>(w + L * 12)};
    size_t off = align_up((size_t)L * 16, 256);
    uint32_t* counts = reinterpret_cast<uint32_t*>(w + off);
    off = align_up(off + radix_sort_counts_words(L, key_bits(kmax)) * 4, 256);
    uint32_t* totals = reinterpret_cast<uint32_t*>(w + off);
    off = align_up(off + (size_t)kSortTotalsWords * 4, 256);
    uint32_t* voff = reinterpret_cast<uint32_t*>(w + off);
    const int grid = std::min(ceil_div64(L, 256), current_sm_count() * 16);
    sample_keys_kernel<<<grid, 256, 0, st>>>(faces, face_idx, B, Nv, Nf, N, keys[0], vals[0]);
    const int cur = radix_sort_pairs(keys, vals, L, key_bits(kmax), counts, totals, st);
    vertex_offsets_kernel<<<std::min(ceil_div64(L + 1, 256), current_sm_count() * 16), 256, 0, st>>>(keys[cur], L, kmax, voff);
    vertex_grad_kernel<<<std::min(ceil_div64(kmax, 256), current_sm_count() * 16), 256, 0, st>>>(vals[cur], voff, bary, grad_points,
                                                                                  kmax, grad_verts);
    return cudaGetLastError();
}

}  // namespace cdk
