// p2s_common.cuh — shared device code of the point-to-surface kernels (p2s.cu, p2s_pruned.cu):
// the packed face record (R24), the packed-FP32 point-to-triangle squared distance, and the fp64
// closest point on the chosen face (R24's plane-or-edges formulation in fp64; the oracle uses the
// region decomposition instead and shares no code with this file).
#pragma once
#include "cd_device.cuh"

namespace cdk {

constexpr int kP2sR = 8;                           // points per thread
constexpr int kP2sQ = kFwdThreads * kP2sR;         // 1024 points per CTA
constexpr int kFaceTile = 128;                     // faces per shared-memory stage (12 KB)
constexpr int kFaceFloats = 24;                    // packed face record
constexpr int kP2sStages = 3;

constexpr int kFaceTileFaces = 128;   // alias used by the pruned path

// face record layout (floats): 0-2 a, 3-5 -e0, 6-8 -e1, 9-11 -e2 (negated edges: every "x - t e"
// is one fma with a positive operand), 12-14 n (unit), 15-17 -1/|e0|^2, -1/|e1|^2, -1/|e2|^2,
// 18-20 -g11/det, g01/det, -g00/det (inverse Gram of e0, e1 applied to -s, -t), 21 u/v offset
// (-1 for a degenerate face: its projection is never "inside"), 22-23 pad
__device__ __forceinline__ void write_face_record(const float* v, int Nv, const int* faces, int f, float* o) {
    const int ia = min(max(faces[3 * f], 0), Nv - 1);
    const int ib = min(max(faces[3 * f + 1], 0), Nv - 1);
    const int ic = min(max(faces[3 * f + 2], 0), Nv - 1);
    float A[3], e0[3], e1[3], e2[3];
    for (int k = 0; k < 3; ++k) {
        A[k] = v[3 * ia + k];
        e0[k] = __fsub_rn(v[3 * ib + k], A[k]);
        e1[k] = __fsub_rn(v[3 * ic + k], A[k]);
        e2[k] = __fsub_rn(v[3 * ic + k], v[3 * ib + k]);
    }
    // normal and Gram matrix in fp64, rounded once (better-conditioned face data)
    const double n0 = (double)e0[1] * e1[2] - (double)e0[2] * e1[1];
    const double n1 = (double)e0[2] * e1[0] - (double)e0[0] * e1[2];
    const double n2 = (double)e0[0] * e1[1] - (double)e0[1] * e1[0];
    const double nl = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
    const double g00 = (double)e0[0] * e0[0] + (double)e0[1] * e0[1] + (double)e0[2] * e0[2];
    const double g01 = (double)e0[0] * e1[0] + (double)e0[1] * e1[1] + (double)e0[2] * e1[2];
    const double g11 = (double)e1[0] * e1[0] + (double)e1[1] * e1[1] + (double)e1[2] * e1[2];
    const double g22 = (double)e2[0] * e2[0] + (double)e2[1] * e2[1] + (double)e2[2] * e2[2];
    const double det = g00 * g11 - g01 * g01;
    for (int k = 0; k < 3; ++k) {
        o[k] = A[k];
        o[3 + k] = -e0[k];
        o[6 + k] = -e1[k];
        o[9 + k] = -e2[k];
    }
    const bool nondeg = nl > 0.0 && det > 0.0;
    o[12] = nondeg ? (float)(n0 / nl) : 0.f;
    o[13] = nondeg ? (float)(n1 / nl) : 0.f;
    o[14] = nondeg ? (float)(n2 / nl) : 0.f;
    o[15] = g00 > 0.0 ? (float)(-1.0 / g00) : 0.f;
    o[16] = g11 > 0.0 ? (float)(-1.0 / g11) : 0.f;
    o[17] = g22 > 0.0 ? (float)(-1.0 / g22) : 0.f;
    o[18] = nondeg ? (float)(-g11 / det) : 0.f;
    o[19] = nondeg ? (float)(g01 / det) : 0.f;
    o[20] = nondeg ? (float)(-g00 / det) : 0.f;
    o[21] = nondeg ? 0.f : -1.f;
    o[22] = 0.f;
    o[23] = 0.f;
}

// clamp(a * b, 0, 1) per lane: f32x2 has no .sat, two scalar FMUL.SAT cost the same two dispatch cycles
__device__ __forceinline__ u64 sat_mul2(u64 a, u64 b) {
    float a0, a1, b0, b1;
    upk2(a, a0, a1);
    upk2(b, b0, b1);
    return pk2(__saturatef(__fmul_rn(a0, b0)), __saturatef(__fmul_rn(a1, b1)));
}
__device__ __forceinline__ u64 bc2(float x) { return pk2(x, x); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// Packed squared distance, per lane, of a point (qx, qy, qz) to a face record (R24, fixed op
// order); F(k) gives face float k as a packed pair.  With ne = -e: s' = ap.ne0 = -ap.e0,
// t0 = sat(s' * (-1/|e0|^2)), x - t0 e0 = fma(t0, ne0, ap).  Both callers below run this one op
// sequence, so a (point, face) pair gets the same bits whichever lane layout evaluates it.
template <class FaceK>
__device__ __forceinline__ void face_dist2_lanes(FaceK F, u64 qx, u64 qy, u64 qz, float& d0, float& d1) {
    const u64 ax = sub2(qx, F(0)), ay = sub2(qy, F(1)), az = sub2(qz, F(2));
    u64 s = mul2(ax, F(3));
    s = fma2(ay, F(4), s);
    s = fma2(az, F(5), s);
    u64 t = mul2(ax, F(6));
    t = fma2(ay, F(7), t);
    t = fma2(az, F(8), t);
    // in-plane coordinates of the projection
    u64 u = fma2(s, F(18), F(21));
    u = fma2(t, F(19), u);
    u64 v = fma2(s, F(19), F(21));
    v = fma2(t, F(20), v);
    // plane distance
    u64 h = mul2(ax, F(12));
    h = fma2(ay, F(13), h);
    h = fma2(az, F(14), h);
    const u64 pl = mul2(h, h);
    // edge a-b
    const u64 t0 = sat_mul2(s, F(15));
    u64 dx = fma2(t0, F(3), ax), dy = fma2(t0, F(4), ay), dz = fma2(t0, F(5), az);
    u64 dab = mul2(dx, dx);
    dab = fma2(dy, dy, dab);
    dab = fma2(dz, dz, dab);
    // edge a-c
    const u64 t1 = sat_mul2(t, F(16));
    dx = fma2(t1, F(6), ax);
    dy = fma2(t1, F(7), ay);
    dz = fma2(t1, F(8), az);
    u64 dac = mul2(dx, dx);
    dac = fma2(dy, dy, dac);
    dac = fma2(dz, dz, dac);
    // edge b-c: bp = ap - e0 = ap + ne0
    const u64 bx = add2(ax, F(3)), by = add2(ay, F(4)), bz = add2(az, F(5));
    u64 s2 = mul2(bx, F(9));
    s2 = fma2(by, F(10), s2);
    s2 = fma2(bz, F(11), s2);
    const u64 t2 = sat_mul2(s2, F(17));
    dx = fma2(t2, F(9), bx);
    dy = fma2(t2, F(10), by);
    dz = fma2(t2, F(11), bz);
    u64 dbc = mul2(dx, dx);
    dbc = fma2(dy, dy, dbc);
    dbc = fma2(dz, dz, dbc);
    float u0, u1, v0, v1, p0, p1, ab0, ab1, ac0, ac1, bc0, bc1;
    upk2(u, u0, u1);
    upk2(v, v0, v1);
    upk2(pl, p0, p1);
    upk2(dab, ab0, ab1);
    upk2(dac, ac0, ac1);
    upk2(dbc, bc0, bc1);
    const float w0 = __fsub_rn(__fsub_rn(1.0f, u0), v0), w1 = __fsub_rn(__fsub_rn(1.0f, u1), v1);
    const bool in0 = fmin3(u0, v0, w0) >= 0.0f, in1 = fmin3(u1, v1, w1) >= 0.0f;
    d0 = fmin3(ab0, ac0, fminf(bc0, in0 ? p0 : INFINITY));
    d1 = fmin3(ab1, ac1, fminf(bc1, in1 ? p1 : INFINITY));
}

// Two points (qx, qy, qz lanes) against one face record (face floats broadcast to both lanes).
__device__ __forceinline__ void face_dist2(const float* f, u64 qx, u64 qy, u64 qz, float& d0, float& d1) {
    face_dist2_lanes([&](int k) { return bc2(f[k]); }, qx, qy, qz, d0, d1);
}

// A 24-float face record (96 B, 16-B aligned) as six 16-byte loads.
__device__ __forceinline__ void load_face_record(const float* src, float* dst) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int k = 0; k < kFaceFloats / 4; ++k) {
        const float4 v = __ldg(s4 + k);
        dst[4 * k] = v.x;
        dst[4 * k + 1] = v.y;
        dst[4 * k + 2] = v.z;
        dst[4 * k + 3] = v.w;
    }
}

// ONE point (px, py, pz) against TWO face records (fa in the low lane, fb in the high lane): used
// where one point meets many faces (the exact-face re-scans).
__device__ __forceinline__ void face_dist2_2f(const float* fa, const float* fb, float px, float py, float pz,
                                              float& da, float& db) {
    face_dist2_lanes([&](int k) { return pk2(fa[k], fb[k]); }, bc2(px), bc2(py), bc2(pz), da, db);
}

// fp64 closest point of p on the triangle (A, B, C) and its squared distance: R24's formulation
// carried out in fp64 for the one face the hot loop chose.  Candidates, in this
// order: the foot of the perpendicular on the face's plane, taken only when its barycentrics
// (solved with the inverse Gram matrix of e0 = B - A, e1 = C - A) are all >= 0; then the nearest
// point of each edge AB, AC, BC (parameter clamped to [0, 1]).  The first candidate at the
// smallest squared distance wins.  A face with zero Gram determinant (a segment or a point) has
// no plane candidate.  lam = barycentric coordinates of the returned point on (A, B, C).
__device__ __forceinline__ double face_foot64(const double p[3], const double A[3], const double Bv[3], const double C[3],
                                              double out[3], double lam[3]) {
    double e0[3], e1[3], e2[3], ap[3], bp[3];
    for (int k = 0; k < 3; ++k) {
        e0[k] = Bv[k] - A[k];
        e1[k] = C[k] - A[k];
        e2[k] = C[k] - Bv[k];
        ap[k] = p[k] - A[k];
        bp[k] = p[k] - Bv[k];
    }
    const double g00 = e0[0] * e0[0] + e0[1] * e0[1] + e0[2] * e0[2];
    const double g01 = e0[0] * e1[0] + e0[1] * e1[1] + e0[2] * e1[2];
    const double g11 = e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2];
    const double g22 = e2[0] * e2[0] + e2[1] * e2[1] + e2[2] * e2[2];
    const double s = ap[0] * e0[0] + ap[1] * e0[1] + ap[2] * e0[2];
    const double t = ap[0] * e1[0] + ap[1] * e1[1] + ap[2] * e1[2];
    const double s2 = bp[0] * e2[0] + bp[1] * e2[1] + bp[2] * e2[2];
    double best = INFINITY;
    auto take = [&](double l0, double l1, double l2) {
        double q[3], dd = 0.0;
        for (int k = 0; k < 3; ++k) {
            q[k] = l0 * A[k] + l1 * Bv[k] + l2 * C[k];
            dd += (p[k] - q[k]) * (p[k] - q[k]);
        }
        if (dd < best) {
            best = dd;
            for (int k = 0; k < 3; ++k) out[k] = q[k];
            lam[0] = l0;
            lam[1] = l1;
            lam[2] = l2;
        }
    };
    const double det = g00 * g11 - g01 * g01;
    if (det > 0.0) {
        const double v = (g11 * s - g01 * t) / det, w = (g00 * t - g01 * s) / det, u = 1.0 - v - w;
        if (u >= 0.0 && v >= 0.0 && w >= 0.0) take(u, v, w);
    }
    const double tab = g00 > 0.0 ? fmin(fmax(s / g00, 0.0), 1.0) : 0.0;
    const double tac = g11 > 0.0 ? fmin(fmax(t / g11, 0.0), 1.0) : 0.0;
    const double tbc = g22 > 0.0 ? fmin(fmax(s2 / g22, 0.0), 1.0) : 0.0;
    take(1.0 - tab, tab, 0.0);
    take(1.0 - tac, 0.0, tac);
    take(0.0, 1.0 - tbc, tbc);
    return best;
}

}  // namespace cdk
