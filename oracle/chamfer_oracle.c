/*
 * chamfer_oracle.c — CPU ORACLE for the batched Chamfer / nearest-neighbour / F-score path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_1911_05063_b200/, libcd.so) never links, imports or calls it, and this file
 * shares no code, header, table or helper with the CUDA path.
 *
 * What it computes (plain definitions, fp64, no blocking / fusion / reordering):
 *
 *   PAPER.md:253-254 (§2.5 "Loss Functions and Metrics"): "comparing ... point clouds
 *   might require matching positions of thousands of points ... Chamfer distance ...
 *   for pointclouds".  The paper does not write the formula; we follow SPEC.md:441
 *   (metrics/chamfer_distance):
 *       CD = (1/|A|) sum_a min_b ||a-b||^2 + (1/|B|) sum_b min_a ||a-b||^2,
 *       "VJP holds the argmin fixed".
 *   Readings taken where the paper is silent are listed in DESIGN.md §3 (R1..R18),
 *   following SURVEY.md §8.c.2.
 *
 * Functions:
 *   oracle_nn            directed nearest neighbour (d1, lowest-index argmin i1, second-
 *                        nearest value d2) for a list of query rows — SPEC.md:441 brute force.
 *   oracle_backward      analytic VJP of the per-point distances with the argmin held fixed
 *                        (SPEC.md:441), accumulated in the defining order (own term, then
 *                        scatter terms in ascending source index) plus the condition scale
 *                        S = sum |terms| used by the gradient gate (R14).
 *   oracle_sample_mesh   NEXT-4: area-proportional face choice (exact integer CDF, R19), square-
 *                        root barycentrics, sampled points — fp64.
 *   oracle_sample_vjp    NEXT-4: VJP of the sampled points w.r.t. the vertices, choices fixed.
 *   oracle_p2s           NEXT-3: point-to-surface: squared distance to the closest
 *                        triangle (region decomposition), lowest face on ties, closest point + its
 *                        barycentric coordinates — fp64.
 *   mirror_nn_f32        NOT the oracle: an fp32 re-evaluation of the distance formula in the
 *                        operation order DESIGN.md §4.2 fixes for the kernel
 *                        (dx=x-y; s=dx*dx; s=fma(dy,dy,s); s=fma(dz,dz,s), all IEEE RN),
 *                        strict-< lowest-index argmin.  Written from that formula, not from
 *                        the kernel source; used to check the GPU's distance BITS.
 *
 * Build (see __graft_entry__.build / oracle/__init__.py):
 *   gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC -o liboracle.so chamfer_oracle.c -lm
 * -ffp-contract=off keeps a*b+c as two roundings wherever the source writes two operations.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_abi_version(void) { return 1; }

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * Directed nearest neighbour, fp64.
 *   q: B x N x 3 (queries), t: B x M x 3 (targets), row-major, fp64.
 *   rows: flattened query rows (b*N + i) to evaluate, nrows of them; rows == NULL means all B*N.
 *   Outputs per evaluated row r (index r in the rows list):
 *     d1[r] = min_j ||q_{b,i} - t_{b,j}||^2            ("min_b ||a-b||^2", squared per SPEC.md:511)
 *     i1[r] = lowest j attaining d1 (strict <, j ascending)   (R3)
 *     d2[r] = min over j != i1 of the same quantity (second-nearest VALUE; may equal d1),
 *             +inf when M == 1.                               (R12 gap rule)
 *   nthreads <= 0: OpenMP default.
 */
int oracle_nn(const double* q, const double* t, int64_t B, int64_t N, int64_t M,
              const int64_t* rows, int64_t nrows,
              double* d1, int32_t* i1, double* d2, int nthreads) {
    if (!q || !t || !d1 || !i1 || B < 1 || N < 1 || M < 1) return 1;
    int64_t total = rows ? nrows : B * N;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < total; ++r) {
        int64_t flat = rows ? rows[r] : r;
        int64_t b = flat / N;
        const double* x = q + 3 * flat;
        const double* yb = t + 3 * b * M;
        double best = INFINITY, second = INFINITY;
        int32_t arg = -1;
        for (int64_t j = 0; j < M; ++j) {
            double dx = x[0] - yb[3 * j + 0];
            double dy = x[1] - yb[3 * j + 1];
            double dz = x[2] - yb[3 * j + 2];
            double e = dx * dx + dy * dy + dz * dz;
            if (e < best) {            /* strict <: the earliest j keeps exact ties */
                second = best;
                best = e;
                arg = (int32_t)j;
            } else if (e < second) {
                second = e;
            }
        }
        d1[r] = best;
        i1[r] = arg;
        if (d2) d2[r] = second;
    }
    return 0;
}

/*
 * Backward (VJP with argmin held fixed), fp64.
 *   x: B x N x 3, y: B x M x 3 (fp64 copies of the fp32 clouds)
 *   idx_xy: B x N (a_i in [0,M)), idx_yx: B x M (b_j in [0,N))
 *   g: B x N upstream dL/dd_xy, h: B x M upstream dL/dd_yx; if g (h) is NULL the scalar
 *   g_scalar (h_scalar) is used for every element (R8: loss gradient is a fill).
 *   Outputs grad_x: B x N x 3, grad_y: B x M x 3 and the per-element condition scales
 *   sx, sy (sum of |term| over every term accumulated into that element; may be NULL).
 *
 *   grad_x_i = 2 g_i (x_i - y_{a_i}) + sum_{j : b_j = i} 2 h_j (x_i - y_j)
 *   grad_y_j = 2 h_j (y_j - x_{b_j}) + sum_{i : a_i = j} 2 g_i (y_j - x_i)
 *   (d/dx ||x - y||^2 = 2 (x - y)).  Order: own term, then scatter terms in ascending
 *   source index (the loops below visit sources in ascending order).
 */
int oracle_backward(const double* x, const double* y, int64_t B, int64_t N, int64_t M,
                    const int32_t* idx_xy, const int32_t* idx_yx,
                    const double* g, const double* h, double g_scalar, double h_scalar,
                    double* grad_x, double* grad_y, double* sx, double* sy) {
    if (!x || !y || !idx_xy || !idx_yx || !grad_x || !grad_y || B < 1 || N < 1 || M < 1) return 1;
    for (int64_t b = 0; b < B; ++b) {
        const double* xb = x + 3 * b * N;
        const double* yb = y + 3 * b * M;
        double* gx = grad_x + 3 * b * N;
        double* gy = grad_y + 3 * b * M;
        double* ssx = sx ? sx + 3 * b * N : NULL;
        double* ssy = sy ? sy + 3 * b * M : NULL;
        /* own terms */
        for (int64_t i = 0; i < N; ++i) {
            int32_t a = idx_xy[b * N + i];
            if (a < 0 || a >= M) return 2;
            double gi = g ? g[b * N + i] : g_scalar;
            for (int c = 0; c < 3; ++c) {
                double term = 2.0 * gi * (xb[3 * i + c] - yb[3 * a + c]);
                gx[3 * i + c] = term;
                if (ssx) ssx[3 * i + c] = fabs(term);
            }
        }
        for (int64_t j = 0; j < M; ++j) {
            int32_t a = idx_yx[b * M + j];
            if (a < 0 || a >= N) return 2;
            double hj = h ? h[b * M + j] : h_scalar;
            for (int c = 0; c < 3; ++c) {
                double term = 2.0 * hj * (yb[3 * j + c] - xb[3 * a + c]);
                gy[3 * j + c] = term;
                if (ssy) ssy[3 * j + c] = fabs(term);
            }
        }
        /* scatter terms of d_xy into grad_y, sources i ascending */
        for (int64_t i = 0; i < N; ++i) {
            int32_t a = idx_xy[b * N + i];
            double gi = g ? g[b * N + i] : g_scalar;
            for (int c = 0; c < 3; ++c) {
                double term = 2.0 * gi * (yb[3 * a + c] - xb[3 * i + c]);
                gy[3 * a + c] += term;
                if (ssy) ssy[3 * a + c] += fabs(term);
            }
        }
        /* scatter terms of d_yx into grad_x, sources j ascending */
        for (int64_t j = 0; j < M; ++j) {
            int32_t a = idx_yx[b * M + j];
            double hj = h ? h[b * M + j] : h_scalar;
            for (int c = 0; c < 3; ++c) {
                double term = 2.0 * hj * (xb[3 * a + c] - yb[3 * j + c]);
                gx[3 * a + c] += term;
                if (ssx) ssx[3 * a + c] += fabs(term);
            }
        }
    }
    return 0;
}

/*
 * fp32 mirror of the kernel's specified arithmetic, NOT the oracle.
 *   q: B x N x 3 fp32, t: B x M x 3 fp32; rows as in oracle_nn.
 *   d[r] = fp32 value of  s = RN(dx*dx); s = fmaf(dy,dy,s); s = fmaf(dz,dz,s)
 *          with dx = RN(x - y) etc., minimised with strict < over j ascending.
 *   idx[r] = lowest j attaining it; -1 (and +inf) if no candidate compares < +inf.
 */
int mirror_nn_f32(const float* q, const float* t, int64_t B, int64_t N, int64_t M,
                  const int64_t* rows, int64_t nrows, float* d, int32_t* idx, int nthreads) {
    if (!q || !t || !d || !idx || B < 1 || N < 1 || M < 1) return 1;
    int64_t total = rows ? nrows : B * N;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < total; ++r) {
        int64_t flat = rows ? rows[r] : r;
        int64_t b = flat / N;
        const float* x = q + 3 * flat;
        const float* yb = t + 3 * b * M;
        float best = INFINITY;
        int32_t arg = -1;
        for (int64_t j = 0; j < M; ++j) {
            float dx = x[0] - yb[3 * j + 0];
            float dy = x[1] - yb[3 * j + 1];
            float dz = x[2] - yb[3 * j + 2];
            float s = dx * dx;
            s = fmaf(dy, dy, s);
            s = fmaf(dz, dz, s);
            if (s < best) {
                best = s;
                arg = (int32_t)j;
            }
        }
        d[r] = best;
        idx[r] = arg;
    }
    return 0;
}

/* ====================================================================================== NEXT-4
 * Differentiable surface sampling ("differentiable surface sampling
 * ... by application of the reparameterization trick").  Plain definitions in fp64; the random
 * numbers are inputs (uint32 r_face, fp32 r1, r2 per sample).  Readings R19-R22 in DESIGN.md §11.
 *
 * R19 face choice with probability proportional to area, made exactly reproducible:
 *   e1 = v1 - v0, e2 = v2 - v0 (fp64 from fp32 vertices, exact);
 *   c  = e1 x e2 (cx = e1y*e2z - e1z*e2y, cy = e1z*e2x - e1x*e2z, cz = e1x*e2y - e1y*e2x);
 *   area_f = 0.5 * sqrt(cx*cx + cy*cy + cz*cz)              (fp64, this op order, no contraction)
 *   k = 52 - e where Nf * max_f area_f = m * 2^e, m in [0.5, 1)  (frexp);  q_f = floor(area_f * 2^k)
 *   P_f = sum_{g <= f} q_g (exact integers), S = P_{Nf-1};  t = (r_face * S) >> 32;
 *   face = min { f : P_f > t }   (S == 0: face 0)
 * R20 barycentrics: s = sqrt(r1); (w0, w1, w2) = (1 - s, s (1 - r2), s r2)
 * R21 point = w0 v_a + w1 v_b + w2 v_c
 * R22 VJP with face choice and weights fixed: grad_v = sum over (sample i, corner k) with
 *     faces[face_i][k] == v of w_{i,k} * g_i, accumulated in ascending (i, k) order.
 */
static double area64(const float* v, const int32_t* f) {
    const float* a = v + 3 * (int64_t)f[0];
    const float* b = v + 3 * (int64_t)f[1];
    const float* c = v + 3 * (int64_t)f[2];
    double e1x = (double)b[0] - (double)a[0], e1y = (double)b[1] - (double)a[1], e1z = (double)b[2] - (double)a[2];
    double e2x = (double)c[0] - (double)a[0], e2y = (double)c[1] - (double)a[1], e2z = (double)c[2] - (double)a[2];
    double cx = e1y * e2z - e1z * e2y;
    double cy = e1z * e2x - e1x * e2z;
    double cz = e1x * e2y - e1y * e2x;
    return 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
}

/* verts B x Nv x 3 fp32, faces Nf x 3 (shared topology), r_face B x N uint32, r_bary B x N x 2 fp32.
 * Outputs: points B x N x 3 (fp64), face_idx B x N, bary B x N x 3 (fp64); cdf (B x Nf uint64, may be
 * NULL) = the inclusive quantised prefix P_f. */
int oracle_sample_mesh(const float* verts, const int32_t* faces, int64_t B, int64_t Nv, int64_t Nf, int64_t N,
                       const uint32_t* r_face, const float* r_bary, double* points, int32_t* face_idx,
                       double* bary, uint64_t* cdf_out) {
    if (!verts || !faces || !r_face || !r_bary || !points || !face_idx || B < 1 || Nv < 1 || Nf < 1 || N < 1) return 1;
    uint64_t* P = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)Nf);
    if (!P) return 3;
    for (int64_t b = 0; b < B; ++b) {
        const float* v = verts + 3 * b * Nv;
        double amax = 0.0;
        for (int64_t f = 0; f < Nf; ++f) {
            for (int k = 0; k < 3; ++k)
                if (faces[3 * f + k] < 0 || faces[3 * f + k] >= Nv) { free(P); return 2; }
            double a = area64(v, faces + 3 * f);
            if (a > amax) amax = a;
        }
        int e = 0;
        if (amax > 0.0) frexp(amax * (double)Nf, &e);
        uint64_t run = 0;
        for (int64_t f = 0; f < Nf; ++f) {
            double a = area64(v, faces + 3 * f);
            uint64_t q = amax > 0.0 ? (uint64_t)floor(ldexp(a, 52 - e)) : 0;
            run += q;
            P[f] = run;
            if (cdf_out) cdf_out[b * Nf + f] = run;
        }
        const uint64_t S = run;
        for (int64_t i = 0; i < N; ++i) {
            const int64_t s = b * N + i;
            int64_t face = 0;
            if (S > 0) {
                const unsigned __int128 prod = (unsigned __int128)r_face[s] * (unsigned __int128)S;
                const uint64_t t = (uint64_t)(prod >> 32);
                /* plain linear scan (the definition: smallest f with P_f > t) */
                face = 0;
                while (face < Nf - 1 && !(P[face] > t)) ++face;
            }
            face_idx[s] = (int32_t)face;
            const double r1 = (double)r_bary[2 * s], r2 = (double)r_bary[2 * s + 1];
            const double sq = sqrt(r1);
            const double w[3] = {1.0 - sq, sq * (1.0 - r2), sq * r2};
            for (int c = 0; c < 3; ++c) {
                double acc = 0.0;
                for (int k = 0; k < 3; ++k) acc += w[k] * (double)v[3 * (int64_t)faces[3 * face + k] + c];
                points[3 * s + c] = acc;
            }
            if (bary)
                for (int k = 0; k < 3; ++k) bary[3 * s + k] = w[k];
        }
    }
    free(P);
    return 0;
}

/* VJP (R22): bary B x N x 3 (the weights used by the forward), face_idx B x N, grad_points B x N x 3;
 * output grad_verts B x Nv x 3 (fp64). */
int oracle_sample_vjp(const double* bary, const int32_t* face_idx, const int32_t* faces, int64_t B, int64_t Nv,
                      int64_t Nf, int64_t N, const double* grad_points, double* grad_verts) {
    if (!bary || !face_idx || !faces || !grad_points || !grad_verts) return 1;
    for (int64_t j = 0; j < B * Nv * 3; ++j) grad_verts[j] = 0.0;
    for (int64_t b = 0; b < B; ++b)
        for (int64_t i = 0; i < N; ++i) {
            const int64_t s = b * N + i;
            const int64_t f = face_idx[s];
            if (f < 0 || f >= Nf) return 2;
            for (int k = 0; k < 3; ++k) {
                const int64_t v = faces[3 * f + k];
                for (int c = 0; c < 3; ++c) grad_verts[3 * (b * Nv + v) + c] += bary[3 * s + k] * grad_points[3 * s + c];
            }
        }
    return 0;
}

/* ====================================================================================== NEXT-3
 * Point-to-surface loss ("the point-to-surface loss [GEOMetrics] for Meshes";
 * "mean over points of squared distance to the closest triangle; VJP: 2(p - closest)/P
 * per point, closest point held fixed").  fp64, brute force over all faces (plain definition).
 * Closest point on a triangle: the standard region decomposition (Voronoi regions of the vertices,
 * edges and face), written out below.  Readings R23-R25 in DESIGN.md §11.
 */
static void closest_on_triangle(const double p[3], const double a[3], const double b[3], const double c[3],
                                double out[3], double lam[3]) {
    double ab[3], ac[3], ap[3], bp[3], cp[3];
    for (int k = 0; k < 3; ++k) {
        ab[k] = b[k] - a[k];
        ac[k] = c[k] - a[k];
        ap[k] = p[k] - a[k];
        bp[k] = p[k] - b[k];
        cp[k] = p[k] - c[k];
    }
    const double d1 = ab[0] * ap[0] + ab[1] * ap[1] + ab[2] * ap[2];
    const double d2 = ac[0] * ap[0] + ac[1] * ap[1] + ac[2] * ap[2];
    const double d3 = ab[0] * bp[0] + ab[1] * bp[1] + ab[2] * bp[2];
    const double d4 = ac[0] * bp[0] + ac[1] * bp[1] + ac[2] * bp[2];
    const double d5 = ab[0] * cp[0] + ab[1] * cp[1] + ab[2] * cp[2];
    const double d6 = ac[0] * cp[0] + ac[1] * cp[1] + ac[2] * cp[2];
    const double vc = d1 * d4 - d3 * d2;
    const double vb = d5 * d2 - d1 * d6;
    const double va = d3 * d6 - d5 * d4;
    double l0, l1, l2;
    if (d1 <= 0.0 && d2 <= 0.0) {                                  /* vertex region A */
        l0 = 1.0; l1 = 0.0; l2 = 0.0;
    } else if (d3 >= 0.0 && d4 <= d3) {                           /* vertex region B */
        l0 = 0.0; l1 = 1.0; l2 = 0.0;
    } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {             /* edge AB */
        const double v = d1 / (d1 - d3);
        l0 = 1.0 - v; l1 = v; l2 = 0.0;
    } else if (d6 >= 0.0 && d5 <= d6) {                           /* vertex region C */
        l0 = 0.0; l1 = 0.0; l2 = 1.0;
    } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {             /* edge AC */
        const double w = d2 / (d2 - d6);
        l0 = 1.0 - w; l1 = 0.0; l2 = w;
    } else if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) { /* edge BC */
        const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        l0 = 0.0; l1 = 1.0 - w; l2 = w;
    } else {                                                       /* face interior */
        const double den = va + vb + vc;
        const double v = vb / den, w = vc / den;
        l0 = 1.0 - v - w; l1 = v; l2 = w;
    }
    for (int k = 0; k < 3; ++k) out[k] = l0 * a[k] + l1 * b[k] + l2 * c[k];
    lam[0] = l0; lam[1] = l1; lam[2] = l2;
}

/* points B x N x 3 fp32; verts B x Nv x 3 fp32; faces Nf x 3 (shared topology).
 * Outputs (per evaluated row; rows == NULL means all B*N): d (min squared distance), face (lowest
 * face index attaining it), d2 (second-smallest over other faces; +inf if Nf == 1), closest point
 * (3) and its barycentric coordinates on that face (3). */
int oracle_p2s(const float* points, const float* verts, const int32_t* faces, int64_t B, int64_t N, int64_t Nv,
               int64_t Nf, const int64_t* rows, int64_t nrows, double* d, int32_t* face, double* d2,
               double* closest, double* lam_out, int nthreads) {
    if (!points || !verts || !faces || !d || !face || B < 1 || N < 1 || Nv < 1 || Nf < 1) return 1;
    for (int64_t f = 0; f < Nf; ++f)
        for (int k = 0; k < 3; ++k)
            if (faces[3 * f + k] < 0 || faces[3 * f + k] >= Nv) return 2;
    int64_t total = rows ? nrows : B * N;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t r = 0; r < total; ++r) {
        const int64_t s = rows ? rows[r] : r;
        const int64_t b = s / N;
        const double p[3] = {points[3 * s], points[3 * s + 1], points[3 * s + 2]};
        const float* v = verts + 3 * b * Nv;
        double best = INFINITY, second = INFINITY, bc[3] = {0, 0, 0}, bl[3] = {0, 0, 0};
        int32_t arg = -1;
        for (int64_t f = 0; f < Nf; ++f) {
            double A[3], Bq[3], C[3], q[3], l[3];
            for (int k = 0; k < 3; ++k) {
                A[k] = v[3 * (int64_t)faces[3 * f] + k];
                Bq[k] = v[3 * (int64_t)faces[3 * f + 1] + k];
                C[k] = v[3 * (int64_t)faces[3 * f + 2] + k];
            }
            closest_on_triangle(p, A, Bq, C, q, l);
            const double e = (p[0] - q[0]) * (p[0] - q[0]) + (p[1] - q[1]) * (p[1] - q[1]) + (p[2] - q[2]) * (p[2] - q[2]);
            if (e < best) {
                second = best;
                best = e;
                arg = (int32_t)f;
                for (int k = 0; k < 3; ++k) { bc[k] = q[k]; bl[k] = l[k]; }
            } else if (e < second) {
                second = e;
            }
        }
        d[r] = best;
        face[r] = arg;
        if (d2) d2[r] = second;
        if (closest) for (int k = 0; k < 3; ++k) closest[3 * r + k] = bc[k];
        if (lam_out) for (int k = 0; k < 3; ++k) lam_out[3 * r + k] = bl[k];
    }
    return 0;
}
