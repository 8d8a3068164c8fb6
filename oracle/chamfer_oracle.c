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
