/*
 * cd.h — C ABI of libcd.so: batched exact nearest-neighbour Chamfer distance, its backward, and
 * the F-score, for B x N x 3 and B x M x 3 fp32 point clouds on one NVIDIA B200 (sm_100a).
 *
 * What the operations are (citations: PAPER.md line, SPEC.md line; readings R1..R18 are listed in
 * DESIGN.md §3):
 *   PAPER.md:253-254 (§2.5 "Loss Functions and Metrics"): Chamfer distance for point clouds,
 *   "matching positions of thousands of points", "CUDA functions are a necessity".
 *   SPEC.md:441 (metrics/chamfer_distance): CD = (1/|A|) sum_a min_b ||a-b||^2
 *   + (1/|B|) sum_b min_a ||a-b||^2; brute-force nearest neighbours; "VJP holds the argmin fixed".
 *   Per-point squared distances and argmin indices, the gradient scatter through those indices and
 *   the F-score at a threshold are the north star's function set (BASELINE.json north_star).
 *
 * Conventions (all entry points):
 *   - Every array argument is a DEVICE pointer to contiguous row-major data owned by the caller.
 *     Clouds are fp32 (x, y, z) triples, AoS: x[(b*N + i)*3 + c].  Indices are int32, 0-based.
 *   - The library never allocates, frees or synchronises (except cd_step_host, which synchronises
 *     nothing either but copies host<->device asynchronously).  Scratch memory comes only from the
 *     caller's workspace (size from cd_workspace_size, 256-byte aligned base).  Every call is
 *     asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream) and capturable in a
 *     CUDA graph.
 *   - Validation happens before any launch.  On error nothing is launched, outputs are untouched,
 *     and cd_last_error_string() (thread-local) describes the problem.  CD_ERR_CUDA reports a
 *     launch failure (the CUDA error string is kept in cd_last_error_string()).
 *   - Determinism: per-point outputs (d, idx, gradients) are bitwise reproducible for given inputs
 *     and independent of tiling, split count and query slicing.
 *   - Preconditions: B, N, M >= 1 (empty cloud -> domain error =
 *     CD_ERR_INVALID_VALUE); finite coordinates.  Non-finite input does not crash: a
 *     query whose every distance is NaN/+inf gets d = +inf, idx = -1 (R6).
 *   - Thread safety: re-entrant.  Mutable state: the thread-local error string and test-hook settings
 *     (cd_set_forward_splits / _mode / _profile_events, per thread), and process-wide per-DEVICE caches
 *     of the SM count and kernel occupancies (filled once per device ordinal, idempotent atomics).
 */
#ifndef CD_H_
#define CD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CD_ABI_VERSION 5
#define CD_MAX_PEERS 16   /* cd_forward_cols_peers: most key arrays reduced on read */

#if defined(__GNUC__)
#define CD_API __attribute__((visibility("default")))
#else
#define CD_API
#endif

typedef void* cd_stream_t; /* cudaStream_t */

typedef enum {
    CD_OK = 0,
    CD_ERR_INVALID_VALUE = 1,     /* null pointer, B/N/M < 1 (empty cloud), tau < 0, bad slice */
    CD_ERR_MISALIGNED = 2,        /* cloud base pointer not 4-byte aligned / workspace not 256-B aligned */
    CD_ERR_TOO_LARGE = 3,         /* B*N or B*M or B*(N+M) exceeds 2^31-1, B > 65535, or workspace too small */
    CD_ERR_UNSUPPORTED_DEVICE = 4,/* current device is not sm_100 */
    CD_ERR_CUDA = 5               /* a CUDA runtime call failed; see cd_last_error_string() */
} cd_status;

typedef enum {
    CD_OP_FORWARD = 0,   /* cd_forward */
    CD_OP_FSCORE = 1,    /* cd_fscore */
    CD_OP_BACKWARD = 2,  /* cd_backward */
    CD_OP_STEP = 3,      /* cd_step_host: forward + finalize + backward (+ staging of the clouds) */
    CD_OP_FORWARD_PRUNED = 4, /* cd_forward_pruned */
    CD_OP_SAMPLE = 5,          /* cd_sample_mesh (cd_sample_workspace_size) */
    CD_OP_SAMPLE_BACKWARD = 6, /* cd_sample_mesh_backward (cd_sample_workspace_size) */
    CD_OP_P2S = 7,             /* cd_p2s_forward (cd_p2s_workspace_size) */
    CD_OP_P2S_BACKWARD = 8,    /* cd_p2s_backward (cd_p2s_workspace_size) */
    CD_OP_P2S_PRUNED = 9       /* cd_p2s_forward_pruned (cd_p2s_workspace_size) */
} cd_op;

/*
 * cd_forward — both nearest-neighbour directions.
 *   x: B x N x 3 fp32, y: B x M x 3 fp32.
 *   Query slices (for query-sharding): X rows [q0, q1) of every batch element are
 *   searched against all of Y, and Y rows [r0, r1) against all of X.  Full problem: q0=0, q1=N,
 *   r0=0, r1=M.  An empty slice (q0 == q1 or r0 == r1) skips that direction.
 *   Outputs (slice-sized, row stride = slice length):
 *     d_xy  [B x (q1-q0)] fp32: min_j ||x_{b,i} - y_{b,j}||^2 (squared, R2), fp32 op order DESIGN.md §4.2
 *     idx_xy[B x (q1-q0)] int32: lowest j attaining it (R3)
 *     d_yx  [B x (r1-r0)], idx_yx[B x (r1-r0)]: the same with the roles swapped
 *     partials [B x 4] fp64 (may be NULL): sum of d_xy over the slice, sum of d_yx over the slice,
 *       hits_xy, hits_yx (exact counts stored as fp64; 0 when tau < 0).  Sums are accumulated in
 *       fp64 in a fixed order (R9).  Partials from several slices/ranks add up (R18).
 *   tau >= 0: F-score hit counting, hit iff (double)d <= (double)tau * (double)tau (R11, R16).
 *   tau < 0: no hit counting.
 */
CD_API cd_status cd_forward(const float* x, const float* y, int B, int N, int M,
                     int q0, int q1, int r0, int r1,
                     float* d_xy, int32_t* idx_xy, float* d_yx, int32_t* idx_yx,
                     double* partials, float tau,
                     void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_forward_rows / cd_forward_cols — the forward split for query sharding: the fused
 * kernel evaluates every distance once for both directions, so a rank that owns X rows [q0, q1)
 * gets (a) the final d_xy / idx_xy for those rows and (b) for EVERY Y point a column key
 *     colkeys[b*M + j] = (float bits of min_{i in [q0,q1)} ||x_i - y_j||^2) << 32 | (first row of the
 *                        lowest 16-row group attaining it)        (int64, always >= 0)
 * or INT64_MAX when no row contributed.  Keys from several row slices combine with an element-wise
 * MIN (e.g. an all-reduce MIN over ranks): the minimum key encodes the minimum distance and the
 * lowest row group.  cd_forward_cols then turns reduced keys into d_yx / idx_yx for Y rows [r0, r1)
 * (re-evaluating the winning group's 16 rows with the same fp32 ops, lowest index).
 *   cd_forward_rows: d_xy, idx_xy [B x (q1-q0)]; colkeys [B x M] (written); partials [B x 4] (may be
 *     NULL): writes columns 0 and 2 only (sum d_xy over the slice, hits_xy).  An empty slice
 *     (q0 == q1, e.g. more ranks than rows) is valid: keys = identity, partials 0.
 *   cd_forward_cols: colkeys [B x M] (read); d_yx, idx_yx [B x (r1-r0)]; partials: writes columns 1
 *     and 3 only.  An empty slice (r0 == r1) is valid and resolves nothing.
 * Results are bit-identical to cd_forward on the full problem.
 */
CD_API cd_status cd_forward_rows(const float* x, const float* y, int B, int N, int M, int q0, int q1,
                          float* d_xy, int32_t* idx_xy, int64_t* colkeys, double* partials, float tau,
                          void* workspace, size_t workspace_bytes, cd_stream_t stream);
CD_API cd_status cd_forward_cols(const float* x, const float* y, int B, int N, int M,
                          const int64_t* colkeys, int r0, int r1, float* d_yx, int32_t* idx_yx,
                          double* partials, float tau,
                          void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_forward_cols_peers — cd_forward_cols with the all-reduce MIN of the column keys fused into the
 * resolve (query sharding without a separate collective): the key of column j is the
 * element-wise MIN over the npeers arrays colkeys[0..npeers) (each B x M int64 as cd_forward_rows
 * writes them), read directly — typically this rank's array and its peers' arrays mapped over
 * NVLink (CUDA peer access / symmetric memory).  Only the keys of the resolved slice [r0, r1) are
 * read (a reduce-scatter's traffic, not an all-reduce's).
 *   colkeys: HOST array of npeers DEVICE pointers, each 8-byte aligned and readable from the
 *     current device; the caller guarantees every array is complete (all ranks' cd_forward_rows
 *     finished, e.g. a cross-device barrier) before the launch and stays unmodified until it ends.
 *   1 <= npeers <= CD_MAX_PEERS, else CD_ERR_INVALID_VALUE; other arguments, outputs and results
 *   exactly as cd_forward_cols given the MIN-reduced keys (bit-identical).
 */
CD_API cd_status cd_forward_cols_peers(const float* x, const float* y, int B, int N, int M,
                                const int64_t* const* colkeys, int npeers, int r0, int r1,
                                float* d_yx, int32_t* idx_yx, double* partials, float tau,
                                void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_forward_pruned — the same outputs as cd_forward on the full problem (q0=0,q1=N,r0=0,r1=M)
 * computed with far fewer distance evaluations on large clouds (the exact
 * accelerated search SPEC.md:441/446 asks to equal brute force): both clouds are sorted along a
 * Hilbert curve per batch element, every 256-row query tile visits 512-point target tiles in order
 * of a strict lower bound of their squared distance and stops once that bound exceeds the largest
 * current minimum among its rows.  Distances are the same fp32 values as the brute force (same op
 * order, every pair that could be a minimum is evaluated) and so are the indices: the lowest index
 * among exactly equal distances (ties inside one 32-point block are settled by the re-scan, ties
 * across blocks by a full scan of the row; R3').  Partials as cd_forward (sum order
 * differs: equal within fp64 rounding).
 * Limits: at most 4,194,304 points per cloud per batch element (CD_ERR_TOO_LARGE).
 * Workspace: cd_workspace_size(CD_OP_FORWARD_PRUNED, B, N, M).
 */
CD_API cd_status cd_forward_pruned(const float* x, const float* y, int B, int N, int M,
                          float* d_xy, int32_t* idx_xy, float* d_yx, int32_t* idx_yx,
                          double* partials, float tau,
                          void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_finalize — per-batch Chamfer, batch loss and F-score from the partials.
 *   partials [B x 4] fp64 (after an optional all-reduce sum across ranks, R18).
 *   cd_per_batch[b] = w1 * partials[b][0] / N + w2 * partials[b][1] / M      (R1)
 *   loss[0] = (1/B) sum_b cd_per_batch[b]  (computed in fp64, stored fp32)
 *   precision[b] = hits_xy / N, recall[b] = hits_yx / M, fscore[b] = 2PR/(P+R), 0 if P+R == 0 (R15).
 *   cd_per_batch, fscore, precision, recall may each be NULL; loss must not be NULL.
 */
CD_API cd_status cd_finalize(const double* partials, int B, int N, int M, float w1, float w2,
                      float* cd_per_batch, float* loss, float* fscore, float* precision,
                      float* recall, cd_stream_t stream);

/*
 * cd_fscore — F-score at radius tau from existing per-point distances (X = prediction,
 * Y = reference).  d_xy [B x N], d_yx [B x M] fp32 (as produced by cd_forward).
 *   Outputs fscore, precision, recall [B] fp32 (precision/recall may be NULL).  tau >= 0 required.
 */
CD_API cd_status cd_fscore(const float* d_xy, const float* d_yx, int B, int N, int M, float tau,
                    float* fscore, float* precision, float* recall,
                    void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_backward — VJP of the per-point distances with the argmin held fixed (
 * SURVEY.md §8.a.6-a.8):
 *   grad_x_i = 2 g_i (x_i - y_{a_i}) + sum_{j : b_j = i} 2 h_j (x_i - y_j)
 *   grad_y_j = 2 h_j (y_j - x_{b_j}) + sum_{i : a_i = j} 2 g_i (y_j - x_i)
 *   x, y: the clouds (full).  idx_xy [B x N], idx_yx [B x M]: FULL index arrays (all rows).
 *   g [B x N] (dL/dd_xy), h [B x M] (dL/dd_yx) fp32, FULL; either may be NULL, in which case the
 *   scalar g_scalar / h_scalar is used for every element (R8: the loss gradient is a fill).
 *   Output slices: grad_x rows [q0, q1) of every batch element, shape B x (q1-q0) x 3, and
 *   grad_y rows [r0, r1), B x (r1-r0) x 3.  Full problem: q0=0, q1=N, r0=0, r1=M.
 *   Each output element is accumulated in fp64: own term first, then the scatter terms in
 *   ascending source index (deterministic; no floating-point atomics), one fp32 write.
 *   Indices outside [0, M) / [0, N) are a precondition violation (results unspecified, no fault:
 *   they are clamped).
 */
CD_API cd_status cd_backward(const float* x, const float* y, int B, int N, int M,
                      const int32_t* idx_xy, const int32_t* idx_yx,
                      const float* g, const float* h, float g_scalar, float h_scalar,
                      int q0, int q1, int r0, int r1,
                      float* grad_x, float* grad_y,
                      void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_loss_backward — gradient of the batch loss that cd_finalize returns,
 *     L = (1/B) sum_b [ w1 (1/N) sum_i d_xy[b,i] + w2 (1/M) sum_j d_yx[b,j] ]   (R1)
 * times a DEVICE-resident upstream scalar u = grad_loss[0] (autograd's dL_total/dL), with the
 * argmin held fixed ("VJP holds the argmin fixed"; R8).  Equivalent to cd_backward with
 * the per-point upstreams filled with
 *     g = RN32(u * RN32(w1 / (B N))),   h = RN32(u * RN32(w2 / (B M)))
 * (RN32(w/(B P)) computed in fp64 and rounded once; the product rounded once in fp32), evaluated
 * inside the kernels: no B x N / B x M upstream array is materialised and u is read on the device,
 * so the call is asynchronous and graph-capturable.  Arguments, slices, outputs, workspace
 * (CD_OP_BACKWARD) and errors as cd_backward; grad_loss == NULL -> CD_ERR_INVALID_VALUE.
 */
CD_API cd_status cd_loss_backward(const float* x, const float* y, int B, int N, int M,
                      const int32_t* idx_xy, const int32_t* idx_yx,
                      const float* grad_loss, float w1, float w2,
                      int q0, int q1, int r0, int r1,
                      float* grad_x, float* grad_y,
                      void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_step_host — one whole training/evaluation step through HOST buffers (the end-to-end entry
 * point): copies x_host, y_host (pinned host memory recommended) into device staging inside the
 * workspace, runs cd_forward (full slices, tau) + cd_finalize + cd_backward of loss = mean_b CD_b
 * (g = w1/(B N), h = w2/(B M)), and copies back to host: loss_host[1], fscore_host[B] (may be NULL),
 * grad_x_host [B x N x 3] and grad_y_host [B x M x 3] (each may be NULL).  Asynchronous on stream:
 * the caller synchronises before reading host outputs.  Workspace: cd_workspace_size(CD_OP_STEP).
 */
CD_API cd_status cd_step_host(const float* x_host, const float* y_host, int B, int N, int M,
                       float tau, float w1, float w2,
                       float* loss_host, float* fscore_host, float* grad_x_host, float* grad_y_host,
                       void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_sample_mesh — differentiable surface sampling, the step before the Chamfer path
 * ("differentiable surface sampling ... by
 * application of the reparameterization trick").  B meshes sharing one topology:
 *   verts [B x Nv x 3] fp32, faces [Nf x 3] int32 (vertex indices, clamped to [0, Nv) if outside);
 *   random inputs (drawn by the caller): r_face [B x N] uint32, r_bary [B x N x 2] fp32 in [0, 1).
 *   Face choice with probability proportional to area, as an exact integer decision (R19):
 *     area_f in fp64 (fixed op order), q_f = floor(area_f * 2^k), k = 52 - e with
 *     Nf * max_f area_f = m 2^e (m in [0.5,1)); P = inclusive prefix of q; t = (r_face * P_last) >> 32;
 *     face = min { f : P_f > t } (face 0 when every area is 0).
 *   Barycentrics (R20): s = sqrt(r1), w = (1 - s, s (1 - r2), s r2) in fp32 .rn;
 *   point = (w0 v_a + w1 v_b) + w2 v_c (fp32 .rn, R21).
 *   Outputs: points [B x N x 3], face_idx [B x N], bary [B x N x 3] (may be NULL; needed by the
 *   backward).  Workspace: cd_sample_workspace_size(CD_OP_SAMPLE, ...).
 * cd_sample_mesh_backward — VJP with the face choice and weights fixed (R22):
 *   grad_verts[b, v] = sum over (sample i, corner k) with faces[face_i][k] == v of
 *   bary[i][k] * grad_points[i], accumulated in fp64 in ascending (i, k) order (stable radix sort,
 *   no floating-point atomics); grad_verts [B x Nv x 3] is fully written (0 for unsampled vertices).
 */
CD_API cd_status cd_sample_mesh(const float* verts, const int32_t* faces, int B, int Nv, int Nf, int N,
                         const uint32_t* r_face, const float* r_bary,
                         float* points, int32_t* face_idx, float* bary,
                         void* workspace, size_t workspace_bytes, cd_stream_t stream);
CD_API cd_status cd_sample_mesh_backward(const int32_t* faces, const int32_t* face_idx, const float* bary,
                         int B, int Nv, int Nf, int N, const float* grad_points, float* grad_verts,
                         void* workspace, size_t workspace_bytes, cd_stream_t stream);
CD_API size_t cd_sample_workspace_size(int op, int B, int Nv, int Nf, int N);
CD_API int cd_sample_launch_count(int op, int B, int Nv, int Nf, int N);

/*
 * cd_p2s_forward — point-to-surface loss ("the point-to-surface
 * loss [GEOMetrics] for Meshes").  points [B x N x 3], verts [B x Nv x 3] fp32,
 * faces [Nf x 3] int32 shared by the B meshes.  Per point (brute force over all faces):
 *   d[b,i] = min_f dist^2(p, triangle f), face[b,i] = lowest f attaining the fp32 minimum of the hot
 *   loop's formulation (R24: plane distance when the projection is inside, else the nearest
 *   edge); d, closest [B x N x 3] and bary [B x N x 3] (barycentrics of the closest point on that
 *   face) are then evaluated in fp64 with the region decomposition and stored as fp32.
 *   per_batch[b] = mean_i d (may be NULL), loss[0] = mean_b per_batch (may be NULL).
 *   closest / bary may be NULL (both are needed by the backward).
 * cd_p2s_backward — VJP of sum_i g_i d_i with the closest point fixed (R25):
 *   grad_points = 2 g (p - c) [B x N x 3] (may be NULL); grad_verts [B x Nv x 3] (may be NULL) =
 *   sum over (point, corner) of bary * (-2 g (p - c)) through the deterministic vertex scatter of
 *   cd_sample_mesh_backward.  g [B x N] or NULL (then g_scalar for every point).
 */
CD_API cd_status cd_p2s_forward(const float* points, const float* verts, const int32_t* faces,
                         int B, int N, int Nv, int Nf, float* d, int32_t* face, float* closest,
                         float* bary, float* per_batch, float* loss,
                         void* workspace, size_t workspace_bytes, cd_stream_t stream);
CD_API cd_status cd_p2s_backward(const float* points, const float* closest, const int32_t* face,
                         const float* bary, const int32_t* faces, int B, int N, int Nv, int Nf,
                         const float* g, float g_scalar, float* grad_points, float* grad_verts,
                         void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_p2s_loss_backward — gradient of the point-to-surface loss cd_p2s_forward returns,
 * L = (1/B) sum_b (1/N) sum_i d[b,i] (R23), times the DEVICE-resident upstream scalar
 * u = grad_loss[0]: cd_p2s_backward with g = RN32(u * RN32(1 / (B N))) for every point, formed in the
 * kernel (no B x N upstream array).  Other arguments, workspace and errors as cd_p2s_backward.
 */
CD_API cd_status cd_p2s_loss_backward(const float* points, const float* closest, const int32_t* face,
                         const float* bary, const int32_t* faces, int B, int N, int Nv, int Nf,
                         const float* grad_loss, float* grad_points, float* grad_verts,
                         void* workspace, size_t workspace_bytes, cd_stream_t stream);
CD_API size_t cd_p2s_workspace_size(int op, int B, int N, int Nv, int Nf);
CD_API int cd_p2s_launch_count(int op, int B, int N, int Nv, int Nf);

/*
 * cd_p2s_forward_pruned — cd_p2s_forward with culling (R26): points and face centroids
 * are Hilbert-sorted per batch element; 64-point query tiles visit 64-face tiles in ascending order
 * of a box lower bound and stop once the bound exceeds every point's current minimum; tiles and
 * 32-face blocks no lane can improve on are skipped.  Boxes are widened by 2^-14 max|coord| so that the bound also
 * holds for the fp32-evaluated distances of the hot loop (R26): the minimum is the brute force's.
 * Same arguments, outputs and tie rule as cd_p2s_forward (the lowest face index among EXACTLY equal
 * fp32 minima): a block whose minimum equals the current one flags the point (also across the
 * culling's chunks, through the value atomicMin returns), and flagged points re-walk their
 * candidate tiles for the lowest original index at the minimum (R3').  Outputs are bit-identical to
 * cd_p2s_forward's.  Workspace: cd_p2s_workspace_size(CD_OP_P2S_PRUNED, ...); 0 = unsupported
 * size (Nf > 524288, B*(N+Nf) >= 2^31, or per-query-tile candidate lists B*ceil(N/64)*ceil(Nf/64)*8
 * bytes > 4 GiB) and the call returns CD_ERR_TOO_LARGE.
 */
CD_API cd_status cd_p2s_forward_pruned(const float* points, const float* verts, const int32_t* faces,
                         int B, int N, int Nv, int Nf, float* d, int32_t* face, float* closest,
                         float* bary, float* per_batch, float* loss,
                         void* workspace, size_t workspace_bytes, cd_stream_t stream);

/*
 * cd_step_host_overlapped — cd_step_host with the host<->device copies overlapped with the compute:
 * the clouds are copied in `nchunks` batch ranges on `copy_stream` (the first range half an equal
 * share, max(1, B / (2 nchunks)) elements, since only its copy is exposed; with nchunks >= 3 the
 * last range is as short, since only its backward and gradient copy are exposed; the rest split
 * equally).  Range c computes on `stream` (c even) or `stream2` (c odd; stream2 == NULL: every range
 * on `stream`), so a range's forward fills the SMs the previous range's last wave leaves idle; its
 * forward starts as soon as range c has landed (cudaStreamWaitEvent) and its loss backward follows
 * at once (the fills w/(B P) use the whole batch's B and do not depend on the loss value; each batch
 * element's gradients depend only on its own clouds and indices), and range c's gradients go back
 * on `copy_stream` while later ranges compute; `stream` then joins `stream2`, runs finalize and the
 * loss / F-score copies, and finally waits for the gradient copies.  Results are identical to cd_step_host (per-batch outputs do not depend on the
 * chunking).  events: nchunks + 1 cudaEvent_t created by the caller (disable-timing events are
 * fine); the copy stream and stream2 first wait for everything already queued on `stream`
 * (events[nchunks] recorded there: the previous step's staging buffers are free) and join `stream`
 * again before the step ends, so the call can be captured in a CUDA graph and replayed (static
 * pointers and sizes).  nchunks in [1, B].  Workspace: cd_workspace_size(CD_OP_STEP) (it holds a
 * scratch region per compute stream).
 */
CD_API cd_status cd_step_host_overlapped(const float* x_host, const float* y_host, int B, int N, int M,
                       float tau, float w1, float w2,
                       float* loss_host, float* fscore_host, float* grad_x_host, float* grad_y_host,
                       int nchunks, void* workspace, size_t workspace_bytes,
                       cd_stream_t stream, cd_stream_t copy_stream, cd_stream_t stream2,
                       void* const* events);

/* Workspace bytes needed by an operation for these sizes (full slices).  0 on invalid sizes. */
CD_API size_t cd_workspace_size(int op, int B, int N, int M);

/* Number of kernel launches one call of `op` makes for these sizes (for launch accounting). */
CD_API int cd_launch_count(int op, int B, int N, int M);

CD_API const char* cd_status_string(cd_status s);
CD_API const char* cd_last_error_string(void);   /* thread-local; "" when no error */
CD_API int cd_abi_version(void);                 /* == CD_ABI_VERSION */

/*
 * Tuning / test hooks (not needed for normal use).  cd_set_forward_splits forces the target-split
 * count (0 = automatic) of the forward kernels and of the brute-force point-to-surface kernel for
 * the calling thread, so tests can check that results are independent of the tiling (DESIGN.md
 * §4.4) and sweeps can fit the split model (§4.3).  Workspace sizes queried afterwards follow the
 * forced count.  Returns the previous value.
 */
CD_API int cd_set_forward_splits(int splits);

/*
 * Measurement hook: when start/stop are non-NULL cudaEvent_t handles, every subsequent cd_forward
 * on the calling thread records `start` immediately before and `stop` immediately after its
 * nearest-neighbour kernel (nn_fwd_kernel), on the call's stream, so a benchmark can time the
 * dominant kernel alone.  Pass NULL, NULL to disable.
 */
CD_API void cd_set_profile_events(void* start, void* stop);

/*
 * Test hook: forward kernel selection for cd_forward on the calling thread.  0 = automatic (the
 * fused bidirectional kernel for full problems, the per-direction kernel for query slices),
 * 1 = always the per-direction kernel, 2 = the fused kernel (full problems), 3 = the tensor-core
 * filter + exact re-scan forward (nn_tc.cu, R27; full problems).  Returns the
 * previous value.  All produce bit-identical outputs.  Mode 3's workspace
 * (per-(128-row query block, column) summaries: ~N*M/8 bytes per batch element) is part of
 * cd_workspace_size(CD_OP_FORWARD / CD_OP_STEP) only while mode 3 is selected; a mode-3 call with a
 * smaller workspace returns CD_ERR_TOO_LARGE before any launch.
 */
CD_API int cd_set_forward_mode(int mode);

#ifdef __cplusplus
}
#endif
#endif /* CD_H_ */
