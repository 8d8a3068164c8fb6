"""Shared parity gates for the GPU tests (readings R12-R16; BASELINE.json north_star
correctness gate): indices bit-exact where the oracle's top-2 gap exceeds 1e-6 relative, otherwise
an accepted near-tie; distances / losses within 1e-5 relative; gradients within 1e-5 of the
oracle's condition scale S = sum |terms|."""
import numpy as np

import oracle

RTOL = 1e-5          # distances, losses, gradients (north_star)
GAP = 1e-6           # top-2 relative gap above which indices must be bit-exact (north_star)


def sqdist64(q, t, idx):
    """fp64 squared distance of rows q (n,3) to t[idx] (n,3)."""
    d = q.astype(np.float64) - t[idx].astype(np.float64)
    return (d * d).sum(axis=1)


def gate_nn(q, t, d_gpu, i_gpu, d1, i1, d2):
    """q: (n,3) queries, t: (M,3) targets of ONE batch element (or flattened rows with per-row t);
    d1/i1/d2 oracle results for those rows."""
    d_gpu = np.asarray(d_gpu, np.float64)
    i_gpu = np.asarray(i_gpu)
    # distances within 1e-5 relative; exact zero must be exact
    zero = d1 == 0
    assert np.all(d_gpu[zero] == 0), "exact zero distance not reproduced"
    rel = np.abs(d_gpu[~zero] - d1[~zero]) / d1[~zero]
    assert rel.size == 0 or rel.max() <= RTOL, f"distance rel err {rel.max():.3g}"
    clear = np.where(d1 == 0, d2 > 0, (d2 - d1) > GAP * d1)
    bad = clear & (i_gpu != i1)
    assert not bad.any(), f"{bad.sum()} index mismatches where gap > {GAP}"
    amb = ~clear
    if amb.any():
        assert np.all(i_gpu[amb] >= 0)
        e = sqdist64(q[amb], t, i_gpu[amb]) if t.ndim == 2 else None
        if e is not None:
            assert np.all(e <= d1[amb] * (1 + GAP) + (d1[amb] == 0) * 0.0), "near-tie index not a near-minimum"
    return clear.mean()


def gate_forward_batch(X, Y, d_xy, i_xy, d_yx, i_yx, rows_x=None, rows_y=None):
    """Compare a (possibly row-sampled) GPU forward against the fp64 oracle, per batch element."""
    B, N, _ = X.shape
    M = Y.shape[1]
    for (Q, T, d, i, rows) in ((X, Y, d_xy, i_xy, rows_x), (Y, X, d_yx, i_yx, rows_y)):
        P = Q.shape[1]
        if rows is None:
            rows = np.arange(B * P)
        d1, i1, d2 = oracle.nn(Q, T, rows=rows)
        bsel = rows // P
        for b in np.unique(bsel):
            m = bsel == b
            r = rows[m] % P
            gate_nn(Q[b][r], T[b], np.asarray(d).reshape(B, P)[b][r], np.asarray(i).reshape(B, P)[b][r],
                    d1[m], i1[m], d2[m])


def gate_mirror(X, Y, d_xy, i_xy, rows=None):
    """Bit-exact check against the fp32 mirror of DESIGN.md §4.2's op order (stricter than the gate)."""
    B, N, _ = X.shape
    dm, im = oracle.mirror_nn_f32(X, Y, rows=rows)
    d = np.asarray(d_xy).reshape(-1)
    i = np.asarray(i_xy).reshape(-1)
    if rows is not None:
        d, i = d[rows], i[rows]
    else:
        dm, im = dm.reshape(-1), im.reshape(-1)
    np.testing.assert_array_equal(d.view(np.uint32), dm.view(np.uint32))
    np.testing.assert_array_equal(i, im)


def gate_grad(g_gpu, g_ref, s_ref):
    """|gpu - ref| <= 1e-5 * S elementwise (R14), plus the headline relative L2 error."""
    g_gpu = np.asarray(g_gpu, np.float64)
    err = np.abs(g_gpu - g_ref)
    tol = RTOL * s_ref + 1e-38
    assert np.all(err <= tol), f"grad err max {np.max(err / np.maximum(s_ref, 1e-38)):.3g} of S"
    n = np.linalg.norm(g_ref)
    if n > 0:
        assert np.linalg.norm(g_gpu - g_ref) / n <= RTOL
