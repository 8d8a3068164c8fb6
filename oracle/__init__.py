"""CPU oracle for batched Chamfer / nearest-neighbour / F-score (fp64).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The product package
``paper_1911_05063_b200`` never imports it, and it never imports the product package: the two
share no code.  Inputs come from the seeded generators in ``paper_1911_05063_b200.synth``
(which hold none of the method's arithmetic).

Every function follows a plain definition, cited:

* ``nn``        — SPEC.md:441 (metrics/chamfer_distance, brute force) for PAPER.md:253-254 (§2.5):
                  per-query min squared distance, lowest-index argmin, second-nearest value.
* ``chamfer``   — SPEC.md:441: CD_b = w1 * mean_i d_xy + w2 * mean_j d_yx (R1, R2);
                  batch loss = mean_b CD_b (R1).  Sums use ``math.fsum`` (exactly
                  rounded), so the loss is the definition up to one final rounding.
* ``fscore``    — DESIGN.md §3.3 (R11, R15, R16): hit iff (double)d <= (double)tau_f32^2;
                  P = hits_xy / N, R = hits_yx / M, F = 2PR/(P+R), F = 0 if P+R = 0.
                  PARITY UNPINNED against the paper (the paper never defines an F-score);
                  pinned only to the stated definition and hand examples.
* ``backward``  — SPEC.md:441 "VJP holds the argmin fixed": see oracle_backward in
                  chamfer_oracle.c.
* ``sample_mesh`` / ``sample_vjp`` — NEXT-4 ("differentiable
                  surface sampling ... reparameterization trick"): area-proportional face choice with
                  an exact integer CDF (R19), square-root barycentrics (R20),
                  points (R21) and the VJP with choices fixed (R22), fp64.
* ``p2s`` / ``p2s_loss`` — NEXT-3 point-to-surface ("the point-to-surface loss [GEOMetrics]
                  for Meshes"): closest triangle by brute force with the region
                  decomposition of the closest point, loss = mean_b mean_i d, VJP 2 g (p - closest)
                  w.r.t. the points and, through the closest point's barycentrics, w.r.t. the vertices
                  (R23-R25).
* ``mirror_nn_f32`` — not the oracle; fp32 re-evaluation of DESIGN.md §4.2's fixed op order,
                  used to check GPU distance bits.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "chamfer_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (the checker; building it is not using it)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            i64, i32p, f64p, f32p, i64p = (ctypes.c_int64, ctypes.POINTER(ctypes.c_int32),
                                           ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_float),
                                           ctypes.POINTER(ctypes.c_int64))
            lib.oracle_nn.argtypes = [f64p, f64p, i64, i64, i64, i64p, i64, f64p, i32p, f64p, ctypes.c_int]
            lib.oracle_nn.restype = ctypes.c_int
            lib.oracle_backward.argtypes = [f64p, f64p, i64, i64, i64, i32p, i32p, f64p, f64p,
                                            ctypes.c_double, ctypes.c_double, f64p, f64p, f64p, f64p]
            lib.oracle_backward.restype = ctypes.c_int
            lib.mirror_nn_f32.argtypes = [f32p, f32p, i64, i64, i64, i64p, i64, f32p, i32p, ctypes.c_int]
            lib.mirror_nn_f32.restype = ctypes.c_int
            lib.oracle_max_threads.restype = ctypes.c_int
            u32p, u64p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)
            lib.oracle_sample_mesh.argtypes = [f32p, i32p, i64, i64, i64, i64, u32p, f32p, f64p, i32p, f64p, u64p]
            lib.oracle_sample_mesh.restype = ctypes.c_int
            lib.oracle_sample_vjp.argtypes = [f64p, i32p, i32p, i64, i64, i64, i64, f64p, f64p]
            lib.oracle_sample_vjp.restype = ctypes.c_int
            lib.oracle_p2s.argtypes = [f32p, f32p, i32p, i64, i64, i64, i64, i64p, i64, f64p, i32p, f64p, f64p, f64p,
                                       ctypes.c_int]
            lib.oracle_p2s.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _cloud64(a) -> np.ndarray:
    a = np.asarray(a)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3 or a.shape[-1] != 3:
        raise ValueError(f"expected (B, P, 3) cloud, got shape {a.shape}")
    return np.ascontiguousarray(a, dtype=np.float64)


def nn(q, t, rows=None, nthreads: int = 0):
    """Directed NN of q (B,N,3) against t (B,M,3) in fp64 (R2-R4, R12).

    rows: optional 1-D array of flattened query rows (b*N + i).  Returns (d1, i1, d2) shaped
    (B, N) when rows is None, else (len(rows),)."""
    q64, t64 = _cloud64(q), _cloud64(t)
    B, N, _ = q64.shape
    Bt, M, _ = t64.shape
    if Bt != B:
        raise ValueError("batch mismatch")
    if N < 1 or M < 1:
        raise ValueError("empty cloud (SPEC.md:440-442: domain error)")
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        n = rows.shape[0]
    else:
        n = B * N
    d1 = np.empty(n, np.float64)
    i1 = np.empty(n, np.int32)
    d2 = np.empty(n, np.float64)
    rc = _load().oracle_nn(_ptr(q64, ctypes.c_double), _ptr(t64, ctypes.c_double), B, N, M,
                           _ptr(rows, ctypes.c_int64), n if rows is not None else 0,
                           _ptr(d1, ctypes.c_double), _ptr(i1, ctypes.c_int32), _ptr(d2, ctypes.c_double),
                           int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_nn failed rc={rc}")
    if rows is None:
        return d1.reshape(B, N), i1.reshape(B, N), d2.reshape(B, N)
    return d1, i1, d2


def chamfer(x, y, w1: float = 1.0, w2: float = 1.0, tau=None, nthreads: int = 0):
    """Full bidirectional Chamfer forward (+ optional F-score) in fp64.

    Returns a dict with d_xy, idx_xy, d2_xy (B,N), d_yx, idx_yx, d2_yx (B,M), cd (B,),
    loss (float) and, when tau is given, fscore/precision/recall (B,) and hits."""
    x64, y64 = _cloud64(x), _cloud64(y)
    d_xy, i_xy, s_xy = nn(x64, y64, nthreads=nthreads)
    d_yx, i_yx, s_yx = nn(y64, x64, nthreads=nthreads)
    cd, loss = chamfer_loss(d_xy, d_yx, w1, w2)
    out = dict(d_xy=d_xy, idx_xy=i_xy, d2_xy=s_xy, d_yx=d_yx, idx_yx=i_yx, d2_yx=s_yx, cd=cd, loss=loss)
    if tau is not None:
        out.update(fscore(d_xy, d_yx, tau))
    return out


def chamfer_loss(d_xy, d_yx, w1: float = 1.0, w2: float = 1.0):
    """CD_b = w1 * (1/N) sum_i d_xy[b,i] + w2 * (1/M) sum_j d_yx[b,j]; loss = (1/B) sum_b CD_b.

    SPEC.md:441 (mean + mean of squared NN distances), R1; fsum = exactly rounded sums."""
    d_xy = np.asarray(d_xy, np.float64)
    d_yx = np.asarray(d_yx, np.float64)
    B, N = d_xy.shape
    _, M = d_yx.shape
    cd = np.array([w1 * (math.fsum(d_xy[b].tolist()) / N) + w2 * (math.fsum(d_yx[b].tolist()) / M)
                   for b in range(B)], np.float64)
    loss = math.fsum(cd.tolist()) / B
    return cd, loss


def tau_sq(tau) -> float:
    """tau is an fp32 Euclidean radius; tau^2 evaluated exactly in fp64 (R11)."""
    t = float(np.float32(tau))
    return t * t


def fscore(d_xy, d_yx, tau):
    """F-score at radius tau (R11, R15, R16).  X = prediction, Y = reference.

    hits_xy = #{i : d_xy <= tau^2}, P = hits_xy / N; hits_yx = #{j : d_yx <= tau^2}, R = hits_yx / M;
    F = 2PR / (P + R), F = 0 when P + R = 0 (no epsilon).  PARITY UNPINNED w.r.t. the paper."""
    t2 = tau_sq(tau)
    d_xy = np.asarray(d_xy, np.float64)
    d_yx = np.asarray(d_yx, np.float64)
    N, M = d_xy.shape[1], d_yx.shape[1]
    hx = (d_xy <= t2).sum(axis=1).astype(np.int64)
    hy = (d_yx <= t2).sum(axis=1).astype(np.int64)
    P = hx / N
    R = hy / M
    F = np.where(P + R > 0, 2.0 * P * R / np.where(P + R > 0, P + R, 1.0), 0.0)
    return dict(fscore=F, precision=P, recall=R, hits_xy=hx, hits_yx=hy)


def fscore_from_hits(hits_xy, hits_yx, N, M):
    """F from given hit counts (used to evaluate the oracle F at the GPU's counts, R16)."""
    P = np.asarray(hits_xy, np.float64) / N
    R = np.asarray(hits_yx, np.float64) / M
    return np.where(P + R > 0, 2.0 * P * R / np.where(P + R > 0, P + R, 1.0), 0.0)


def backward(x, y, idx_xy, idx_yx, g=None, h=None, g_scalar: float = 0.0, h_scalar: float = 0.0):
    """VJP with the argmin held fixed, fp64.  Returns (grad_x, grad_y, sx, sy).

    g (B,N) / h (B,M) upstream cotangents of d_xy / d_yx, or None to use the scalars."""
    x64, y64 = _cloud64(x), _cloud64(y)
    B, N, _ = x64.shape
    _, M, _ = y64.shape
    ixy = np.ascontiguousarray(idx_xy, np.int32).reshape(B, N)
    iyx = np.ascontiguousarray(idx_yx, np.int32).reshape(B, M)
    g64 = None if g is None else np.ascontiguousarray(g, np.float64).reshape(B, N)
    h64 = None if h is None else np.ascontiguousarray(h, np.float64).reshape(B, M)
    gx = np.empty((B, N, 3), np.float64)
    gy = np.empty((B, M, 3), np.float64)
    sx = np.empty((B, N, 3), np.float64)
    sy = np.empty((B, M, 3), np.float64)
    rc = _load().oracle_backward(_ptr(x64, ctypes.c_double), _ptr(y64, ctypes.c_double), B, N, M,
                                 _ptr(ixy, ctypes.c_int32), _ptr(iyx, ctypes.c_int32),
                                 _ptr(g64, ctypes.c_double), _ptr(h64, ctypes.c_double),
                                 float(g_scalar), float(h_scalar),
                                 _ptr(gx, ctypes.c_double), _ptr(gy, ctypes.c_double),
                                 _ptr(sx, ctypes.c_double), _ptr(sy, ctypes.c_double))
    if rc != 0:
        raise ValueError(f"oracle_backward failed rc={rc}")
    return gx, gy, sx, sy


def loss_grad(x, y, idx_xy, idx_yx, w1: float = 1.0, w2: float = 1.0):
    """Gradient of loss = mean_b CD_b: upstream g = w1/(B*N), h = w2/(B*M) (R8)."""
    x64, y64 = _cloud64(x), _cloud64(y)
    B, N, _ = x64.shape
    M = y64.shape[1]
    return backward(x64, y64, idx_xy, idx_yx, g_scalar=w1 / (B * N), h_scalar=w2 / (B * M))


def mirror_nn_f32(q, t, rows=None, nthreads: int = 0):
    """fp32 re-evaluation of DESIGN.md §4.2's op order (see chamfer_oracle.c).  Returns (d, idx)."""
    q32 = np.ascontiguousarray(q, np.float32)
    t32 = np.ascontiguousarray(t, np.float32)
    if q32.ndim == 2:
        q32, t32 = q32[None], t32[None]
    B, N, _ = q32.shape
    M = t32.shape[1]
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        n = rows.shape[0]
    else:
        n = B * N
    d = np.empty(n, np.float32)
    idx = np.empty(n, np.int32)
    rc = _load().mirror_nn_f32(_ptr(q32, ctypes.c_float), _ptr(t32, ctypes.c_float), B, N, M,
                               _ptr(rows, ctypes.c_int64), n if rows is not None else 0,
                               _ptr(d, ctypes.c_float), _ptr(idx, ctypes.c_int32), int(nthreads))
    if rc != 0:
        raise ValueError(f"mirror_nn_f32 failed rc={rc}")
    if rows is None:
        return d.reshape(B, N), idx.reshape(B, N)
    return d, idx


def sample_mesh(verts, faces, r_face, r_bary):
    """NEXT-4 forward (R19-R21).  verts (B,Nv,3) fp32, faces (Nf,3) int32, r_face (B,N) uint32,
    r_bary (B,N,2) fp32 uniforms.  Returns (points fp64 (B,N,3), face_idx (B,N), bary fp64 (B,N,3),
    cdf uint64 (B,Nf))."""
    v = np.ascontiguousarray(verts, np.float32)
    f = np.ascontiguousarray(faces, np.int32)
    rf = np.ascontiguousarray(r_face, np.uint32)
    rb = np.ascontiguousarray(r_bary, np.float32)
    B, Nv, _ = v.shape
    Nf = f.shape[0]
    N = rf.shape[1]
    pts = np.empty((B, N, 3), np.float64)
    fi = np.empty((B, N), np.int32)
    bary = np.empty((B, N, 3), np.float64)
    cdf = np.empty((B, Nf), np.uint64)
    rc = _load().oracle_sample_mesh(_ptr(v, ctypes.c_float), _ptr(f, ctypes.c_int32), B, Nv, Nf, N,
                                    _ptr(rf, ctypes.c_uint32), _ptr(rb, ctypes.c_float), _ptr(pts, ctypes.c_double),
                                    _ptr(fi, ctypes.c_int32), _ptr(bary, ctypes.c_double), _ptr(cdf, ctypes.c_uint64))
    if rc != 0:
        raise ValueError(f"oracle_sample_mesh failed rc={rc}")
    return pts, fi, bary, cdf


def sample_vjp(bary, face_idx, faces, Nv, grad_points):
    """NEXT-4 VJP (R22): grad w.r.t. the vertices of sum(grad_points * points), choices fixed."""
    ba = np.ascontiguousarray(bary, np.float64)
    fi = np.ascontiguousarray(face_idx, np.int32)
    f = np.ascontiguousarray(faces, np.int32)
    g = np.ascontiguousarray(grad_points, np.float64)
    B, N, _ = ba.shape
    out = np.empty((B, Nv, 3), np.float64)
    rc = _load().oracle_sample_vjp(_ptr(ba, ctypes.c_double), _ptr(fi, ctypes.c_int32), _ptr(f, ctypes.c_int32), B, Nv,
                                   f.shape[0], N, _ptr(g, ctypes.c_double), _ptr(out, ctypes.c_double))
    if rc != 0:
        raise ValueError(f"oracle_sample_vjp failed rc={rc}")
    return out


def p2s(points, verts, faces, rows=None, nthreads: int = 0):
    """NEXT-3: per point min squared distance to the mesh (B,N), face (lowest on ties), second-best d,
    closest point (B,N,3) and its barycentrics (B,N,3) — fp64 brute force."""
    P = np.ascontiguousarray(points, np.float32)
    V = np.ascontiguousarray(verts, np.float32)
    F = np.ascontiguousarray(faces, np.int32)
    B, N, _ = P.shape
    Nv = V.shape[1]
    Nf = F.shape[0]
    if rows is not None:
        rows = np.ascontiguousarray(rows, np.int64)
        n = rows.shape[0]
    else:
        n = B * N
    d = np.empty(n, np.float64)
    fi = np.empty(n, np.int32)
    d2 = np.empty(n, np.float64)
    cl = np.empty((n, 3), np.float64)
    la = np.empty((n, 3), np.float64)
    rc = _load().oracle_p2s(_ptr(P, ctypes.c_float), _ptr(V, ctypes.c_float), _ptr(F, ctypes.c_int32), B, N, Nv, Nf,
                            _ptr(rows, ctypes.c_int64), n if rows is not None else 0, _ptr(d, ctypes.c_double),
                            _ptr(fi, ctypes.c_int32), _ptr(d2, ctypes.c_double), _ptr(cl, ctypes.c_double),
                            _ptr(la, ctypes.c_double), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_p2s failed rc={rc}")
    if rows is None:
        return d.reshape(B, N), fi.reshape(B, N), d2.reshape(B, N), cl.reshape(B, N, 3), la.reshape(B, N, 3)
    return d, fi, d2, cl, la


def p2s_loss(d):
    """loss = mean_b mean_i d ("mean over points", batch mean as R1)."""
    d = np.asarray(d, np.float64)
    return math.fsum((math.fsum(row.tolist()) / d.shape[1] for row in d)) / d.shape[0]


def p2s_grads(points, verts, faces, face, closest, lam, g):
    """VJP of sum_i g_i d_i with the closest point held fixed: grad_p = 2 g (p - c);
    grad_v = sum over (point, corner) of -2 g (p - c) lam_k (R25).  Returns (grad_p, grad_v) fp64."""
    P = np.asarray(points, np.float64)
    g = np.asarray(g, np.float64)
    diff = P - np.asarray(closest, np.float64)
    gp = 2.0 * g[..., None] * diff
    gv = sample_vjp(np.asarray(lam, np.float64), face, faces, np.asarray(verts).shape[1], -gp)
    return gp, gv
