"""Pins for the NEXT-4 oracle (differentiable surface sampling) — no GPU.
Statistical and closed-form facts the paper/SPEC fix (area-proportional faces, uniform points per
triangle, simplex weights, vertex-corner gradients, finite differences), never the oracle itself."""
import numpy as np
import pytest

import oracle
from paper_1911_05063_b200 import synth


def _rand(B, N, seed):
    return synth.sampling_randoms(B, N, seed=seed)


def test_single_triangle_all_face0_in_simplex():
    # SPEC.md:233 "single triangle, any seed -> all face_indices = 0, points inside the triangle"
    V = np.array([[[0, 0, 0], [1, 0, 0], [0, 2, 0]]], np.float32)
    F = np.array([[0, 1, 2]], np.int32)
    rf, rb = _rand(1, 5000, 1)
    p, fi, ba, _ = oracle.sample_mesh(V, F, rf, rb)
    assert np.all(fi == 0)
    assert np.all(ba >= 0) and np.allclose(ba.sum(-1), 1.0, atol=1e-15)
    assert np.all(p[..., 0] >= 0) and np.all(p[..., 1] >= 0) and np.all(2 * p[..., 0] + p[..., 1] <= 2 + 1e-12)


def test_area_ratio_3_to_1():
    # SPEC.md:234 "two triangles with area ratio 3:1, n = 100k -> face-0 fraction = 0.75 within 0.01"
    V = np.array([[[0, 0, 0], [3, 0, 0], [0, 1, 0], [10, 0, 0], [11, 0, 0], [10, 1, 0]]], np.float32)
    F = np.array([[0, 1, 2], [3, 4, 5]], np.int32)
    rf, rb = _rand(1, 100000, 2)
    _, fi, _, _ = oracle.sample_mesh(V, F, rf, rb)
    frac = (fi == 0).mean()
    sigma = np.sqrt(0.75 * 0.25 / 1e5)
    assert abs(frac - 0.75) < 6 * sigma


def test_unit_square_mean():
    # SPEC.md:235 "unit-square mesh (2 triangles), n = 100k -> sample mean -> (0.5, 0.5, 0) within 0.005"
    V = np.array([[[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]]], np.float32)
    F = np.array([[0, 1, 2], [0, 2, 3]], np.int32)
    rf, rb = _rand(1, 100000, 3)
    p, _, _, _ = oracle.sample_mesh(V, F, rf, rb)
    np.testing.assert_allclose(p[0].mean(0), [0.5, 0.5, 0.0], atol=0.005)


def test_triangle_moments_uniform():
    # uniform density on a triangle: E[p] = centroid, E[(p-c)(p-c)^T] = known closed form
    A, Bv, C = np.array([0., 0, 0]), np.array([2., 0, 0]), np.array([0., 1, 0])
    V = np.array([[A, Bv, C]], np.float32)
    F = np.array([[0, 1, 2]], np.int32)
    rf, rb = _rand(1, 200000, 4)
    p, _, _, _ = oracle.sample_mesh(V, F, rf, rb)
    c = (A + Bv + C) / 3
    np.testing.assert_allclose(p[0].mean(0), c, atol=4e-3)
    # covariance of the uniform distribution on a triangle: (1/12) sum_i (v_i - c)(v_i - c)^T
    cov = sum(np.outer(v - c, v - c) for v in (A, Bv, C)) / 12.0
    np.testing.assert_allclose(np.cov(p[0].T), cov, atol=3e-3)


def test_face_frequencies_proportional_to_area():
    V, F = synth.mesh_batch(1, subdiv=2)
    rf, rb = _rand(1, 400000, 5)
    _, fi, _, _ = oracle.sample_mesh(V, F, rf, rb)
    v = V[0].astype(np.float64)
    area = 0.5 * np.linalg.norm(np.cross(v[F[:, 1]] - v[F[:, 0]], v[F[:, 2]] - v[F[:, 0]]), axis=1)
    p = area / area.sum()
    counts = np.bincount(fi[0], minlength=F.shape[0])
    expect = p * fi.size
    chi2 = ((counts - expect) ** 2 / expect).sum()
    dof = F.shape[0] - 1
    assert chi2 < dof + 6 * np.sqrt(2 * dof)


def test_zero_area_faces_never_chosen_and_monotone_in_r():
    V = np.array([[[0, 0, 0], [1, 0, 0], [0, 1, 0], [2, 2, 2], [2, 2, 2], [3, 3, 3]]], np.float32)
    F = np.array([[3, 4, 5], [0, 1, 2], [3, 4, 5], [0, 2, 1]], np.int32)   # faces 0, 2 degenerate
    r = np.sort(np.random.default_rng(0).integers(0, 2 ** 32, size=(1, 3000), dtype=np.uint64)).astype(np.uint32)
    _, fi, _, cdf = oracle.sample_mesh(V, F, r, _rand(1, 3000, 6)[1])
    assert set(np.unique(fi)) <= {1, 3}
    assert np.all(np.diff(fi[0]) >= 0)                      # larger r -> later (or equal) face
    assert cdf[0, 0] == 0 and cdf[0, 1] == cdf[0, 2]


def test_points_are_barycentric_combinations():
    V, F = synth.mesh_batch(2, subdiv=3)
    rf, rb = _rand(2, 3000, 7)
    p, fi, ba, _ = oracle.sample_mesh(V, F, rf, rb)
    for b in range(2):
        corners = V[b][F[fi[b]]].astype(np.float64)          # (N, 3, 3)
        np.testing.assert_allclose(p[b], (ba[b][:, :, None] * corners).sum(1), rtol=0, atol=1e-15)
    # SPEC.md:231 square-root barycentrics
    s = np.sqrt(rb[..., 0].astype(np.float64))
    np.testing.assert_allclose(ba[..., 0], 1 - s, atol=0)
    np.testing.assert_allclose(ba[..., 2], s * rb[..., 1], atol=0)


def test_vjp_examples_and_finite_differences():
    V, F = synth.mesh_batch(1, subdiv=1)
    Nv = V.shape[1]
    rf, rb = _rand(1, 200, 8)
    rb[0, 0] = [0.0, 0.3]                                  # r1 = 0 -> weights (1, 0, 0): sample at corner 0
    p, fi, ba, _ = oracle.sample_mesh(V, F, rf, rb)
    # SPEC.md:242 upstream zeros -> zero gradient
    assert np.all(oracle.sample_vjp(ba, fi, F, Nv, np.zeros_like(p)) == 0)
    # SPEC.md:243 one sample at a vertex -> gradient flows entirely to that vertex
    g = np.zeros_like(p)
    g[0, 0] = [1.0, -2.0, 0.5]
    gv = oracle.sample_vjp(ba, fi, F, Nv, g)
    v0 = F[fi[0, 0], 0]
    np.testing.assert_array_equal(gv[0, v0], [1.0, -2.0, 0.5])
    assert np.count_nonzero(np.abs(gv).sum(-1)) == 1
    # SPEC.md:244 random upstream vs central differences of the fixed-weights forward map
    rng = np.random.default_rng(9)
    g = rng.normal(size=p.shape)
    gv = oracle.sample_vjp(ba, fi, F, Nv, g)

    def fwd(Vd):
        corners = Vd[0][F[fi[0]]]
        return (ba[0][:, :, None] * corners).sum(1)

    Vd = V.astype(np.float64)
    for vi in rng.choice(Nv, 12, replace=False):
        for c in range(3):
            eps = 1e-5 * max(1.0, abs(Vd[0, vi, c]))
            Vp, Vm = Vd.copy(), Vd.copy()
            Vp[0, vi, c] += eps
            Vm[0, vi, c] -= eps
            fd = ((fwd(Vp) - fwd(Vm)) * g[0]).sum() / (2 * eps)
            a = gv[0, vi, c]
            assert abs(a - fd) / max(abs(a), abs(fd), 1e-8) < 1e-6


def test_pipeline_sample_chamfer_gradient_fd():
    # the sample -> chamfer pipeline gradient w.r.t. the mesh vertices passes central
    # differences (choices and barycentric weights held fixed: the reparameterisation)
    V, F = synth.mesh_batch(1, subdiv=1)
    Nv = V.shape[1]
    rf, rb = _rand(1, 60, 10)
    Y = synth.uniform_pair(1, 50, 50, seed=11)[1] * 0.8
    p, fi, ba, _ = oracle.sample_mesh(V, F, rf, rb)

    def loss_of(Vd):
        corners = Vd[0][F[fi[0]]]
        pts = (ba[0][:, :, None] * corners).sum(1)[None]
        out = oracle.chamfer(pts, Y.astype(np.float64))
        return out["loss"], out["idx_xy"], out["idx_yx"], pts

    Vd = V.astype(np.float64)
    L0, ixy, iyx, pts = loss_of(Vd)
    gx, _, _, _ = oracle.loss_grad(pts, Y.astype(np.float64), ixy, iyx)
    gv = oracle.sample_vjp(ba, fi, F, Nv, gx)
    rng = np.random.default_rng(12)
    checked = 0
    for vi in rng.choice(Nv, 20, replace=False):
        for c in range(3):
            eps = 1e-5 * max(1.0, abs(Vd[0, vi, c]))
            Vp, Vm = Vd.copy(), Vd.copy()
            Vp[0, vi, c] += eps
            Vm[0, vi, c] -= eps
            Lp, ixp, iyp, _ = loss_of(Vp)
            Lm, ixm, iym, _ = loss_of(Vm)
            if not (np.array_equal(ixp, ixy) and np.array_equal(ixm, ixy) and np.array_equal(iyp, iyx)
                    and np.array_equal(iym, iyx)):
                continue
            fd = (Lp - Lm) / (2 * eps)
            a = gv[0, vi, c]
            assert abs(a - fd) / max(abs(a), abs(fd), 1e-8) < 1e-5
            checked += 1
    assert checked >= 48
