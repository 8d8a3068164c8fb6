"""Pins for the CPU oracle (no GPU).  Each test checks the oracle against something other than
itself: values from SPEC.md / hand derivations (tests/golden), closed forms, invariants, an exact
rational brute force (tests/exact_ref.py), scipy's exact k-d tree, and central finite differences.
"""
import glob
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_1911_05063_b200 import synth
from tests import exact_ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- golden worked examples
@pytest.mark.parametrize("name", ["spec_s445_unit_pair.json", "e2_two_vs_one.json", "tie_two_targets.json"])
def test_golden_forward_and_grad(name):
    g = _golden(name)
    x = np.array(g["x"], np.float32)
    y = np.array(g["y"], np.float32)
    e = g["expect"]
    out = oracle.chamfer(x, y, g["w1"], g["w2"])
    np.testing.assert_array_equal(out["d_xy"], np.array(e["d_xy"]))
    np.testing.assert_array_equal(out["idx_xy"], np.array(e["idx_xy"]))
    np.testing.assert_array_equal(out["d_yx"], np.array(e["d_yx"]))
    np.testing.assert_array_equal(out["idx_yx"], np.array(e["idx_yx"]))
    np.testing.assert_array_equal(out["cd"], np.array(e["cd"]))
    assert out["loss"] == e["loss"]
    gx, gy, _, _ = oracle.loss_grad(x, y, out["idx_xy"], out["idx_yx"], g["w1"], g["w2"])
    np.testing.assert_array_equal(gx, np.array(e["grad_x"]))
    np.testing.assert_array_equal(gy, np.array(e["grad_y"]))


def test_golden_fscore():
    g = _golden("fscore_example.json")
    out = oracle.chamfer(np.array(g["x"], np.float32), np.array(g["y"], np.float32), tau=g["tau"])
    e = g["expect"]
    np.testing.assert_array_equal(out["hits_xy"], e["hits_xy"])
    np.testing.assert_array_equal(out["hits_yx"], e["hits_yx"])
    np.testing.assert_allclose(out["precision"], e["precision"], rtol=0, atol=0)
    np.testing.assert_allclose(out["recall"], e["recall"], rtol=0, atol=0)
    np.testing.assert_allclose(out["fscore"], e["fscore"], rtol=1e-15)


def test_fscore_from_hits_pins():
    """oracle.fscore_from_hits (it evaluates the oracle F at the GPU's hit counts, R16) against the
    golden example's counts, exact rationals F = 2 hx hy / (hx M + hy N) (R15 written over the
    integers), the degenerate P + R = 0 case, and oracle.fscore on random distances."""
    from fractions import Fraction
    g = _golden("fscore_example.json")
    N, M = len(g["x"][0]), len(g["y"][0])
    e = g["expect"]
    np.testing.assert_allclose(oracle.fscore_from_hits(e["hits_xy"], e["hits_yx"], N, M), e["fscore"], rtol=1e-15)
    # roles: hits_xy / N is the precision, hits_yx / M the recall; with N != M a swap changes F
    assert abs(oracle.fscore_from_hits([1], [3], 2, 4)[0] - 0.6) < 1e-15
    assert abs(oracle.fscore_from_hits([3], [1], 2, 4)[0] - 0.6) > 0.1
    assert oracle.fscore_from_hits([0], [0], 5, 7)[0] == 0.0
    assert oracle.fscore_from_hits([0], [7], 5, 7)[0] == 0.0          # P = 0, R = 1 -> F = 0
    rng = np.random.default_rng(11)
    for _ in range(200):
        N, M = (int(v) for v in rng.integers(1, 10 ** 6, size=2))
        hx, hy = int(rng.integers(0, N + 1)), int(rng.integers(0, M + 1))
        exact = Fraction(0) if hx == 0 or hy == 0 else Fraction(2 * hx * hy, hx * M + hy * N)
        got = oracle.fscore_from_hits([hx], [hy], N, M)[0]
        assert abs(Fraction(got) - exact) <= Fraction(4, 2 ** 53) * exact
    d_xy = rng.uniform(0, 4e-4, size=(3, 500))
    d_yx = rng.uniform(0, 4e-4, size=(3, 700))
    ref = oracle.fscore(d_xy, d_yx, 0.01)
    np.testing.assert_array_equal(oracle.fscore_from_hits(ref["hits_xy"], ref["hits_yx"], 500, 700), ref["fscore"])


def test_golden_same_cloud_prints_zero():
    g = _golden("spec_s613_same_cloud.json")
    x = np.array(g["x"], np.float32)
    out = oracle.chamfer(x, np.array(g["y"], np.float32))
    assert out["loss"] == 0.0
    assert f"chamfer {out['loss']:.12f}" == g["expect"]["printed"]
    np.testing.assert_array_equal(out["idx_xy"], g["expect"]["idx_xy"])
    np.testing.assert_array_equal(out["idx_yx"], g["expect"]["idx_yx"])


def test_golden_files_cite_sources():
    for path in glob.glob(os.path.join(GOLDEN, "*.json")):
        with open(path) as f:
            assert "source" in json.load(f), path


# ---------------------------------------------------------------- exact rational brute force
def _dyadic_cloud(rng, B, P, bits=6):
    # coordinates k / 2^bits, |k| <= 2^bits: every fp64 operation in the oracle is exact
    return (rng.integers(-(2 ** bits), 2 ** bits + 1, size=(B, P, 3)) / 2.0 ** bits).astype(np.float32)


@pytest.mark.parametrize("seed,B,N,M", [(0, 1, 7, 5), (1, 2, 16, 23), (2, 3, 31, 9), (3, 1, 64, 64)])
def test_oracle_matches_exact_rational_dyadic(seed, B, N, M):
    rng = np.random.default_rng(seed)
    x = _dyadic_cloud(rng, B, N, bits=3)   # coarse lattice: many exact ties
    y = _dyadic_cloud(rng, B, M, bits=3)
    ex = exact_ref.chamfer_exact(x, y)
    out = oracle.chamfer(x, y)
    for key in ("d_xy", "d_yx"):
        np.testing.assert_array_equal(out[key], np.array([[float(v) for v in row] for row in ex[key]]))
    for key in ("idx_xy", "idx_yx"):
        np.testing.assert_array_equal(out[key], np.array(ex[key]))
    for key in ("d2_xy", "d2_yx"):
        ref = np.array([[math.inf if v is None else float(v) for v in row] for row in ex[key]])
        np.testing.assert_array_equal(out[key], ref)
    # CD_b and the loss take a few fp64 roundings (division, weighting, batch mean)
    assert abs(out["loss"] - float(ex["loss"])) <= 4e-16 * abs(float(ex["loss"]))
    np.testing.assert_allclose(out["cd"], [float(c) for c in ex["cd"]], rtol=4e-16, atol=0)
    # gradients with random dyadic upstream (exact in fp64)
    g = (rng.integers(-8, 9, size=(B, N)) / 8.0)
    h = (rng.integers(-8, 9, size=(B, M)) / 8.0)
    from fractions import Fraction
    gx_e, gy_e = exact_ref.grad_exact(ex["X"], ex["Y"], ex["idx_xy"], ex["idx_yx"],
                                      [[Fraction(v) for v in r] for r in g], [[Fraction(v) for v in r] for r in h])
    gx, gy, _, _ = oracle.backward(x, y, out["idx_xy"], out["idx_yx"], g, h)
    np.testing.assert_array_equal(gx, np.array([[[float(c) for c in p] for p in cl] for cl in gx_e]))
    np.testing.assert_array_equal(gy, np.array([[[float(c) for c in p] for p in cl] for cl in gy_e]))


def test_oracle_matches_exact_rational_generic():
    # non-dyadic fp32 inputs: fp64 result within a few ulp of the exact value; exact argmin where
    # the exact top-2 gap is wider than the fp64 rounding (relative 1e-12)
    rng = np.random.default_rng(11)
    x = rng.uniform(-0.5, 0.5, size=(2, 40, 3)).astype(np.float32)
    y = rng.uniform(-0.5, 0.5, size=(2, 33, 3)).astype(np.float32)
    ex = exact_ref.chamfer_exact(x, y)
    out = oracle.chamfer(x, y)
    for dk, ik, sk in (("d_xy", "idx_xy", "d2_xy"), ("d_yx", "idx_yx", "d2_yx")):
        ref = np.array([[float(v) for v in row] for row in ex[dk]])
        np.testing.assert_allclose(out[dk], ref, rtol=1e-15)
        gap_ok = np.array([[(s - d) > d * 1e-12 for d, s in zip(r1, r2)] for r1, r2 in zip(ex[dk], ex[sk])])
        assert gap_ok.mean() > 0.9
        np.testing.assert_array_equal(out[ik][gap_ok], np.array(ex[ik])[gap_ok])
    assert abs(out["loss"] - float(ex["loss"])) <= 1e-15 * float(ex["loss"])


# ---------------------------------------------------------------- invariants
def test_self_distance_zero_identity_index():
    X, _ = synth.uniform_pair(2, 300, 10, seed=3)
    out = oracle.chamfer(X, X, tau=0.0)
    assert out["loss"] == 0.0
    assert np.all(out["d_xy"] == 0) and np.all(out["d_yx"] == 0)
    np.testing.assert_array_equal(out["idx_xy"], np.tile(np.arange(300), (2, 1)))
    np.testing.assert_array_equal(out["fscore"], 1.0)  # F = 1 for every tau >= 0


def test_duplicates_take_lowest_index():
    rng = np.random.default_rng(5)
    base = rng.uniform(-0.5, 0.5, size=(1, 50, 3)).astype(np.float32)
    dup_at = rng.permutation(50)[:10]
    y = np.concatenate([base, base[:, dup_at]], axis=1)      # later copies of 10 points
    out = oracle.chamfer(base, y)
    np.testing.assert_array_equal(out["idx_xy"][0], np.arange(50))  # first copy (lowest index) wins
    assert np.all(out["d_xy"] == 0)
    # CD = 0 <=> equal as sets: duplicated/permuted copy is still distance 0
    perm = rng.permutation(y.shape[1])
    assert oracle.chamfer(base, y[:, perm])["loss"] == 0.0


def test_symmetry_exact():
    X, Y = synth.shape_pair(2, 500, 700, config_index=7)
    a = oracle.chamfer(X, Y)
    b = oracle.chamfer(Y, X)
    assert a["loss"] == b["loss"]
    np.testing.assert_array_equal(a["d_xy"], b["d_yx"])
    np.testing.assert_array_equal(a["idx_xy"], b["idx_yx"])


def test_lattice_closed_form():
    h = 2.0 ** -5
    k = np.arange(8)
    g = np.stack(np.meshgrid(k, k, k, indexing="ij"), -1).reshape(-1, 3) * h
    delta = 2.0 ** -8  # 0 < delta < h/2
    X = g[None].astype(np.float32)
    Y = (g + np.array([0, 0, delta]))[None].astype(np.float32)
    out = oracle.chamfer(X, Y, tau=delta)
    np.testing.assert_array_equal(out["d_xy"], delta ** 2)
    np.testing.assert_array_equal(out["d_yx"], delta ** 2)
    np.testing.assert_array_equal(out["idx_xy"][0], np.arange(g.shape[0]))
    assert out["loss"] == 2 * delta ** 2
    assert out["fscore"][0] == 1.0
    assert oracle.chamfer(X, Y, tau=delta * 0.999)["fscore"][0] == 0.0


def test_power_of_two_scaling_exact():
    X, Y = synth.shape_pair(1, 400, 300, config_index=8)
    a = oracle.chamfer(X, Y)
    for kexp in (-3, 2, 5):
        s = np.float32(2.0 ** kexp)
        b = oracle.chamfer(X * s, Y * s)
        np.testing.assert_array_equal(b["idx_xy"], a["idx_xy"])
        np.testing.assert_array_equal(b["d_xy"], a["d_xy"] * 4.0 ** kexp)
        assert b["loss"] == a["loss"] * 4.0 ** kexp


def test_permutation_equivariance():
    X, Y = synth.uniform_pair(1, 256, 300, seed=9)
    perm = np.random.default_rng(0).permutation(300)
    a = oracle.chamfer(X, Y)
    b = oracle.chamfer(X, Y[:, perm])
    inv = np.argsort(perm)
    np.testing.assert_array_equal(b["d_xy"], a["d_xy"])
    np.testing.assert_array_equal(b["idx_xy"], inv[a["idx_xy"]])
    assert b["loss"] == a["loss"]


def test_translation_invariance_approx():
    X, Y = synth.shape_pair(1, 300, 300, config_index=9)
    t = np.array([0.25, -0.125, 0.5], np.float32)   # exact shifts, approx invariance (R13 text)
    a = oracle.chamfer(X, Y)
    b = oracle.chamfer(X + t, Y + t)
    assert abs(a["loss"] - b["loss"]) <= 1e-5 * a["loss"]


# ---------------------------------------------------------------- library special case: exact k-d tree
def test_matches_scipy_ckdtree():
    from scipy.spatial import cKDTree
    X, Y = synth.shape_pair(2, 4000, 5000, config_index=10)
    out = oracle.chamfer(X, Y)
    for b in range(2):
        dd, ii = cKDTree(Y[b].astype(np.float64)).query(X[b].astype(np.float64), k=2)
        np.testing.assert_allclose(out["d_xy"][b], dd[:, 0] ** 2, rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(out["d2_xy"][b], dd[:, 1] ** 2, rtol=1e-12, atol=1e-300)
        clear = (dd[:, 1] ** 2 - dd[:, 0] ** 2) > 1e-9 * dd[:, 0] ** 2
        np.testing.assert_array_equal(out["idx_xy"][b][clear], ii[clear, 0])
        dd2, ii2 = cKDTree(X[b].astype(np.float64)).query(Y[b].astype(np.float64), k=1)
        np.testing.assert_allclose(out["d_yx"][b], dd2 ** 2, rtol=1e-12, atol=1e-300)


# ---------------------------------------------------------------- gradients
def _loss_fd(x, y, w1=1.0, w2=1.0):
    out = oracle.chamfer(x, y, w1, w2)
    return out["loss"], out["idx_xy"], out["idx_yx"]


def test_gradient_central_differences():
    # Well-separated tiny clouds (SPEC.md:545 'chamfer on well-separated clouds -> pass at tol 1e-6').
    rng = np.random.default_rng(21)
    B, N, M = 2, 6, 5
    x = rng.uniform(-1, 1, size=(B, N, 3))
    y = rng.uniform(-1, 1, size=(B, M, 3))
    w1, w2 = 0.7, 1.3
    L0, ixy, iyx = _loss_fd(x, y, w1, w2)
    gx, gy, _, _ = oracle.backward(x, y, ixy, iyx, g_scalar=w1 / (B * N), h_scalar=w2 / (B * M))
    checked = skipped = 0
    for arr, grad in ((x, gx), (y, gy)):
        for idx in np.ndindex(arr.shape):
            eps = 1e-5 * max(1.0, abs(arr[idx]))
            old = arr[idx]
            arr[idx] = old + eps
            Lp, ixp, iyp = _loss_fd(x, y, w1, w2)
            arr[idx] = old - eps
            Lm, ixm, iym = _loss_fd(x, y, w1, w2)
            arr[idx] = old
            if not (np.array_equal(ixp, ixy) and np.array_equal(ixm, ixy)
                    and np.array_equal(iyp, iyx) and np.array_equal(iym, iyx)):
                skipped += 1                          # argmin flip: discontinuity filter
                continue
            fd = (Lp - Lm) / (2 * eps)
            a = grad[idx]
            rel = abs(a - fd) / max(abs(a), abs(fd), 1e-8)
            assert rel < 1e-6, (idx, a, fd, rel)
            checked += 1
    assert skipped <= 0.2 * (checked + skipped)


def test_vjp_linearity_exact():
    # SPEC.md:531 vjp(2u) = 2 vjp(u); power-of-two scaling is exact in fp64
    X, Y = synth.shape_pair(1, 200, 250, config_index=12)
    out = oracle.chamfer(X, Y)
    rng = np.random.default_rng(1)
    g = rng.normal(size=(1, 200))
    h = rng.normal(size=(1, 250))
    a = oracle.backward(X, Y, out["idx_xy"], out["idx_yx"], g, h)
    b = oracle.backward(X, Y, out["idx_xy"], out["idx_yx"], 2 * g, 2 * h)
    np.testing.assert_array_equal(b[0], 2 * a[0])
    np.testing.assert_array_equal(b[1], 2 * a[1])


def test_grad_scalar_fill_equals_array():
    X, Y = synth.shape_pair(1, 100, 120, config_index=13)
    out = oracle.chamfer(X, Y)
    a = oracle.loss_grad(X, Y, out["idx_xy"], out["idx_yx"], 1.0, 1.0)
    b = oracle.backward(X, Y, out["idx_xy"], out["idx_yx"], np.full((1, 100), 1 / 100), np.full((1, 120), 1 / 120))
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_grad_condition_scale_bounds_grad():
    X, Y = synth.shape_pair(1, 300, 200, config_index=14)
    out = oracle.chamfer(X, Y)
    gx, gy, sx, sy = oracle.loss_grad(X, Y, out["idx_xy"], out["idx_yx"])
    assert np.all(np.abs(gx) <= sx * (1 + 1e-12)) and np.all(np.abs(gy) <= sy * (1 + 1e-12))


# ---------------------------------------------------------------- fp32 mirror
def test_mirror_close_to_oracle():
    X, Y = synth.shape_pair(2, 2000, 1500, config_index=15)
    d, i = oracle.mirror_nn_f32(X, Y)
    d1, i1, d2 = oracle.nn(X, Y)
    # fp32 squared distance of fp32 points: <= ~4 ulp relative (all terms non-negative)
    np.testing.assert_allclose(d.astype(np.float64), d1, rtol=5e-7, atol=0)
    clear = (d2 - d1) > 1e-6 * d1
    assert clear.mean() > 0.99
    np.testing.assert_array_equal(i[clear], i1[clear])


def test_mirror_exact_on_dyadic():
    rng = np.random.default_rng(2)
    x = _dyadic_cloud(rng, 2, 50, bits=4)
    y = _dyadic_cloud(rng, 2, 60, bits=4)
    d, i = oracle.mirror_nn_f32(x, y)
    d1, i1, _ = oracle.nn(x, y)
    np.testing.assert_array_equal(d.astype(np.float64), d1)   # all ops exact => identical
    np.testing.assert_array_equal(i, i1)


def test_rows_subset_matches_full():
    X, Y = synth.shape_pair(3, 500, 400, config_index=16)
    full = oracle.nn(X, Y)
    rows = np.array([0, 7, 499, 500, 1234, 1499])
    sub = oracle.nn(X, Y, rows=rows)
    for a, b in zip(sub, full):
        np.testing.assert_array_equal(a, b.reshape(-1)[rows])


def test_empty_cloud_is_domain_error():
    with pytest.raises(ValueError):
        oracle.nn(np.zeros((1, 0, 3)), np.zeros((1, 3, 3)))
