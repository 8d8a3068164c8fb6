"""GPU parity for NEXT-3 (point-to-surface loss) through the C ABI against the fp64 oracle
(tests/test_oracle_p2s.py pins it).  Gate (R24): the face index must equal the oracle's
where the oracle's best and second-best face distances differ by more than 1e-6 d + delta,
delta = 2^-22 R^2 (R = coordinate scale; the fp32 hot loop's absolute error bound); elsewhere any
face within that band of the minimum is accepted.  The kernels evaluate d, the closest point and its
barycentrics in fp64 for the chosen face with R24's plane-or-edges formulation; the oracle uses the
region decomposition (no shared code): within 1e-5 relative (plus delta for d).  Gradients: the
elementwise R28 gate (_grad_gate)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
from paper_1911_05063_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1911_05063_b200 import api
    return api


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _face_d2(P, V, F, fidx):
    """fp64 distance of each point to a given face (oracle, one face per point)."""
    B, N, _ = P.shape
    out = np.empty((B, N))
    for b in range(B):
        for i in range(N):
            d, _, _, _, _ = oracle.p2s(P[b:b + 1, i:i + 1], V[b:b + 1], F[fidx[b, i]:fidx[b, i] + 1])
            out[b, i] = d[0, 0]
    return out


def _gate(P, V, F, out, rows=None, min_clear=0.3):
    d, fi, cl, ba = (o.cpu().numpy() for o in out[:4])
    B, N, _ = P.shape
    R = max(np.abs(P).max(), np.abs(V).max())
    delta = 2.0 ** -22 * R * R
    if rows is None:
        rows = np.arange(B * N)
    d1, f1, d2, c1, l1 = oracle.p2s(P, V, F, rows=rows)
    dg, fg = d.reshape(-1)[rows], fi.reshape(-1)[rows]
    clear = (d2 - d1) > 1e-6 * d1 + delta
    assert clear.mean() >= min_clear
    np.testing.assert_array_equal(fg[clear], f1[clear])
    np.testing.assert_allclose(dg[clear], d1[clear], rtol=1e-5, atol=delta)
    amb = ~clear
    if amb.any():
        b = rows[amb] // N
        i = rows[amb] % N
        Pa = P[b, i][:, None]
        dd = np.array([oracle.p2s(Pa[k:k + 1], V[b[k]:b[k] + 1], F[fg[amb][k]:fg[amb][k] + 1])[0][0, 0]
                       for k in range(Pa.shape[0])])
        assert np.all(dd <= d1[amb] * (1 + 1e-6) + delta)
        np.testing.assert_allclose(dg[amb], dd, rtol=1e-5, atol=delta)
    # closest point / barycentrics consistent with the chosen face
    cg = cl.reshape(-1, 3)[rows]
    lg = ba.reshape(-1, 3)[rows]
    assert np.all(lg >= -1e-6) and np.allclose(lg.sum(1), 1.0, atol=1e-5)
    bb = rows // N
    corners = V[bb[:, None], F[fg]]                       # (n, 3, 3)
    np.testing.assert_allclose(cg, (lg[:, :, None] * corners).sum(1), atol=1e-5 * R)
    # and equal to the oracle's own closest point / barycentrics (region decomposition, fp64) on the
    # same face: the kernels' plane-or-edges evaluation differs only by fp64 rounding, then the fp32
    # store (2^-24 relative); barycentrics to fp32 rounding of values in [0, 1]
    np.testing.assert_allclose(cg[clear], c1[clear], rtol=0, atol=2.0 ** -22 * R)
    # (a zero-area face's barycentrics are not unique: compare them on proper faces only)
    c64 = corners.astype(np.float64)
    area2 = np.linalg.norm(np.cross(c64[:, 1] - c64[:, 0], c64[:, 2] - c64[:, 0]), axis=1)
    proper = clear & (area2 > 1e-6 * R * R)
    np.testing.assert_allclose(lg[proper], l1[proper], rtol=0, atol=2.0 ** -20)
    return d1, f1, clear


@pytest.mark.parametrize("B,N,subdiv,near", [(1, 1, 0, False), (2, 3000, 3, False), (2, 2000, 3, True),
                                             (1, 5000, 1, False)])
def test_p2s_parity(cd, B, N, subdiv, near):
    V, F = synth.mesh_batch(B, subdiv=subdiv, config_index=120)
    if near:   # points sampled on the mesh itself (d ~ 0) plus small offsets
        rf, rb = synth.sampling_randoms(B, N, seed=9)
        P, _, _, _ = oracle.sample_mesh(V, F, rf, rb)
        P = (P + np.random.default_rng(1).normal(scale=1e-3, size=P.shape)).astype(np.float32)
    else:
        P = synth.shape_pair(B, N, 8, config_index=121)[0]
    out = cd.p2s_forward(_t(P), _t(V), _t(F))
    torch.cuda.synchronize()
    _gate(P, V, F, out, min_clear=0.0 if N == 1 else 0.3)
    # loss = mean_b mean_i d (fp64 sums of the GPU's d)
    d = out[0].cpu().numpy().astype(np.float64)
    assert abs(out[5].item() - d.mean()) <= 1e-6 * d.mean() + 1e-30


def test_p2s_large_sampled(cd):
    B, N = 4, 16384
    V, F = synth.mesh_batch(B, subdiv=4, config_index=122)
    P = synth.shape_pair(B, N, 8, config_index=123)[0]
    out = cd.p2s_forward(_t(P), _t(V), _t(F))
    rows = np.random.default_rng(2).choice(B * N, 1500, replace=False)
    _gate(P, V, F, out, rows=rows)


def test_p2s_backward(cd):
    B, N = 2, 2500
    V, F = synth.mesh_batch(B, subdiv=3, config_index=124)
    P = synth.shape_pair(B, N, 8, config_index=125)[0]
    d, fi, cl, ba, pb, loss = cd.p2s_forward(_t(P), _t(V), _t(F))
    g = np.random.default_rng(3).normal(size=(B, N)).astype(np.float32)
    gp, gv = cd.p2s_backward(_t(P), cl, fi, ba, _t(F), V.shape[1], g=_t(g))
    torch.cuda.synchronize()
    # oracle VJPs evaluated on the GPU's chosen faces (backward-only mode)
    fi_n = fi.cpu().numpy()
    same = fi_n == oracle.p2s(P, V, F)[1]
    gp_ref, gv_ref = oracle.p2s_grads(P, V, F, fi_n, cl.cpu().numpy(), ba.cpu().numpy(), g)
    np.testing.assert_allclose(gp.cpu().numpy(), gp_ref, rtol=1e-5, atol=1e-7)
    scale = oracle.sample_vjp(np.abs(ba.cpu().numpy()).astype(np.float64), fi_n, F, V.shape[1],
                              np.abs(gp_ref))
    assert np.all(np.abs(gv.cpu().numpy() - gv_ref) <= 1e-5 * scale + 1e-7)
    assert same.mean() > 0.5


def _grad_gate(P, V, F, fi_gpu, gp, gv, g):
    """Elementwise gradient gate (R14 / R28) in full fwd+bwd mode.  The reference is the
    oracle's VJP at the oracle's closest face, except where the GPU chose another face inside the
    R24 ambiguity band (the forward gate accepts it): there the oracle's fp64 closest point ON THE
    GPU's FACE is used, so every point is compared.  Scale per element: the sum of the magnitudes
    of the difference's terms, S_p = 2|g|(|p| + |c|) for grad_p and S_v = sum_k lam_k S_p over the
    vertex's (point, corner) pairs — the fp32 closest point alone carries 2^-24 |c| of rounding."""
    B, N, _ = P.shape
    _, fi, _, cl, la = oracle.p2s(P, V, F)
    amb = np.argwhere(fi != fi_gpu)
    fi_ref = fi.copy()
    for b, i in amb:
        f = int(fi_gpu[b, i])
        _, _, _, c1, l1 = oracle.p2s(P[b:b + 1, i:i + 1], V[b:b + 1], F[f:f + 1])
        fi_ref[b, i], cl[b, i], la[b, i] = f, c1[0, 0], l1[0, 0]
    gp_ref, gv_ref = oracle.p2s_grads(P, V, F, fi_ref, cl, la, g)
    Sp = 2.0 * np.abs(np.asarray(g, np.float64))[..., None] * (np.abs(P.astype(np.float64)) + np.abs(cl))
    Sv = oracle.sample_vjp(np.abs(la), fi_ref, F, V.shape[1], Sp)
    assert np.all(np.abs(gp - gp_ref) <= 1e-5 * Sp)
    assert np.all(np.abs(gv - gv_ref) <= 1e-5 * Sv + 1e-30)
    # headline over the same scale (near the surface |p - c| << |c|, and the fp32 closest point's own
    # rounding alone is ~2^-24 |c| / |p - c| relative to grad_p: the plain relative L2 is ill-conditioned)
    assert np.linalg.norm(gp - gp_ref) <= 1e-5 * np.linalg.norm(Sp)
    return len(amb)


def test_p2s_autograd(cd):
    B, N = 2, 3000
    V, F = synth.mesh_batch(B, subdiv=3, config_index=126)
    P = synth.shape_pair(B, N, 8, config_index=127)[0]
    p = _t(P).requires_grad_(True)
    v = _t(V).requires_grad_(True)
    loss = cd.point_to_surface(p, v, _t(F))
    loss.backward()
    d = oracle.p2s(P, V, F)[0]
    assert abs(loss.item() - d.mean()) <= 1e-5 * d.mean()
    fi_gpu = cd.p2s_forward(_t(P), _t(V), _t(F))[1].cpu().numpy()
    _grad_gate(P, V, F, fi_gpu, p.grad.cpu().numpy(), v.grad.cpu().numpy(), np.full((B, N), 1.0 / (B * N)))


def test_p2s_autograd_near_surface(cd):
    """Points within ~1e-3 of the surface (p - c small: the conditioning case of R28) with a random
    upstream through the explicit backward entry point."""
    B, N = 2, 2500
    V, F = synth.mesh_batch(B, subdiv=3, config_index=128)
    rf, rb = synth.sampling_randoms(B, N, seed=21)
    P, _, _, _ = oracle.sample_mesh(V, F, rf, rb)
    P = (P + np.random.default_rng(22).normal(scale=1e-3, size=P.shape)).astype(np.float32)
    d, fi, cl, ba, _, _ = cd.p2s_forward(_t(P), _t(V), _t(F))
    g = np.random.default_rng(23).normal(size=(B, N)).astype(np.float32)
    gp, gv = cd.p2s_backward(_t(P), cl, fi, ba, _t(F), V.shape[1], g=_t(g))
    torch.cuda.synchronize()
    _grad_gate(P, V, F, fi.cpu().numpy(), gp.cpu().numpy(), gv.cpu().numpy(), g)


# ---------------------------------------------------------------------------------- culled path (R26)
def _pruned_vs_brute(cd, P, V, F, rows=None, min_clear=0.3):
    """The culled forward against the oracle (same gate) and against the brute-force kernel: the
    same face for every point — the lowest original face index among the faces at the exact fp32
    minimum, ties included (R3') — and then bit-identical d / closest / bary (both evaluate the
    chosen face with the same fp64 code)."""
    outp = cd.p2s_forward(_t(P), _t(V), _t(F), algorithm="pruned")
    outb = cd.p2s_forward(_t(P), _t(V), _t(F))
    torch.cuda.synchronize()
    d1, f1, clear = _gate(P, V, F, outp, rows=rows, min_clear=min_clear)
    dp, fp, cp, bp = (o.cpu().numpy() for o in outp[:4])
    db, fb, cb, bb = (o.cpu().numpy() for o in outb[:4])
    np.testing.assert_array_equal(fp, fb)
    np.testing.assert_array_equal(dp, db)
    np.testing.assert_array_equal(cp, cb)
    np.testing.assert_array_equal(bp, bb)
    # loss: fp64 sums of the per-point d (summation order differs from the brute force)
    assert abs(outp[5].item() - dp.astype(np.float64).mean()) <= 1e-6 * dp.mean() + 1e-30
    np.testing.assert_allclose(outp[4].cpu().numpy(), dp.astype(np.float64).mean(1), rtol=1e-6)
    return outp


@pytest.mark.parametrize("B,N,subdiv,near", [(1, 1, 0, False), (2, 3000, 3, False), (2, 2000, 3, True),
                                             (1, 5000, 1, False), (3, 777, 2, True), (2, 4097, 4, True)])
def test_p2s_pruned_parity(cd, B, N, subdiv, near):
    V, F = synth.mesh_batch(B, subdiv=subdiv, config_index=130)
    if near:
        rf, rb = synth.sampling_randoms(B, N, seed=11)
        P, _, _, _ = oracle.sample_mesh(V, F, rf, rb)
        P = (P + np.random.default_rng(4).normal(scale=1e-3, size=P.shape)).astype(np.float32)
    else:
        P = synth.shape_pair(B, N, 8, config_index=131)[0]
    rows = None if B * N <= 6000 else np.random.default_rng(5).choice(B * N, 2000, replace=False)
    _pruned_vs_brute(cd, P, V, F, rows=rows, min_clear=0.0 if N == 1 else 0.3)


def test_p2s_pruned_far_and_exact_surface(cd):
    """Points far outside the mesh (little culling) and points exactly on faces (d = 0 ties between
    neighbouring faces at shared edges)."""
    B, N = 2, 3000
    V, F = synth.mesh_batch(B, subdiv=3, config_index=132)
    Pfar = (synth.shape_pair(B, N, 8, config_index=133)[0] * 5.0 + 3.0).astype(np.float32)
    _pruned_vs_brute(cd, Pfar, V, F, min_clear=0.0)   # mostly vertex-closest: exact ties between blocks
    rf, rb = synth.sampling_randoms(B, N, seed=12)
    Pon, _, _, _ = oracle.sample_mesh(V, F, rf, rb)
    _pruned_vs_brute(cd, Pon.astype(np.float32), V, F, min_clear=0.0)


def test_p2s_pruned_bench_config_sampled(cd):
    """The bench's NEXT-3 workload (B=8, icosphere-5 with 20480 faces, 16384 points per mesh):
    the culled path agrees with the brute-force kernel everywhere and with the oracle on samples."""
    B, N = 8, 16384
    V, F = synth.mesh_batch(B, subdiv=5, config_index=134)
    rf, rb = synth.sampling_randoms(B, N, seed=13)
    P, _, _, _ = oracle.sample_mesh(V, F, rf, rb)
    P = (P + np.random.default_rng(6).normal(scale=1e-2, size=P.shape)).astype(np.float32)
    rows = np.random.default_rng(7).choice(B * N, 1500, replace=False)
    _pruned_vs_brute(cd, P, V, F, rows=rows)


def test_p2s_pruned_autograd(cd):
    B, N = 2, 3000
    V, F = synth.mesh_batch(B, subdiv=3, config_index=135)
    P = synth.shape_pair(B, N, 8, config_index=136)[0]
    p = _t(P).requires_grad_(True)
    v = _t(V).requires_grad_(True)
    loss = cd.point_to_surface(p, v, _t(F), algorithm="pruned")
    loss.backward()
    p2 = _t(P).requires_grad_(True)
    v2 = _t(V).requires_grad_(True)
    loss2 = cd.point_to_surface(p2, v2, _t(F))
    loss2.backward()
    assert abs(loss.item() - loss2.item()) <= 1e-6 * abs(loss2.item())
    # the culled forward's faces / closest points / barycentrics are bit-identical to the brute
    # force's, and the backward is deterministic: the gradients are bit-identical too
    np.testing.assert_array_equal(p.grad.cpu().numpy(), p2.grad.cpu().numpy())
    np.testing.assert_array_equal(v.grad.cpu().numpy(), v2.grad.cpu().numpy())
    fi_gpu = cd.p2s_forward(_t(P), _t(V), _t(F), algorithm="pruned")[1].cpu().numpy()
    _grad_gate(P, V, F, fi_gpu, p.grad.cpu().numpy(), v.grad.cpu().numpy(), np.full((B, N), 1.0 / (B * N)))


def test_p2s_degenerate_faces(cd):
    """Zero-area faces (a repeated vertex): the brute-force and culled kernels still pass the oracle
    gate (a degenerate face is a segment; its 'inside' test never fires, R24)."""
    B, N = 2, 3000
    V, F = synth.mesh_batch(B, subdiv=3, config_index=137)
    F = F.copy()
    sel = np.random.default_rng(14).choice(len(F), size=len(F) // 8, replace=False)
    F[sel, 2] = F[sel, 1]
    P = synth.shape_pair(B, N, 8, config_index=138)[0]
    for algo in ("brute", "pruned"):
        out = cd.p2s_forward(_t(P), _t(V), _t(F), algorithm=algo)
        torch.cuda.synchronize()
        _gate(P, V, F, out)


def test_p2s_pruned_nonfinite_points(cd):
    """Non-finite query points (R6): no finite candidate -> (+inf, face -1, closest 0, bary 0) as the
    oracle, from both kernels; every other point is unaffected (bit-identical to the brute force)."""
    B, N = 2, 3000
    V, F = synth.mesh_batch(B, subdiv=3, config_index=139)
    P = synth.shape_pair(B, N, 8, config_index=140)[0].copy()
    bad = [(0, 3), (0, 9), (1, 17)]
    P[0, 3] = np.nan
    P[0, 9, 1] = np.inf
    P[1, 17, 2] = -np.inf
    do, fo = oracle.p2s(P, V, F)[:2]
    for algo in ("brute", "pruned"):
        out = [o.cpu().numpy() for o in cd.p2s_forward(_t(P), _t(V), _t(F), algorithm=algo)[:4]]
        for i in bad:
            assert out[0][i] == np.inf and out[1][i] == -1 and do[i] == np.inf and fo[i] == -1
            assert not out[2][i].any() and not out[3][i].any()
        if algo == "brute":
            brute = out
        else:
            for a, b in zip(out, brute):
                np.testing.assert_array_equal(a, b)
    finite = np.isfinite(P).all(-1)
    assert np.isfinite(brute[0][finite]).all()
