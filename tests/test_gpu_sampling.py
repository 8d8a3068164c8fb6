"""GPU parity for NEXT-4 (differentiable surface sampling -> Chamfer), through the C ABI, against
the fp64 oracle (tests/test_oracle_mesh.py pins the oracle).  Face choices are integer decisions taken
in the same precision on both sides (R19): bit-exact.  Points and weights: fp32 vs fp64
within a few ulp.  The vertex gradient, given the GPU's weights, uses the oracle's accumulation order:
bit-exact."""
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


@pytest.mark.parametrize("B,N,subdiv", [(1, 1, 1), (2, 1000, 3), (4, 20000, 5), (32, 16384, 5)])
def test_sample_forward_parity(cd, B, N, subdiv):
    V, F = synth.mesh_batch(B, subdiv=subdiv)
    rf, rb = synth.sampling_randoms(B, N, seed=B + N)
    pts, fi, ba = cd.sample_mesh(_t(V), _t(F), _t(rf), _t(rb))
    torch.cuda.synchronize()
    p_ref, fi_ref, ba_ref, _ = oracle.sample_mesh(V, F, rf, rb)
    np.testing.assert_array_equal(fi.cpu().numpy(), fi_ref)                 # integer decision: exact
    np.testing.assert_allclose(ba.cpu().numpy(), ba_ref, rtol=0, atol=4e-7)  # fp32 weights (|w| <= 1)
    scale = np.abs(V[np.arange(B)[:, None, None], F[fi_ref]]).sum(2)     # (B,N,3): sum_k |v_k| per coordinate
    err = np.abs(pts.cpu().numpy() - p_ref)
    assert np.all(err <= 1e-6 * scale + 1e-30)


def test_sample_degenerate_and_single_face(cd):
    V = np.array([[[0, 0, 0], [1, 0, 0], [0, 1, 0], [2, 2, 2], [2, 2, 2], [3, 3, 3]]], np.float32)
    F = np.array([[3, 4, 5], [0, 1, 2], [3, 4, 5], [0, 2, 1]], np.int32)
    rf, rb = synth.sampling_randoms(1, 5000, seed=3)
    _, fi, _ = cd.sample_mesh(_t(V), _t(F), _t(rf), _t(rb))
    _, fi_ref, _, _ = oracle.sample_mesh(V, F, rf, rb)
    np.testing.assert_array_equal(fi.cpu().numpy(), fi_ref)
    Z = np.zeros((1, 3, 3), np.float32)    # all-degenerate mesh: face 0 (documented), no fault
    _, fz, _ = cd.sample_mesh(_t(Z), _t(np.array([[0, 1, 2]], np.int32)), _t(rf[:, :10]), _t(rb[:, :10]))
    assert np.all(fz.cpu().numpy() == 0)


@pytest.mark.parametrize("B,N,subdiv", [(1, 7, 1), (2, 3000, 3), (8, 16384, 5)])
def test_sample_backward_parity(cd, B, N, subdiv):
    V, F = synth.mesh_batch(B, subdiv=subdiv)
    Nv = V.shape[1]
    rf, rb = synth.sampling_randoms(B, N, seed=7 * B + N)
    pts, fi, ba = cd.sample_mesh(_t(V), _t(F), _t(rf), _t(rb))
    g = np.random.default_rng(N).normal(size=(B, N, 3)).astype(np.float32)
    gv = cd.sample_mesh_backward(_t(F), fi, ba, Nv, _t(g))
    torch.cuda.synchronize()
    ref = oracle.sample_vjp(ba.cpu().numpy().astype(np.float64), fi.cpu().numpy(), F, Nv, g.astype(np.float64))
    np.testing.assert_array_equal(gv.cpu().numpy(), ref.astype(np.float32))
    # against the oracle's own fp64 weights: within the fp32-weight rounding
    _, fi_ref, ba_ref, _ = oracle.sample_mesh(V, F, rf, rb)
    ref64 = oracle.sample_vjp(ba_ref, fi_ref, F, Nv, g.astype(np.float64))
    scale = oracle.sample_vjp(np.abs(ba_ref), fi_ref, F, Nv, np.abs(g).astype(np.float64))
    # fp32 weights carry an ABSOLUTE rounding error of a few 2^-24 (e.g. w0 = 1 - sqrt(r1) near 0)
    gsum = oracle.sample_vjp(np.ones_like(ba_ref), fi_ref, F, Nv, np.abs(g).astype(np.float64))
    assert np.all(np.abs(gv.cpu().numpy() - ref64) <= 1e-5 * scale + 2.0 ** -21 * gsum + 1e-30)


def test_sample_chamfer_autograd_pipeline(cd):
    """mesh -> sample -> chamfer -> backward to vertices, against the oracle pipeline gradient."""
    B, N, M = 2, 4096, 3000
    V, F = synth.mesh_batch(B, subdiv=4)
    Y = synth.shape_pair(B, 8, M, config_index=90)[1]
    rf, rb = synth.sampling_randoms(B, N, seed=21)
    v = _t(V).requires_grad_(True)
    pts, fi = cd.sample_points(v, _t(F), _t(rf), _t(rb))
    loss = cd.chamfer(pts, _t(Y))
    loss.backward()
    torch.cuda.synchronize()
    # oracle pipeline on the GPU's sampled points (face choices match exactly)
    P = pts.detach().cpu().numpy()
    ref = oracle.chamfer(P, Y)
    assert abs(loss.item() - ref["loss"]) <= 1e-5 * ref["loss"]
    gx, _, sx, _ = oracle.loss_grad(P, Y, ref["idx_xy"], ref["idx_yx"])
    _, fi_ref, ba_ref, _ = oracle.sample_mesh(V, F, rf, rb)
    np.testing.assert_array_equal(fi.cpu().numpy(), fi_ref)
    gv_ref = oracle.sample_vjp(ba_ref, fi_ref, F, V.shape[1], gx)
    scale = oracle.sample_vjp(ba_ref, fi_ref, F, V.shape[1], sx)
    gsum = oracle.sample_vjp(np.ones_like(ba_ref), fi_ref, F, V.shape[1], np.abs(gx))
    assert np.all(np.abs(v.grad.cpu().numpy() - gv_ref) <= 1e-5 * scale + 2.0 ** -21 * gsum + 1e-30)
