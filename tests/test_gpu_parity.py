"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element, on
seeded synthetic inputs — small configs in full, large configs on sampled rows —
plus the fp32 mirror (bit-exact), determinism, slicing and edge cases."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
from paper_1911_05063_b200 import synth
from tests.gpu_helpers import gate_forward_batch, gate_grad, gate_mirror, GAP, RTOL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1911_05063_b200 import api
    return api


def _run(cd, X, Y, tau=None, **kw):
    x = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    y = torch.from_numpy(np.ascontiguousarray(Y)).cuda()
    out = cd.forward(x, y, tau=tau, **kw)
    torch.cuda.synchronize()
    return x, y, [o.cpu().numpy() if o is not None else None for o in out]


def _full_check(cd, X, Y, tau=None, mirror=True, backward=True):
    x, y, (d_xy, i_xy, d_yx, i_yx, part) = _run(cd, X, Y, tau=tau)
    gate_forward_batch(X, Y, d_xy, i_xy, d_yx, i_yx)
    if mirror:
        gate_mirror(X, Y, d_xy, i_xy)
        gate_mirror(Y, X, d_yx, i_yx)
    ref = oracle.chamfer(X, Y, tau=tau)
    B, N, M = X.shape[0], X.shape[1], Y.shape[1]
    # partials vs oracle sums (fp64 sums of the GPU's own distances, R9)
    np.testing.assert_allclose(part[:, 0], np.asarray(d_xy, np.float64).sum(1), rtol=1e-12)
    np.testing.assert_allclose(part[:, 1], np.asarray(d_yx, np.float64).sum(1), rtol=1e-12)
    cdb, loss, F, P, R = cd.finalize(torch.from_numpy(part).cuda(), N, M)
    torch.cuda.synchronize()
    np.testing.assert_allclose(cdb.cpu().numpy(), ref["cd"], rtol=RTOL)
    assert abs(loss.item() - ref["loss"]) <= RTOL * abs(ref["loss"]) + (ref["loss"] == 0) * 0
    if tau is not None:
        t2 = oracle.tau_sq(tau)
        band = 1e-6 * t2
        for dist, hits, col in ((ref["d_xy"], part[:, 2], "xy"), (ref["d_yx"], part[:, 3], "yx")):
            lo = (dist < t2 - band).sum(1)
            hi = (dist <= t2 + band).sum(1)
            assert np.all((hits >= lo) & (hits <= hi)), col
        Fref = oracle.fscore_from_hits(part[:, 2], part[:, 3], N, M)
        np.testing.assert_allclose(F.cpu().numpy(), Fref, rtol=RTOL, atol=1e-7)
    if backward:
        rng = np.random.default_rng(7)
        g = rng.normal(size=(B, N)).astype(np.float32)
        h = rng.normal(size=(B, M)).astype(np.float32)
        gx, gy = cd.backward(x, y, torch.from_numpy(i_xy).cuda(), torch.from_numpy(i_yx).cuda(),
                             torch.from_numpy(g).cuda(), torch.from_numpy(h).cuda())
        torch.cuda.synchronize()
        gxr, gyr, sx, sy = oracle.backward(X, Y, i_xy, i_yx, g, h)   # backward-only mode: GPU indices
        # identical fp64 accumulation order => identical fp32 results (stricter than the gate)
        np.testing.assert_array_equal(gx.cpu().numpy(), gxr.astype(np.float32))
        np.testing.assert_array_equal(gy.cpu().numpy(), gyr.astype(np.float32))
        gate_grad(gx.cpu().numpy(), gxr, sx)
        gate_grad(gy.cpu().numpy(), gyr, sy)
    return d_xy, i_xy, d_yx, i_yx, part


# ------------------------------------------------------------------------------ configs
def test_c1_uniform(cd):
    X, Y = synth.uniform_pair(1, 1024, 1024, seed=1)
    _full_check(cd, X, Y, tau=0.05)


def test_c1_shapes(cd):
    X, Y = synth.config_inputs("c1")
    _full_check(cd, X, Y, tau=0.01)


def test_c2_full(cd):
    X, Y = synth.config_inputs("c2")
    _full_check(cd, X, Y, tau=0.01)


def test_c2_full_per_direction_kernel(cd):
    X, Y = synth.config_inputs("c2")
    old = cd.set_forward_mode(1)
    try:
        _full_check(cd, X, Y, tau=0.01)
    finally:
        cd.set_forward_mode(old)


def test_c3_full(cd):
    """The headline config (the one naming F@0.01) on EVERY row of both directions: distances and
    indices vs the fp64 oracle (R12/R13), distance bits and indices vs the fp32 mirror, partials,
    CD_b and loss within 1e-5, hit counts inside the R16 band, F at the GPU's counts, and the
    backward (random upstream) bit-identical to the oracle's; then the loss gradient."""
    X, Y = synth.config_inputs("c3")
    d_xy, i_xy, d_yx, i_yx, part = _full_check(cd, X, Y, tau=0.01)
    B, N, M = X.shape[0], X.shape[1], Y.shape[1]
    x = torch.from_numpy(X).cuda()
    y = torch.from_numpy(Y).cuda()
    gx, gy = cd.backward(x, y, torch.from_numpy(i_xy).cuda(), torch.from_numpy(i_yx).cuda(),
                         g_scalar=1.0 / (B * N), h_scalar=1.0 / (B * M))
    gxr, gyr, sx, sy = oracle.backward(X, Y, i_xy, i_yx, g_scalar=np.float32(1.0 / (B * N)),
                                       h_scalar=np.float32(1.0 / (B * M)))
    np.testing.assert_array_equal(gx.cpu().numpy(), gxr.astype(np.float32))
    np.testing.assert_array_equal(gy.cpu().numpy(), gyr.astype(np.float32))
    gate_grad(gx.cpu().numpy(), gxr, sx)
    gate_grad(gy.cpu().numpy(), gyr, sy)


@pytest.mark.parametrize("name,nrows", [("c4", 3000), ("c5", 600)])
def test_large_configs_sampled(cd, name, nrows):
    X, Y = synth.config_inputs(name)
    x, y, (d_xy, i_xy, d_yx, i_yx, part) = _run(cd, X, Y, tau=0.01)
    B, N, M = X.shape[0], X.shape[1], Y.shape[1]
    rng = np.random.default_rng(4)
    rows_x = np.unique(np.concatenate([rng.choice(B * N, nrows, replace=False), [0, N - 1, B * N - 1]]))
    rows_y = np.unique(np.concatenate([rng.choice(B * M, nrows, replace=False), [0, M - 1, B * M - 1]]))
    gate_forward_batch(X, Y, d_xy, i_xy, d_yx, i_yx, rows_x=rows_x, rows_y=rows_y)
    gate_mirror(X, Y, d_xy, i_xy, rows=rows_x)
    # properties that hold at any size: indices in range, distance = |x - y_idx|^2 in fp32 mirror order
    assert i_xy.min() >= 0 and i_xy.max() < M and i_yx.min() >= 0 and i_yx.max() < N
    b = np.repeat(np.arange(B), N)
    dd = X.reshape(-1, 3).astype(np.float64) - Y[b, i_xy.reshape(-1)].astype(np.float64)
    np.testing.assert_allclose(d_xy.reshape(-1), (dd * dd).sum(1), rtol=RTOL)
    np.testing.assert_allclose(part[:, 0], d_xy.astype(np.float64).sum(1), rtol=1e-12)
    # backward on the full problem vs the oracle backward (O(N+M), cheap at any size)
    gx, gy = cd.backward(x, y, torch.from_numpy(i_xy).cuda(), torch.from_numpy(i_yx).cuda(),
                         g_scalar=1.0 / (B * N), h_scalar=1.0 / (B * M))
    gxr, gyr, sx, sy = oracle.backward(X, Y, i_xy, i_yx, g_scalar=np.float32(1.0 / (B * N)),
                                       h_scalar=np.float32(1.0 / (B * M)))
    np.testing.assert_array_equal(gx.cpu().numpy(), gxr.astype(np.float32))
    np.testing.assert_array_equal(gy.cpu().numpy(), gyr.astype(np.float32))


def test_c4_every_row_fp32_mirror(cd):
    """c4 (B=8, N=M=100,000) on EVERY row of both directions against the fp32 mirror of DESIGN.md
    §4.2's op order (oracle/, written from the formula): distance bits and indices identical, ties
    included (the mirror takes the lowest index in the same fp32 arithmetic)."""
    X, Y = synth.config_inputs("c4")
    x, y, (d_xy, i_xy, d_yx, i_yx, part) = _run(cd, X, Y, tau=0.01)
    gate_mirror(X, Y, d_xy, i_xy)
    gate_mirror(Y, X, d_yx, i_yx)


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_large_configs_all_points_kdtree(cd, name):
    """Every point of c4 / c5 (not a sample): the GPU minimum equals the exact nearest-neighbour
    distance from scipy's cKDTree (fp64, k=2) within 1e-5 relative, and the index is exact wherever
    the top-2 gap exceeds 1e-6 relative (SURVEY §8.c.4 "large configs"; readings R12, R13); the
    pruned forward reproduces the brute force's d / idx / hit counts on every point; loss, CD_b and the hit counts
    (R16 band) / F from the exact distances."""
    from scipy.spatial import cKDTree
    X, Y = synth.config_inputs(name)
    x, y, (d_xy, i_xy, d_yx, i_yx, part) = _run(cd, X, Y, tau=0.01)
    # the pruned path on every point of the same problem: bit for bit the brute force's results
    pr = [t.cpu().numpy() for t in cd.forward(x, y, tau=0.01, algorithm="pruned")]
    for a, b in zip(pr[:4], (d_xy, i_xy, d_yx, i_yx)):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(pr[4][:, 2:], part[:, 2:])
    refs = []
    for Q, T, d, i in ((X, Y, d_xy, i_xy), (Y, X, d_yx, i_yx)):
        ref_d = []
        for b in range(Q.shape[0]):
            dist, idx = cKDTree(T[b].astype(np.float64)).query(Q[b].astype(np.float64), k=2, workers=-1)
            d1, d2 = dist[:, 0] ** 2, dist[:, 1] ** 2
            np.testing.assert_allclose(d[b].astype(np.float64), d1, rtol=RTOL, atol=0)
            clear = (d2 - d1) > GAP * d1
            np.testing.assert_array_equal(i[b][clear], idx[clear, 0])
            ref_d.append(d1)
        refs.append(np.stack(ref_d))
    # loss, hit counts inside the R16 band and F at the GPU's counts, from the exact distances
    B, N, M = X.shape[0], X.shape[1], Y.shape[1]
    cdb, loss, F, P, R = cd.finalize(torch.from_numpy(part).cuda(), N, M)
    cd_ref, loss_ref = oracle.chamfer_loss(refs[0], refs[1])
    assert abs(loss.item() - loss_ref) <= RTOL * loss_ref
    np.testing.assert_allclose(cdb.cpu().numpy(), cd_ref, rtol=RTOL)
    t2 = oracle.tau_sq(0.01)
    for dist, hits in ((refs[0], part[:, 2]), (refs[1], part[:, 3])):
        lo = (dist < t2 * (1 - GAP)).sum(1)
        hi = (dist <= t2 * (1 + GAP)).sum(1)
        assert np.all((hits >= lo) & (hits <= hi))
    np.testing.assert_allclose(F.cpu().numpy(), oracle.fscore_from_hits(part[:, 2], part[:, 3], N, M),
                               rtol=RTOL, atol=1e-7)


# ------------------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("N,M", [(1, 1), (1, 5000), (5000, 1), (3, 7), (1000, 1024), (2049, 513), (4097, 2047)])
def test_ragged_sizes(cd, N, M):
    X, Y = synth.uniform_pair(2, N, M, seed=N * 31 + M)
    _full_check(cd, X, Y, tau=0.1)


def test_identical_clouds(cd):
    X, _ = synth.shape_pair(2, 3000, 10, config_index=20)
    d_xy, i_xy, d_yx, i_yx, part = _full_check(cd, X, X.copy(), tau=0.0)
    assert np.all(d_xy == 0) and np.all(d_yx == 0)
    np.testing.assert_array_equal(i_xy, np.tile(np.arange(3000), (2, 1)))
    assert np.all(part[:, 2] == 3000)


def test_duplicates_lowest_index(cd):
    rng = np.random.default_rng(8)
    base = rng.uniform(-0.5, 0.5, size=(1, 1500, 3)).astype(np.float32)
    Y = np.concatenate([base, base[:, ::-1]], axis=1)   # every point twice; first copy lowest
    x, y, (d_xy, i_xy, d_yx, i_yx, part) = _run(cd, base, Y)
    np.testing.assert_array_equal(i_xy[0], np.arange(1500))
    assert np.all(d_xy == 0)
    # each Y point's nearest X is itself (lowest index among exact ties = the unique copy)
    np.testing.assert_array_equal(i_yx[0], np.concatenate([np.arange(1500), np.arange(1500)[::-1]]))


def test_lattice_exact_ties(cd):
    h = 2.0 ** -5
    k = np.arange(16)
    g = np.stack(np.meshgrid(k, k, k, indexing="ij"), -1).reshape(-1, 3) * h
    X = g[None].astype(np.float32)
    # queries at cell centres: 8 lattice points at exactly equal distance -> lowest index wins
    Q = (g[:500] + h / 2)[None].astype(np.float32)
    x, y, (d_xy, i_xy, _, _, _) = _run(cd, Q, X)
    d1, i1, d2 = oracle.nn(Q, X)
    np.testing.assert_array_equal(i_xy, i1)
    np.testing.assert_array_equal(d_xy.astype(np.float64), d1)
    gate_mirror(Q, X, d_xy, i_xy)


def test_clustered_far_long_segments(cd):
    # all X near one Y point: one segment of length N in the backward (degenerate scatter)
    rng = np.random.default_rng(9)
    Y = rng.uniform(-0.5, 0.5, size=(1, 2000, 3)).astype(np.float32)
    X = (Y[:, :1] + 10.0 + rng.normal(scale=1e-3, size=(1, 5000, 3))).astype(np.float32)
    _full_check(cd, X, Y, tau=0.01)


def test_scaling_invariance_bit_exact(cd):
    X, Y = synth.shape_pair(2, 2000, 1800, config_index=21)
    _, _, a = _run(cd, X, Y)
    _, _, b = _run(cd, X * np.float32(4.0), Y * np.float32(4.0))
    np.testing.assert_array_equal(b[1], a[1])
    np.testing.assert_array_equal(b[0], a[0] * np.float32(16.0))


# ------------------------------------------------------------------------------ determinism
def test_rerun_and_split_independence(cd):
    X, Y = synth.shape_pair(3, 5000, 7000, config_index=22)
    _, _, ref = _run(cd, X, Y, tau=0.01)
    for _ in range(2):
        _, _, again = _run(cd, X, Y, tau=0.01)
        for a, b in zip(ref[:4], again[:4]):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(ref[4], again[4])
    for s in (1, 2, 3, 7, 14):
        old = cd.set_forward_splits(s)
        try:
            _, _, out = _run(cd, X, Y, tau=0.01)
        finally:
            cd.set_forward_splits(old)
        for a, b in zip(ref[:4], out[:4]):
            np.testing.assert_array_equal(a, b)


def test_query_slices_match_full(cd):
    X, Y = synth.shape_pair(2, 6000, 5000, config_index=23)
    x, y, full = _run(cd, X, Y, tau=0.01)
    parts = np.zeros((2, 4))
    for (q0, q1), (r0, r1) in (((0, 2500), (0, 1)), ((2500, 6000), (1, 5000))):
        out = cd.forward(x, y, tau=0.01, q_slice=(q0, q1), r_slice=(r0, r1))
        torch.cuda.synchronize()
        o = [t.cpu().numpy() for t in out]
        np.testing.assert_array_equal(o[0], full[0][:, q0:q1])
        np.testing.assert_array_equal(o[1], full[1][:, q0:q1])
        np.testing.assert_array_equal(o[2], full[2][:, r0:r1])
        np.testing.assert_array_equal(o[3], full[3][:, r0:r1])
        parts += o[4]
    np.testing.assert_allclose(parts, full[4], rtol=1e-12)
    np.testing.assert_array_equal(parts[:, 2:], full[4][:, 2:])


def test_backward_slices_match_full(cd):
    X, Y = synth.shape_pair(2, 3000, 2500, config_index=24)
    x, y, (d_xy, i_xy, d_yx, i_yx, _) = _run(cd, X, Y)
    ixy, iyx = torch.from_numpy(i_xy).cuda(), torch.from_numpy(i_yx).cuda()
    gx, gy = cd.backward(x, y, ixy, iyx, g_scalar=0.5, h_scalar=0.25)
    sx, sy = cd.backward(x, y, ixy, iyx, g_scalar=0.5, h_scalar=0.25, q_slice=(1000, 2000), r_slice=(7, 2500))
    np.testing.assert_array_equal(sx.cpu().numpy(), gx.cpu().numpy()[:, 1000:2000])
    np.testing.assert_array_equal(sy.cpu().numpy(), gy.cpu().numpy()[:, 7:2500])


def test_backward_slices_radix_path(cd):
    """Clouds above the on-chip limit (global radix passes + the edge-major gradient pass): sliced
    outputs equal the full backward's rows, and the full backward equals the oracle bit for bit with a
    per-point upstream (weights indexed by source row) and with the loss fill."""
    rng = np.random.default_rng(91)
    B, N, M = 2, 30011, 26003
    X = rng.normal(size=(B, N, 3)).astype(np.float32)
    Y = rng.normal(size=(B, M, 3)).astype(np.float32)
    ixy = (M * rng.random(size=(B, N)) ** 2).astype(np.int32)
    iyx = rng.integers(0, N, size=(B, M)).astype(np.int32)
    iyx[1, :100] = N - 1                            # the last target of a segment with many sources
    g = rng.normal(size=(B, N)).astype(np.float32)
    h = rng.normal(size=(B, M)).astype(np.float32)
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    ti, tj = torch.from_numpy(ixy).cuda(), torch.from_numpy(iyx).cuda()
    gx, gy = cd.backward(x, y, ti, tj, torch.from_numpy(g).cuda(), torch.from_numpy(h).cuda())
    sx, sy = cd.backward(x, y, ti, tj, torch.from_numpy(g).cuda(), torch.from_numpy(h).cuda(),
                         q_slice=(7000, 19000), r_slice=(0, 13))
    torch.cuda.synchronize()
    gxr, gyr, _, _ = oracle.backward(X, Y, ixy, iyx, g, h)
    np.testing.assert_array_equal(gx.cpu().numpy(), gxr.astype(np.float32))
    np.testing.assert_array_equal(gy.cpu().numpy(), gyr.astype(np.float32))
    np.testing.assert_array_equal(sx.cpu().numpy(), gx.cpu().numpy()[:, 7000:19000])
    np.testing.assert_array_equal(sy.cpu().numpy(), gy.cpu().numpy()[:, 0:13])


@pytest.mark.parametrize("N,M", [(24576, 700), (24577, 700), (3, 24576), (5000, 24577)])
def test_backward_segment_sort_boundary(cd, N, M):
    """max(N, M) <= 24576 sorts each (direction, batch) segment on chip (seg_sort_grad_kernel), larger
    clouds take the global radix passes: both against the oracle bit for bit, with skewed in-degree
    (many sources on few targets) and a single-target segment."""
    rng = np.random.default_rng(N + 7 * M)
    B = 2
    X = rng.normal(size=(B, N, 3)).astype(np.float32)
    Y = rng.normal(size=(B, M, 3)).astype(np.float32)
    ixy = (M * rng.random(size=(B, N)) ** 4).astype(np.int32)
    iyx = (N * rng.random(size=(B, M)) ** 4).astype(np.int32)
    ixy[1] = M - 1                                   # batch 1: every x on one y
    g = rng.normal(size=(B, N)).astype(np.float32)
    h = rng.normal(size=(B, M)).astype(np.float32)
    gx, gy = cd.backward(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), torch.from_numpy(ixy).cuda(),
                         torch.from_numpy(iyx).cuda(), torch.from_numpy(g).cuda(), torch.from_numpy(h).cuda())
    torch.cuda.synchronize()
    gxr, gyr, _, _ = oracle.backward(X, Y, ixy, iyx, g, h)
    np.testing.assert_array_equal(gx.cpu().numpy(), gxr.astype(np.float32))
    np.testing.assert_array_equal(gy.cpu().numpy(), gyr.astype(np.float32))


@pytest.mark.parametrize("B", [5, 12, 32, 40])
def test_backward_segment_sort_parts(cd, B):
    """The on-chip segment sort splits each (direction, batch) segment over 2^lparts CTAs while the
    2B segments alone leave SMs idle (nn_backward.cu): on 148 SMs B = 5 -> 3 (the cap), 12 -> 2,
    32 -> 1, 40 -> 0.  Every split against the oracle bit for bit, near the on-chip limit (24576)
    with skewed in-degree and one batch element whose sources all land on one target."""
    rng = np.random.default_rng(100 + B)
    N, M = 24000, 23001
    X = rng.normal(size=(B, N, 3)).astype(np.float32)
    Y = rng.normal(size=(B, M, 3)).astype(np.float32)
    ixy = (M * rng.random(size=(B, N)) ** 3).astype(np.int32)
    iyx = (N * rng.random(size=(B, M)) ** 5).astype(np.int32)
    ixy[B // 2] = 17
    g = rng.normal(size=(B, N)).astype(np.float32)
    h = rng.normal(size=(B, M)).astype(np.float32)
    gx, gy = cd.backward(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), torch.from_numpy(ixy).cuda(),
                         torch.from_numpy(iyx).cuda(), torch.from_numpy(g).cuda(), torch.from_numpy(h).cuda())
    torch.cuda.synchronize()
    gxr, gyr, _, _ = oracle.backward(X, Y, ixy, iyx, g, h)
    np.testing.assert_array_equal(gx.cpu().numpy(), gxr.astype(np.float32))
    np.testing.assert_array_equal(gy.cpu().numpy(), gyr.astype(np.float32))


def test_vjp_linearity_bit_exact(cd):
    X, Y = synth.shape_pair(1, 4000, 3000, config_index=25)
    x, y, (d_xy, i_xy, d_yx, i_yx, _) = _run(cd, X, Y)
    rng = np.random.default_rng(1)
    g = torch.from_numpy(rng.normal(size=(1, 4000)).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.normal(size=(1, 3000)).astype(np.float32)).cuda()
    ixy, iyx = torch.from_numpy(i_xy).cuda(), torch.from_numpy(i_yx).cuda()
    a = cd.backward(x, y, ixy, iyx, g, h)
    b = cd.backward(x, y, ixy, iyx, 2 * g, 2 * h)
    assert torch.equal(b[0], 2 * a[0]) and torch.equal(b[1], 2 * a[1])


# ------------------------------------------------------------------------------ API layers
def test_fscore_from_distances_matches_fused(cd):
    X, Y = synth.shape_pair(4, 3000, 3500, config_index=26)
    x, y, (d_xy, i_xy, d_yx, i_yx, part) = _run(cd, X, Y, tau=0.01)
    F, P, R = cd.fscore_from_distances(torch.from_numpy(d_xy).cuda(), torch.from_numpy(d_yx).cuda(), 0.01)
    _, _, F2, P2, R2 = cd.finalize(torch.from_numpy(part).cuda(), 3000, 3500)
    torch.cuda.synchronize()
    assert torch.equal(F, F2) and torch.equal(P, P2) and torch.equal(R, R2)
    ref = oracle.fscore(d_xy, d_yx, 0.01)
    np.testing.assert_allclose(F.cpu().numpy(), ref["fscore"], rtol=RTOL)


def test_step_host_matches_device_path(cd):
    X, Y = synth.shape_pair(2, 2048, 1536, config_index=27)
    out = cd.step_host(cd.pinned_copy(X).numpy(), cd.pinned_copy(Y).numpy(), tau=0.01)
    ref = oracle.chamfer(X, Y, tau=0.01)
    assert abs(float(out["loss"][0]) - ref["loss"]) <= RTOL * ref["loss"]
    np.testing.assert_allclose(out["fscore"].numpy(), ref["fscore"], rtol=RTOL)
    x, y, (d_xy, i_xy, d_yx, i_yx, _) = _run(cd, X, Y)
    gx, gy = cd.backward(x, y, torch.from_numpy(i_xy).cuda(), torch.from_numpy(i_yx).cuda(),
                         g_scalar=np.float32(1.0 / (2 * 2048)), h_scalar=np.float32(1.0 / (2 * 1536)))
    np.testing.assert_array_equal(out["grad_x"].numpy(), gx.cpu().numpy())
    np.testing.assert_array_equal(out["grad_y"].numpy(), gy.cpu().numpy())


def test_autograd_loss_and_grad(cd):
    X, Y = synth.shape_pair(2, 1500, 1700, config_index=28)
    x = torch.from_numpy(X).cuda().requires_grad_(True)
    y = torch.from_numpy(Y).cuda().requires_grad_(True)
    loss = cd.chamfer(x, y, 0.5, 2.0)
    loss.backward()
    ref = oracle.chamfer(X, Y, 0.5, 2.0)
    assert abs(loss.item() - ref["loss"]) <= RTOL * ref["loss"]
    gxr, gyr, sx, sy = oracle.loss_grad(X, Y, ref["idx_xy"], ref["idx_yx"], 0.5, 2.0)
    gate_grad(x.grad.cpu().numpy(), gxr, sx)
    gate_grad(y.grad.cpu().numpy(), gyr, sy)


def test_errors_raise(cd):
    from paper_1911_05063_b200._lib import CdError
    x = torch.zeros((1, 0, 3), device="cuda")
    y = torch.zeros((1, 4, 3), device="cuda")
    with pytest.raises(CdError):
        cd.forward(x, y)
    with pytest.raises(TypeError):
        cd.forward(torch.zeros((1, 4, 3)), y)   # CPU tensor: no fallback


# ------------------------------------------------------------------------------ fused vs per-direction
@pytest.mark.parametrize("B,N,M", [(1, 1, 1), (2, 3, 7), (2, 1000, 1024), (3, 2049, 4097), (1, 5000, 1),
                                   (4, 8192, 3000), (32, 2048, 2048), (8, 4096, 1000), (2, 300, 70000)])
def test_fused_equals_unfused_bitwise(cd, B, N, M):
    """Also covers the fused kernel's block-granular target splits (small M: partial tiles) and the
    tile-granular ones (large M)."""
    X, Y = synth.shape_pair(B, N, M, config_index=40 + N % 7)
    _, _, fused = _run(cd, X, Y, tau=0.01)
    old = cd.set_forward_mode(1)
    try:
        _, _, unf = _run(cd, X, Y, tau=0.01)
    finally:
        cd.set_forward_mode(old)
    for a, b in zip(fused[:4], unf[:4]):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_allclose(fused[4], unf[4], rtol=1e-12)
    np.testing.assert_array_equal(fused[4][:, 2:], unf[4][:, 2:])


def test_pack_alignment_paths_agree(cd):
    """pack_kernel reads four points per thread with 16-byte loads when a cloud is 16-B aligned with
    n % 4 == 0, and one point per thread otherwise: the same clouds at a 4-B offset (scalar path) give
    bit-identical results."""
    X, Y = synth.shape_pair(3, 4096, 2048, config_index=46)
    x = torch.from_numpy(X).cuda()
    y = torch.from_numpy(Y).cuda()
    bx = torch.empty(x.numel() + 1, dtype=torch.float32, device="cuda")
    by = torch.empty(y.numel() + 1, dtype=torch.float32, device="cuda")
    xm = bx[1:].view(x.shape)
    ym = by[1:].view(y.shape)
    xm.copy_(x)
    ym.copy_(y)
    assert xm.data_ptr() % 16 != 0 and ym.data_ptr() % 16 != 0
    a = cd.forward(x, y, tau=0.01)
    m = cd.forward(xm, ym, tau=0.01)
    for p, q in zip(a, m):
        assert torch.equal(p, q)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_rows_cols_sharding_emulated(cd, world):
    """Query sharding on one GPU: every 'rank' runs cd_forward_rows on its X slice, the column keys
    are combined with an element-wise MIN (what the NCCL all-reduce does), each rank resolves its
    Y slice with cd_forward_cols.  Per-point results must equal the 1-GPU forward bit for bit."""
    from paper_1911_05063_b200.distributed import shard_range
    X, Y = synth.shape_pair(2, 5000, 4100, config_index=50)
    x, y, full = _run(cd, X, Y, tau=0.01)
    B, N, M = 2, 5000, 4100
    keys = None
    rows = []
    part = torch.zeros((B, 4), dtype=torch.float64, device="cuda")
    for r in range(world):
        d, i, k, p = cd.forward_rows(x, y, shard_range(N, r, world), tau=0.01)
        rows.append((d, i))
        part += p
        keys = k if keys is None else torch.minimum(keys, k)
    cols = []
    for r in range(world):
        d, i, p = cd.forward_cols(x, y, keys, shard_range(M, r, world), tau=0.01)
        cols.append((d, i))
        part += p
    torch.cuda.synchronize()
    np.testing.assert_array_equal(torch.cat([d for d, _ in rows], 1).cpu().numpy(), full[0])
    np.testing.assert_array_equal(torch.cat([i for _, i in rows], 1).cpu().numpy(), full[1])
    np.testing.assert_array_equal(torch.cat([d for d, _ in cols], 1).cpu().numpy(), full[2])
    np.testing.assert_array_equal(torch.cat([i for _, i in cols], 1).cpu().numpy(), full[3])
    np.testing.assert_allclose(part.cpu().numpy(), full[4], rtol=1e-12)
    np.testing.assert_array_equal(part.cpu().numpy()[:, 2:], full[4][:, 2:])


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_cols_peers_fused_reduce(cd, world):
    """cd_forward_cols_peers (the column-key all-reduce fused into the resolve: MIN over the ranks'
    key arrays as they are read) on one GPU with each emulated rank's keys in its own array: every
    rank's Y slice equals cd_forward_cols on the MIN-reduced keys and the full forward, bit for bit;
    the partials' columns 1 and 3 as well."""
    from paper_1911_05063_b200.distributed import shard_range
    X, Y = synth.shape_pair(2, 5000, 4100, config_index=51)
    x, y, full = _run(cd, X, Y, tau=0.01)
    B, N, M = 2, 5000, 4100
    keys = []
    for r in range(world):
        kr = torch.empty((B, M), dtype=torch.int64, device="cuda")
        cd.forward_rows(x, y, shard_range(N, r, world), tau=0.01, keys=kr)
        keys.append(kr)
    red = keys[0].clone()
    for k in keys[1:]:
        red = torch.minimum(red, k)
    dcat, icat = [], []
    for r in range(world):
        sl = shard_range(M, r, world)
        d1, i1, p1 = cd.forward_cols_peers(x, y, keys, sl, tau=0.01)
        d2, i2, p2 = cd.forward_cols(x, y, red, sl, tau=0.01)
        assert torch.equal(d1, d2) and torch.equal(i1, i2) and torch.equal(p1, p2)
        dcat.append(d1)
        icat.append(i1)
    np.testing.assert_array_equal(torch.cat(dcat, 1).cpu().numpy(), full[2])
    np.testing.assert_array_equal(torch.cat(icat, 1).cpu().numpy(), full[3])
    # raw device pointers are accepted too (peer buffers), and bad counts are rejected
    d3, i3, _ = cd.forward_cols_peers(x, y, [k.data_ptr() for k in keys], (0, M), tau=0.01)
    np.testing.assert_array_equal(d3.cpu().numpy(), full[2])
    with pytest.raises(Exception):
        cd.forward_cols_peers(x, y, [], (0, M))


# ------------------------------------------------------------------------------ exact pruned path (NEXT-2)
def _check_pruned_vs_brute(cd, X, Y, tau=0.01):
    """cd_forward_pruned must give the brute-force results bit for bit: distances, and indices
    including the lowest index among exactly equal distances (R3': ties across blocks
    of the Hilbert order are re-solved by a full scan of the row)."""
    x, y, brute = _run(cd, X, Y, tau=tau)
    pr = [t.cpu().numpy() for t in cd.forward(x, y, tau=tau, algorithm="pruned")]
    torch.cuda.synchronize()
    for dk, ik in ((0, 1), (2, 3)):
        np.testing.assert_array_equal(pr[dk].view(np.uint32), brute[dk].view(np.uint32))
        np.testing.assert_array_equal(pr[ik], brute[ik])
    np.testing.assert_allclose(pr[4], brute[4], rtol=1e-12)
    np.testing.assert_array_equal(pr[4][:, 2:], brute[4][:, 2:])
    return brute, pr


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_pruned_equals_brute_configs(cd, name):
    X, Y = synth.config_inputs(name)
    brute, pr = _check_pruned_vs_brute(cd, X, Y)
    # random surface samples have no exact ties: indices identical
    np.testing.assert_array_equal(pr[1], brute[1])
    np.testing.assert_array_equal(pr[3], brute[3])


@pytest.mark.parametrize("B,N,M", [(1, 1, 1), (2, 3, 7), (1, 1, 5000), (2, 5000, 1), (3, 2049, 4097),
                                   (2, 100000, 30000), (3, 30001, 25999)])
def test_pruned_ragged(cd, B, N, M):
    X, Y = synth.shape_pair(B, N, M, config_index=70 + N % 5)
    _check_pruned_vs_brute(cd, X, Y)


def test_pruned_adversarial(cd):
    rng = np.random.default_rng(12)
    # uniform cube (poor culling), duplicates (exact ties), clustered far away, identical clouds
    X, Y = synth.uniform_pair(2, 6000, 5000, seed=5)
    _check_pruned_vs_brute(cd, X, Y)
    base = rng.uniform(-0.5, 0.5, size=(1, 3000, 3)).astype(np.float32)
    _check_pruned_vs_brute(cd, base, np.concatenate([base, base[:, ::-1]], axis=1))
    Yc = rng.uniform(-0.5, 0.5, size=(1, 4000, 3)).astype(np.float32)
    Xc = (Yc[:, :1] + 10.0 + rng.normal(scale=1e-3, size=(1, 3000, 3))).astype(np.float32)
    _check_pruned_vs_brute(cd, Xc, Yc)
    S, _ = synth.shape_pair(2, 4000, 10, config_index=71)
    _, pr = _check_pruned_vs_brute(cd, S, S.copy(), tau=0.0)
    assert np.all(pr[0] == 0)
    k = np.arange(12)
    g = (np.stack(np.meshgrid(k, k, k, indexing="ij"), -1).reshape(-1, 3) * 2.0 ** -5)[None].astype(np.float32)
    _check_pruned_vs_brute(cd, (g[:, :700] + 2.0 ** -6).astype(np.float32), g)   # exact 8-way ties


@pytest.mark.parametrize("B,N,M", [(1, 2000, 1800), (2, 30000, 26000)])
def test_pruned_nonfinite(cd, B, N, M):
    """Non-finite coordinates (R6): the pruned path (on-chip and global-radix Hilbert sorts) returns
    what the brute force returns — NaN distances never win, an all-+inf row is (+inf, -1)."""
    X, Y = synth.shape_pair(B, N, M, config_index=74)
    X = X.copy()
    Y = Y.copy()
    X[0, 5] = np.nan
    X[0, 7, 1] = np.inf
    Y[0, 11] = np.nan
    Y[0, 13, 2] = -np.inf
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    brute = [t.cpu().numpy() for t in cd.forward(x, y, tau=0.01)]
    pr = [t.cpu().numpy() for t in cd.forward(x, y, tau=0.01, algorithm="pruned")]
    for k in range(4):
        np.testing.assert_array_equal(pr[k], brute[k])   # NaN == NaN for assert_array_equal
    np.testing.assert_array_equal(pr[4][:, 2:], brute[4][:, 2:])


def test_pruned_large_sampled(cd):
    X, Y = synth.config_inputs("c5")
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    pr = [t.cpu().numpy() for t in cd.forward(x, y, tau=0.01, algorithm="pruned")]
    B, N, M = X.shape[0], X.shape[1], Y.shape[1]
    rng = np.random.default_rng(6)
    rows = np.unique(np.concatenate([rng.choice(B * N, 400, replace=False), [0, N - 1, B * N - 1]]))
    d1, i1, d2 = oracle.nn(X, Y, rows=rows)
    dm, im = oracle.mirror_nn_f32(X, Y, rows=rows)
    np.testing.assert_array_equal(pr[0].reshape(-1)[rows], dm)
    clear = (d2 - d1) > 1e-6 * d1
    np.testing.assert_array_equal(pr[1].reshape(-1)[rows][clear], i1[clear])


def test_step_host_overlapped_equals_step_host(cd):
    X, Y = synth.shape_pair(8, 3000, 2500, config_index=29)
    xh, yh = cd.pinned_copy(X), cd.pinned_copy(Y)
    ref = cd.step_host(xh.numpy(), yh.numpy(), tau=0.01, want_grads=True)
    for nchunks, graph, two in ((1, False, True), (2, False, True), (3, False, True), (8, False, True),
                                (None, False, True), (None, True, True), (3, True, True), (4, False, False),
                                (5, True, False)):
        st = cd.HostStepper(8, 3000, 2500, tau=0.01, nchunks=nchunks, graph=graph, two_streams=two)
        for _ in range(2):                      # back-to-back steps reuse the staging buffers
            loss, fs, gx, gy = st.step(xh, yh)
        torch.cuda.synchronize()
        assert float(loss[0]) == float(ref["loss"][0])
        np.testing.assert_array_equal(fs.numpy(), ref["fscore"].numpy())
        np.testing.assert_array_equal(gx.numpy(), ref["grad_x"].numpy())
        np.testing.assert_array_equal(gy.numpy(), ref["grad_y"].numpy())
        assert st.d2h_bytes() == 4 + 4 * 8 + 12 * 8 * (3000 + 2500)
    # the end-to-end gradients are the loss backward of the oracle (g = w1/(B N) fill, R8)
    _, i_xy, _, i_yx = (t.cpu().numpy() for t in cd.forward(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())[:4])
    gxr, gyr, sx, sy = oracle.backward(X, Y, i_xy, i_yx, g_scalar=np.float32(1.0 / (8 * 3000)),
                                       h_scalar=np.float32(1.0 / (8 * 2500)))
    np.testing.assert_array_equal(ref["grad_x"].numpy(), gxr.astype(np.float32))
    np.testing.assert_array_equal(ref["grad_y"].numpy(), gyr.astype(np.float32))


def test_host_stepper_graph_replay_sees_new_inputs(cd):
    """A captured HostStepper replays the H2D copies: new data written into the same pinned buffers
    gives that data's results (graph replay is not a cached output)."""
    X1, Y1 = synth.shape_pair(4, 2000, 1500, config_index=33)
    X2, Y2 = synth.shape_pair(4, 2000, 1500, config_index=34)
    xh, yh = cd.pinned_copy(X1), cd.pinned_copy(Y1)
    st = cd.HostStepper(4, 2000, 1500, tau=0.01, graph=True)
    st.step(xh, yh)
    torch.cuda.synchronize()
    xh.numpy()[...] = X2
    yh.numpy()[...] = Y2
    loss, fs, gx, gy = st.step(xh, yh)
    torch.cuda.synchronize()
    ref = cd.step_host(cd.pinned_copy(X2).numpy(), cd.pinned_copy(Y2).numpy(), tau=0.01, want_grads=True)
    assert float(loss[0]) == float(ref["loss"][0])
    np.testing.assert_array_equal(gx.numpy(), ref["grad_x"].numpy())
    np.testing.assert_array_equal(gy.numpy(), ref["grad_y"].numpy())


def test_loss_backward_device_upstream(cd):
    """cd_loss_backward (the autograd path): the upstream scalar u is read on the device and the fills
    are g = RN32(u * RN32(w1/(B N))), h = RN32(u * RN32(w2/(B M))) (include/cd.h); gradients equal the
    oracle's backward with those fills bit for bit, for u != 1 and unequal weights."""
    X, Y = synth.shape_pair(3, 2100, 1700, config_index=31)
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    _, i_xy, _, i_yx, _ = cd.forward(x, y)
    B, N, M = 3, 2100, 1700
    for u, w1, w2 in ((1.0, 1.0, 1.0), (-2.75, 0.3, 1.7)):
        gl = torch.tensor([u], dtype=torch.float32, device="cuda")
        gx, gy = cd.loss_backward(x, y, i_xy, i_yx, gl, w1, w2)
        # w1, w2 cross the C ABI as fp32; the fill is RN32(w / (B P)) of that value (include/cd.h)
        g = np.float32(u) * np.float32(float(np.float32(w1)) / (B * N))
        h = np.float32(u) * np.float32(float(np.float32(w2)) / (B * M))
        gxr, gyr, sx, sy = oracle.backward(X, Y, i_xy.cpu().numpy(), i_yx.cpu().numpy(), g_scalar=g, h_scalar=h)
        np.testing.assert_array_equal(gx.cpu().numpy(), gxr.astype(np.float32))
        np.testing.assert_array_equal(gy.cpu().numpy(), gyr.astype(np.float32))
    # autograd with a non-unit upstream goes through the same entry point
    xg, yg = x.clone().requires_grad_(True), y.clone().requires_grad_(True)
    (cd.chamfer(xg, yg, 0.3, 1.7) * -2.75).backward()
    np.testing.assert_array_equal(xg.grad.cpu().numpy(), gx.cpu().numpy())
    np.testing.assert_array_equal(yg.grad.cpu().numpy(), gy.cpu().numpy())


def test_auto_algorithm_and_pruned_autograd(cd):
    """algorithm="auto" (pruned for >= 8192-point clouds) and the autograd loss through the pruned
    forward equal the brute force bit for bit (the pruned results are identical, R3')."""
    X, Y = synth.shape_pair(2, 9000, 8500, config_index=81)
    x = torch.from_numpy(X).cuda()
    y = torch.from_numpy(Y).cuda()
    a = [t.cpu().numpy() for t in cd.forward(x, y, tau=0.01, algorithm="auto")]
    b = [t.cpu().numpy() for t in cd.forward(x, y, tau=0.01)]
    for p, q in zip(a[:4], b[:4]):
        np.testing.assert_array_equal(p, q)
    grads = []
    for algo in ("brute", "pruned"):
        xg = x.clone().requires_grad_(True)
        yg = y.clone().requires_grad_(True)
        loss = cd.chamfer(xg, yg, algorithm=algo)
        loss.backward()
        grads.append((loss.item(), xg.grad.cpu().numpy(), yg.grad.cpu().numpy()))
    assert abs(grads[0][0] - grads[1][0]) <= 1e-12 * abs(grads[0][0])
    np.testing.assert_array_equal(grads[0][1], grads[1][1])
    np.testing.assert_array_equal(grads[0][2], grads[1][2])
