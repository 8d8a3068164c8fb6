"""Randomised GPU parity sweep: many seeded (B, N, M, distribution) draws through cd_forward (fused),
the per-direction kernel, cd_forward_pruned and cd_backward, each against the fp64 oracle with the
north-star gate (tests/gpu_helpers.py).  Sizes cross every tile boundary (512 / 2048) and the
ragged tails; distributions include clusters, duplicates and coincident clouds."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
from tests.gpu_helpers import gate_forward_batch, gate_grad, gate_mirror

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1911_05063_b200 import api
    return api


def _draw(rng):
    B = int(rng.integers(1, 5))
    N = int(rng.choice([1, 2, 31, 511, 512, 513, 2047, 2048, 2049, int(rng.integers(1, 6000))]))
    M = int(rng.choice([1, 3, 511, 512, 513, 2049, 4096, int(rng.integers(1, 6000))]))
    kind = rng.choice(["uniform", "clusters", "dups", "scaled", "same"])
    X = rng.uniform(-0.5, 0.5, size=(B, N, 3))
    Y = rng.uniform(-0.5, 0.5, size=(B, M, 3))
    if kind == "clusters":
        c = rng.normal(size=(B, 4, 3))
        X = c[:, rng.integers(0, 4, N)] + 0.01 * rng.normal(size=(B, N, 3))
        Y = c[:, rng.integers(0, 4, M)] + 0.01 * rng.normal(size=(B, M, 3))
    elif kind == "dups":
        Y = X[:, rng.integers(0, N, M)] if N > 0 else Y
    elif kind == "scaled":
        s = 10.0 ** rng.uniform(-3, 3)
        X, Y = X * s, Y * s
    elif kind == "same":
        M = N
        Y = X.copy()
    return X.astype(np.float32), Y.astype(np.float32), str(kind)


@pytest.mark.parametrize("seed", range(24))
def test_random_parity(cd, seed):
    rng = np.random.default_rng(1000 + seed)
    X, Y, kind = _draw(rng)
    B, N, M = X.shape[0], X.shape[1], Y.shape[1]
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    fused = [t.cpu().numpy() for t in cd.forward(x, y, tau=0.05)]
    gate_forward_batch(X, Y, *fused[:4])
    gate_mirror(X, Y, fused[0], fused[1])
    gate_mirror(Y, X, fused[2], fused[3])
    old = cd.set_forward_mode(1)
    try:
        unf = [t.cpu().numpy() for t in cd.forward(x, y, tau=0.05)]
    finally:
        cd.set_forward_mode(old)
    for a, b in zip(fused[:4], unf[:4]):
        np.testing.assert_array_equal(a, b)
    pr = [t.cpu().numpy() for t in cd.forward(x, y, tau=0.05, algorithm="pruned")]
    np.testing.assert_array_equal(pr[0], fused[0])
    np.testing.assert_array_equal(pr[2], fused[2])
    np.testing.assert_array_equal(pr[4][:, 2:], fused[4][:, 2:])
    g = rng.normal(size=(B, N)).astype(np.float32)
    h = rng.normal(size=(B, M)).astype(np.float32)
    gx, gy = cd.backward(x, y, torch.from_numpy(fused[1]).cuda(), torch.from_numpy(fused[3]).cuda(),
                         torch.from_numpy(g).cuda(), torch.from_numpy(h).cuda())
    gxr, gyr, sx, sy = oracle.backward(X, Y, fused[1], fused[3], g, h)
    np.testing.assert_array_equal(gx.cpu().numpy(), gxr.astype(np.float32))
    np.testing.assert_array_equal(gy.cpu().numpy(), gyr.astype(np.float32))
