"""GPU parity of the tensor-core forward (cd_set_forward_mode(3): nn_tc.cu, R27)
against the FP32 fused forward: the tcgen05 MMA only FILTERS (an fp16-split approximation of every
squared distance); every reported distance / index is re-evaluated with the fixed fp32 formula, so
the outputs must equal the fused kernel's bit for bit — including lowest-index ties and the
partials — on every input, plus the oracle gate on sampled rows of c3."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
from paper_1911_05063_b200 import synth
from tests.gpu_helpers import gate_forward_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1911_05063_b200 import api
    return api


def _fwd(cd, X, Y, mode, tau=0.01):
    x = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).cuda()
    y = torch.from_numpy(np.ascontiguousarray(Y, dtype=np.float32)).cuda()
    old = cd.set_forward_mode(mode)
    try:
        out = cd.forward(x, y, tau=tau)
        torch.cuda.synchronize()
    finally:
        cd.set_forward_mode(old)
    return [o.cpu().numpy() for o in out]


def _same(cd, X, Y, tau=0.01):
    f = _fwd(cd, X, Y, 2, tau)
    t = _fwd(cd, X, Y, 3, tau)
    for k in range(4):
        np.testing.assert_array_equal(t[k], f[k])
    np.testing.assert_array_equal(t[4], f[4])
    return t


@pytest.mark.parametrize("B,N,M", [(1, 1, 1), (1, 1, 5000), (2, 5000, 1), (1, 1025, 129), (3, 1000, 2047),
                                   (2, 4097, 3001), (1, 8192, 8192)])
def test_tensor_equals_fused_shapes(cd, B, N, M):
    X, Y = synth.shape_pair(B, N, M, config_index=60 + N % 11)
    _same(cd, X, Y)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_tensor_equals_fused_configs(cd, name):
    X, Y = synth.config_inputs(name)
    _same(cd, X, Y, tau=synth.CONFIGS[name]["tau"])


def test_tensor_adversarial(cd):
    rng = np.random.default_rng(21)
    X, Y = synth.uniform_pair(2, 6000, 5000, seed=9)                       # uniform cube
    _same(cd, X, Y)
    base = rng.uniform(-0.5, 0.5, size=(1, 3000, 3)).astype(np.float32)
    _same(cd, base, np.concatenate([base, base[:, ::-1]], axis=1))           # duplicates: exact ties
    S, _ = synth.shape_pair(2, 4000, 10, config_index=72)
    t = _same(cd, S, S.copy(), tau=0.0)                                       # identical clouds
    assert np.all(t[0] == 0) and np.all(t[1] == np.arange(4000))
    Yc = rng.uniform(-0.5, 0.5, size=(1, 4000, 3)).astype(np.float32)
    Xc = (Yc[:, :1] + 10.0 + rng.normal(scale=1e-3, size=(1, 3000, 3))).astype(np.float32)
    _same(cd, Xc, Yc)                                                         # far cluster (huge scale)
    k = np.arange(12)
    g = (np.stack(np.meshgrid(k, k, k, indexing="ij"), -1).reshape(-1, 3) * 2.0 ** -5)[None].astype(np.float32)
    _same(cd, (g[:, :700] + 2.0 ** -6).astype(np.float32), g)                # exact 8-way ties (band fallback)
    big = (synth.shape_pair(1, 3000, 3000, config_index=73)[0] * 1000.0 + 5000.0).astype(np.float32)
    _same(cd, big, (big[:, ::-1] + 0.5).astype(np.float32))                  # offset / scaled coordinates


def test_tensor_nonfinite(cd):
    X, Y = synth.shape_pair(1, 2000, 1800, config_index=74)
    X = X.copy()
    Y = Y.copy()
    X[0, 5] = np.nan
    X[0, 7, 1] = np.inf
    Y[0, 11] = np.nan
    Y[0, 13, 2] = -np.inf
    _same(cd, X, Y)


def test_tensor_c3_oracle_sampled(cd):
    X, Y = synth.config_inputs("c3")
    t = _same(cd, X, Y)
    B, N = X.shape[:2]
    M = Y.shape[1]
    rng = np.random.default_rng(8)
    rx = rng.choice(B * N, 600, replace=False)
    ry = rng.choice(B * M, 600, replace=False)
    gate_forward_batch(X, Y, t[0], t[1], t[2], t[3], rows_x=rx, rows_y=ry)


def test_all_infinite_column_is_no_candidate(cd):
    """R6 in the column direction of the fused kernel: a Y row whose distances are all +inf (an
    infinite coordinate) has no finite candidate -> (+inf, -1), as the row direction and the oracle."""
    X, Y = synth.shape_pair(1, 300, 200, config_index=75)
    Y = Y.copy()
    Y[0, 13, 2] = -np.inf
    for mode in (1, 2, 3):
        out = _fwd(cd, X, Y, mode)
        assert out[2][0, 13] == np.inf and out[3][0, 13] == -1
    d1, i1, _ = oracle.nn(Y, X, rows=np.array([13]))
    assert d1[0] == np.inf and i1[0] == -1
