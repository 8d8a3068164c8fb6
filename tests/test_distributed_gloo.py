"""Multi-process (gloo, CPU) tests of the sharding host logic in paper_1911_05063_b200.distributed,
with the oracle-backed engine standing in for the CUDA kernels.  world_size 2 and 3:
batch sharding (weak scaling, one all-reduce of the B x 4 partials) and query sharding (row /
column split with a MIN all-reduce of the column keys, all-gather of the index slices for the
backward).  Every rank's outputs must equal the matching slice of the single-process result."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, result_q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_05063_b200 import distributed as pd
        from paper_1911_05063_b200 import synth
        from tests.dist_engine import FusedOracleEngine, OracleEngine
        tau = 0.01
        if mode == "batch":
            B = 2
            X, Y = synth.shape_pair(B, 300, 260, config_index=60, b0=rank * B)
            out = pd.batch_sharded_step(OracleEngine(), torch.from_numpy(X), torch.from_numpy(Y), B * world, rank * B,
                                        tau=tau, w1=0.5, w2=2.0)
        elif mode == "batch_strong":   # bench.py's c4 under --gpus N: a fixed batch split over the ranks
            Bg = 5
            b0, b1 = pd.shard_range(Bg, rank, world)
            X, Y = synth.shape_pair(b1 - b0, 300, 260, config_index=62, b0=b0)
            out = pd.batch_sharded_step(OracleEngine(), torch.from_numpy(X), torch.from_numpy(Y), Bg, b0,
                                        tau=tau, w1=0.5, w2=2.0)
        else:
            X, Y = synth.shape_pair(2, 301, 277, config_index=61)
            x, y = torch.from_numpy(X), torch.from_numpy(Y)
            if rank != 0:          # only rank 0 holds the data: the broadcast must deliver it
                x.zero_()
                y.zero_()
            pd.broadcast_clouds(x, y, src=0)
            eng = FusedOracleEngine() if mode in ("query_fused", "query_peer") else OracleEngine()
            peer = None
            if mode == "query_peer":   # the fused-reduce orchestration (peer reads emulated on gloo)
                from tests.dist_engine import GlooPeerKeys
                assert pd.PeerColKeys.create(2, 277, "cpu") is None   # no symmetric memory on gloo
                peer = GlooPeerKeys(2, 277)
            out = pd.query_sharded_step(eng, x, y, tau=tau, w1=0.5, w2=2.0, peer=peer)
        res = {k: (v.numpy() if isinstance(v, torch.Tensor) else v) for k, v in out.items()}
        result_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        rank, res = q.get(timeout=300)
        results[rank] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def _reference(X, Y, tau, w1, w2):
    from tests.dist_engine import OracleEngine
    e = OracleEngine()
    x, y = torch.from_numpy(X), torch.from_numpy(Y)
    d_xy, i_xy, d_yx, i_yx, part = e.forward(x, y, tau=tau)
    cd, loss, F, P, R = e.finalize(part, X.shape[1], Y.shape[1], w1, w2)
    gx, gy = e.backward(x, y, i_xy, i_yx, g_scalar=w1 / (X.shape[0] * X.shape[1]),
                        h_scalar=w2 / (X.shape[0] * Y.shape[1]))
    return dict(d_xy=d_xy.numpy(), idx_xy=i_xy.numpy(), d_yx=d_yx.numpy(), idx_yx=i_yx.numpy(), loss=loss.numpy(),
                fscore=F.numpy(), cd=cd.numpy(), grad_x=gx.numpy(), grad_y=gy.numpy())


@pytest.mark.parametrize("world", [2, 3])
def test_batch_sharded(world):
    from paper_1911_05063_b200 import synth
    res = _run(world, "batch")
    B = 2
    X, Y = synth.shape_pair(B * world, 300, 260, config_index=60)
    ref = _reference(X, Y, 0.01, 0.5, 2.0)
    for r in range(world):
        out = res[r]
        np.testing.assert_allclose(out["loss"], ref["loss"], rtol=1e-12)
        np.testing.assert_allclose(out["fscore"], ref["fscore"], rtol=1e-12)
        np.testing.assert_allclose(out["cd"], ref["cd"], rtol=1e-12)
        sl = slice(r * B, (r + 1) * B)
        np.testing.assert_array_equal(out["idx_xy"], ref["idx_xy"][sl])
        np.testing.assert_array_equal(out["d_yx"], ref["d_yx"][sl])
        np.testing.assert_array_equal(out["grad_x"], ref["grad_x"][sl])
        np.testing.assert_array_equal(out["grad_y"], ref["grad_y"][sl])


@pytest.mark.parametrize("world", [2, 3])
def test_batch_sharded_strong(world):
    """A fixed global batch (B = 5) split over the ranks (strong scaling, bench.py's c4 mode): every
    rank's per-point outputs and gradients equal its slice of the 1-process result, and the loss / F
    (after the partials all-reduce) are the global ones."""
    from paper_1911_05063_b200 import synth
    from paper_1911_05063_b200.distributed import shard_range
    res = _run(world, "batch_strong")
    X, Y = synth.shape_pair(5, 300, 260, config_index=62)
    ref = _reference(X, Y, 0.01, 0.5, 2.0)
    for r in range(world):
        out = res[r]
        b0, b1 = shard_range(5, r, world)
        np.testing.assert_allclose(out["loss"], ref["loss"], rtol=1e-12)
        np.testing.assert_allclose(out["fscore"], ref["fscore"], rtol=1e-12)
        np.testing.assert_array_equal(out["idx_xy"], ref["idx_xy"][b0:b1])
        np.testing.assert_array_equal(out["idx_yx"], ref["idx_yx"][b0:b1])
        np.testing.assert_array_equal(out["grad_x"], ref["grad_x"][b0:b1])
        np.testing.assert_array_equal(out["grad_y"], ref["grad_y"][b0:b1])


@pytest.mark.parametrize("world,mode", [(2, "query_fused"), (3, "query_fused"), (2, "query_slices"),
                                        (2, "query_peer"), (3, "query_peer")])
def test_query_sharded(world, mode):
    from paper_1911_05063_b200 import synth
    from paper_1911_05063_b200.distributed import shard_range
    res = _run(world, mode)
    X, Y = synth.shape_pair(2, 301, 277, config_index=61)
    ref = _reference(X, Y, 0.01, 0.5, 2.0)
    N, M = 301, 277
    for r in range(world):
        out = res[r]
        q0, q1 = shard_range(N, r, world)
        r0, r1 = shard_range(M, r, world)
        assert tuple(out["q_slice"]) == (q0, q1) and tuple(out["r_slice"]) == (r0, r1)
        np.testing.assert_allclose(out["loss"], ref["loss"], rtol=1e-6)
        np.testing.assert_array_equal(out["idx_xy"], ref["idx_xy"][:, q0:q1])
        np.testing.assert_array_equal(out["idx_yx"], ref["idx_yx"][:, r0:r1])
        np.testing.assert_allclose(out["d_yx"], ref["d_yx"][:, r0:r1], rtol=1e-6)
        np.testing.assert_array_equal(out["grad_x"], ref["grad_x"][:, q0:q1])
        np.testing.assert_array_equal(out["grad_y"], ref["grad_y"][:, r0:r1])


def test_shard_ranges_cover_exactly():
    from paper_1911_05063_b200.distributed import shard_range
    for n in (1, 7, 100, 1048576):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
