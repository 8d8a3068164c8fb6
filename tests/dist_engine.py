"""Oracle-backed stand-in for the CUDA engine, so paper_1911_05063_b200.distributed's host logic
(shard ranges, all-reduce of partials, MIN all-reduce of column keys, all-gather of index slices)
runs under gloo on CPU.  TEST INFRASTRUCTURE: it calls oracle/ and mirrors the C-ABI contracts of
include/cd.h (cd_forward slices, cd_forward_rows / cd_forward_cols keys, cd_finalize,
cd_backward slices) with torch CPU tensors."""
import numpy as np
import torch
import torch.distributed as dist

import oracle

EMPTY = (1 << 63) - 1
GROUP = 16   # rows per column-key group (kR in the kernel; the key's low word is the group's first row)


def _np(t):
    return t.detach().cpu().numpy()


class OracleEngine:
    """Per-direction engine (cd_forward with query slices)."""

    def forward(self, x, y, tau=None, q_slice=None, r_slice=None):
        X, Y = _np(x), _np(y)
        B, N, M = X.shape[0], X.shape[1], Y.shape[1]
        q0, q1 = q_slice or (0, N)
        r0, r1 = r_slice or (0, M)
        dxy, ixy, _ = oracle.nn(X, Y)
        dyx, iyx, _ = oracle.nn(Y, X)
        dxy, ixy, dyx, iyx = dxy[:, q0:q1], ixy[:, q0:q1], dyx[:, r0:r1], iyx[:, r0:r1]
        part = np.zeros((B, 4))
        part[:, 0] = dxy.astype(np.float32).astype(np.float64).sum(1)
        part[:, 1] = dyx.astype(np.float32).astype(np.float64).sum(1)
        if tau is not None:
            t2 = oracle.tau_sq(tau)
            part[:, 2] = (dxy <= t2).sum(1)
            part[:, 3] = (dyx <= t2).sum(1)
        return (torch.from_numpy(dxy.astype(np.float32)), torch.from_numpy(ixy), torch.from_numpy(dyx.astype(np.float32)),
                torch.from_numpy(iyx), torch.from_numpy(part))

    def finalize(self, partials, N, M, w1=1.0, w2=1.0):
        p = _np(partials)
        cd = w1 * p[:, 0] / N + w2 * p[:, 1] / M
        P, R = p[:, 2] / N, p[:, 3] / M
        F = np.where(P + R > 0, 2 * P * R / np.where(P + R > 0, P + R, 1), 0.0)
        return (torch.from_numpy(cd), torch.tensor([cd.mean()]), torch.from_numpy(F), torch.from_numpy(P),
                torch.from_numpy(R))

    def backward(self, x, y, idx_xy, idx_yx, g=None, h=None, g_scalar=0.0, h_scalar=0.0, q_slice=None,
                 r_slice=None):
        X, Y = _np(x), _np(y)
        N, M = X.shape[1], Y.shape[1]
        q0, q1 = q_slice or (0, N)
        r0, r1 = r_slice or (0, M)
        gx, gy, _, _ = oracle.backward(X, Y, _np(idx_xy), _np(idx_yx), None if g is None else _np(g),
                                       None if h is None else _np(h), g_scalar, h_scalar)
        return torch.from_numpy(gx[:, q0:q1].astype(np.float32)), torch.from_numpy(gy[:, r0:r1].astype(np.float32))


class FusedOracleEngine(OracleEngine):
    """Adds the cd_forward_rows / cd_forward_cols contract (column keys)."""

    def forward_rows(self, x, y, q_slice, tau=None, partials=None, keys=None):
        out_keys = keys
        X, Y = _np(x), _np(y)
        B, N, M = X.shape[0], X.shape[1], Y.shape[1]
        q0, q1 = q_slice
        dxy, ixy, _ = oracle.nn(X[:, q0:q1], Y)
        # column keys over the rows of this slice: (f32 bits of min d) << 32 | first row of its group
        dc, ic, _ = oracle.nn(Y, np.ascontiguousarray(X[:, q0:q1]))
        d32 = dc.astype(np.float32)
        row = q0 + ic
        group = q0 + ((row - q0) // GROUP) * GROUP
        keys = (d32.view(np.uint32).astype(np.int64) << 32) | group.astype(np.int64)
        part = np.zeros((B, 4)) if partials is None else _np(partials).copy()
        part[:, 0] = dxy.astype(np.float32).astype(np.float64).sum(1)
        part[:, 2] = (dxy <= oracle.tau_sq(tau)).sum(1) if tau is not None else 0
        kt = torch.from_numpy(keys)
        if out_keys is not None:
            out_keys.copy_(kt)
            kt = out_keys
        return (torch.from_numpy(dxy.astype(np.float32)), torch.from_numpy((ixy + 0).astype(np.int32)),
                kt, torch.from_numpy(part))

    def forward_cols(self, x, y, keys, r_slice, tau=None, partials=None):
        X, Y = _np(x), _np(y)
        B, N, M = X.shape[0], X.shape[1], Y.shape[1]
        r0, r1 = r_slice
        K = _np(keys)[:, r0:r1]
        d = (K >> 32).astype(np.uint32).view(np.float32)
        g = (K & 0xffffffff).astype(np.int64)
        idx = np.empty_like(g, dtype=np.int32)
        for b in range(B):
            for j in range(r1 - r0):
                rows = np.arange(g[b, j], min(g[b, j] + GROUP, N))
                e = ((X[b, rows].astype(np.float64) - Y[b, r0 + j].astype(np.float64)) ** 2).sum(1)
                idx[b, j] = rows[np.argmin(e)]
        part = np.zeros((B, 4)) if partials is None else _np(partials).copy()
        part[:, 1] = d.astype(np.float64).sum(1)
        part[:, 3] = (d <= oracle.tau_sq(tau)).sum(1) if tau is not None else 0
        return torch.from_numpy(d.copy()), torch.from_numpy(idx), torch.from_numpy(part)

    def forward_cols_peers(self, x, y, keys_list, r_slice, tau=None, partials=None):
        """The cd_forward_cols_peers contract: the element-wise MIN of the given key arrays, then
        forward_cols."""
        red = keys_list[0].clone()
        for k in keys_list[1:]:
            red = torch.minimum(red, k)
        return self.forward_cols(x, y, red, r_slice, tau=tau, partials=partials)


class GlooPeerKeys:
    """Test stand-in for distributed.PeerColKeys on gloo/CPU: the peer reads are emulated by an
    all-gather of every rank's key array after the barrier (the orchestration — keys into the
    rank's own array, barrier, MIN-reducing resolve, barrier — is what is tested)."""

    def __init__(self, B, M):
        self.buf = torch.empty((B, M), dtype=torch.int64)

    def barrier(self):
        dist.barrier()

    def sources(self):
        out = [torch.empty_like(self.buf) for _ in range(dist.get_world_size())]
        dist.all_gather(out, self.buf)
        return out
