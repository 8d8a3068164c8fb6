"""Multi-GPU sharding of the hot path.  One process per GPU,
torch.distributed (NCCL over NVLink on the B200 box; gloo in the CPU tests) for the plumbing.

Two partitionings, both from BASELINE.json's configs:

* batch sharding (c3/c4 style, weak scaling): rank r owns a contiguous block of batch elements.
  The per-point work needs no collective; the only exchange is ONE all-reduce (sum) of the B x 4
  fp64 partial vector (sum d_xy, sum d_yx, hits_xy, hits_yx), after which every rank finalizes the
  global loss / F-score (R18).  Gradients are local.
* query sharding (c5, strong scaling): every rank holds full replicas of X and Y (broadcast from
  rank 0 when the data originates there), searches its slice of X rows against all of Y and its
  slice of Y rows against all of X, all-reduces the partials, and for the backward all-gathers the
  index slices so each rank can build the inverse map and write the gradients of its own rows.
  Per-point outputs and gradients are bit-identical to the 1-GPU run.

The compute is delegated to an ``engine`` with the signatures of ``paper_1911_05063_b200.api``
(forward / finalize / backward); the product passes the CUDA engine (``api``).  Tests pass an
oracle-backed engine so that this host logic is covered on CPU with gloo.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class CollectiveTimer:
    """Optional CUDA-event brackets around every collective of a step (name -> list of (start, end)
    events on the current stream), so a caller can report the time a step spends in collectives.
    The events measure how long the launching stream waits for the collective."""

    def __init__(self):
        self.spans = []

    def __call__(self, name, fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        self.spans.append((name, a, b))
        return r

    def total_ms(self):
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for _, a, b in self.spans)

    def by_name_ms(self):
        torch.cuda.synchronize()
        out = {}
        for n, a, b in self.spans:
            out[n] = out.get(n, 0.0) + a.elapsed_time(b)
        return out

    def reset(self):
        self.spans = []


def _coll(prof, name, fn):
    return prof(name, fn) if prof is not None else fn()


def shard_range(n: int, rank: int, world: int):
    """Balanced contiguous [lo, hi) slice of n items for `rank` of `world`."""
    return (n * rank) // world, (n * (rank + 1)) // world


def _world(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def allreduce_partials(part_local: torch.Tensor, B_global: int, b0: int, group=None, prof=None) -> torch.Tensor:
    """Place the local B_l x 4 partials at rows [b0, b0+B_l) of a zero B_global x 4 tensor and
    all-reduce (sum).  With B_global == B_l and b0 == 0 this is the query-sharded sum."""
    rank, world = _world(group)
    if world == 1 and B_global == part_local.shape[0]:
        return part_local
    full = torch.zeros((B_global, 4), dtype=torch.float64, device=part_local.device)
    full[b0:b0 + part_local.shape[0]] = part_local
    if world > 1:
        _coll(prof, "all_reduce_partials", lambda: dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group))
    return full


def all_gather_rows(local: torch.Tensor, n_total: int, group=None, prof=None) -> torch.Tensor:
    """Gather (B, n_r, ...) row slices produced by shard_range into (B, n_total, ...)."""
    rank, world = _world(group)
    if world == 1:
        return local
    width = -(-n_total // world)
    B = local.shape[0]
    pad = torch.zeros((B, width) + tuple(local.shape[2:]), dtype=local.dtype, device=local.device)
    pad[:, :local.shape[1]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    _coll(prof, "all_gather_idx", lambda: dist.all_gather(bufs, pad, group=group))
    parts = []
    for r in range(world):
        lo, hi = shard_range(n_total, r, world)
        parts.append(bufs[r][:, :hi - lo])
    return torch.cat(parts, dim=1).contiguous()


def broadcast_clouds(x: torch.Tensor, y: torch.Tensor, src: int = 0, group=None, prof=None):
    """Replicate the clouds from `src` (the "target broadcast over NVLink" of config c5)."""
    _, world = _world(group)
    if world > 1:
        _coll(prof, "broadcast_clouds", lambda: (dist.broadcast(x, src=src, group=group),
                                                 dist.broadcast(y, src=src, group=group)))
    return x, y


def batch_sharded_step(engine, x_local, y_local, B_global: int, b0: int, tau=None, w1: float = 1.0,
                       w2: float = 1.0, group=None, backward: bool = True, prof=None):
    """One fwd(+F)+loss+bwd step on this rank's batch block.  Returns a dict with the global loss,
    per-batch CD / F (global), and this rank's per-point outputs and gradients."""
    N, M = x_local.shape[1], y_local.shape[1]
    d_xy, i_xy, d_yx, i_yx, part = engine.forward(x_local, y_local, tau=tau)
    part = allreduce_partials(part, B_global, b0, group, prof)
    cd, loss, F, P, R = engine.finalize(part, N, M, w1, w2)
    out = dict(d_xy=d_xy, idx_xy=i_xy, d_yx=d_yx, idx_yx=i_yx, partials=part, cd=cd, loss=loss, fscore=F,
               precision=P, recall=R)
    if backward:
        gx, gy = engine.backward(x_local, y_local, i_xy, i_yx, g_scalar=w1 / (B_global * N),
                                 h_scalar=w2 / (B_global * M))
        out.update(grad_x=gx, grad_y=gy)
    return out


def allreduce_colkeys(keys: torch.Tensor, group=None, prof=None) -> torch.Tensor:
    """Element-wise MIN of the int64 column keys across ranks (keys are >= 0, so signed MIN is the
    lexicographic (distance, row group) minimum)."""
    _, world = _world(group)
    if world > 1:
        _coll(prof, "all_reduce_min_colkeys", lambda: dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group))
    return keys


class PeerColKeys:
    """The column-key exchange of query sharding without a separate collective: every rank's
    [B, M] int64 key array lives in torch symmetric memory (CUDA peer-mapped over NVLink); each rank's
    cd_forward_rows writes its own array, a cross-device barrier publishes them, and each rank's
    cd_forward_cols_peers reads the keys of ITS Y slice from every array and takes the MIN as it reads
    (the all-reduce fused into the resolve kernel: a reduce-scatter's NVLink traffic, no NCCL call).
    A second barrier before the arrays are rewritten.  create() returns None where symmetric memory is
    unavailable (gloo, one rank, no peer access): callers keep the NCCL all-reduce path."""

    def __init__(self, buf, handle, ptrs):
        self.buf = buf
        self.handle = handle
        self.ptrs = ptrs

    @staticmethod
    def create(B: int, M: int, device, group=None):
        try:
            if not dist.is_initialized() or dist.get_world_size(group) < 2 or dist.get_backend(group) != "nccl":
                return None
            import torch.distributed._symmetric_memory as symm
            grp = group if group is not None else dist.group.WORLD
            if hasattr(symm, "enable_symm_mem_for_group"):
                symm.enable_symm_mem_for_group(grp.group_name)
            buf = symm.empty(B, M, dtype=torch.int64, device=device)
            handle = symm.rendezvous(buf, grp)
            ptrs = [int(p) for p in handle.buffer_ptrs]
            if len(ptrs) != dist.get_world_size(group) or any(p == 0 for p in ptrs):
                return None
            return PeerColKeys(buf, handle, ptrs)
        except Exception:   # no symmetric memory / peer access on this node: the all-reduce path
            return None

    def sources(self):
        return self.ptrs

    def barrier(self):
        self.handle.barrier(channel=0)


def query_sharded_step(engine, x, y, tau=None, w1: float = 1.0, w2: float = 1.0, group=None,
                       backward: bool = True, prof=None, peer=None):
    """One step with query rows split across ranks; x, y are full replicas on every rank.

    Rank r evaluates X rows q_r against all of Y ONCE (fused kernel): its d_xy rows are final and
    it produces column keys for every Y point; an all-reduce MIN of the keys completes the Y
    direction, and each rank resolves its own Y rows r_r.  Work per rank = B*N*M / world."""
    rank, world = _world(group)
    B, N, M = x.shape[0], x.shape[1], y.shape[1]
    q = shard_range(N, rank, world)
    r = shard_range(M, rank, world)
    if peer is not None and hasattr(engine, "forward_cols_peers"):
        # keys into this rank's peer-visible array; barrier; the resolve MIN-reduces every rank's
        # keys of its Y slice as it reads them; barrier before the arrays are written again
        d_xy, i_xy, _, part = engine.forward_rows(x, y, q, tau=tau, keys=peer.buf)
        _coll(prof, "peer_barrier_keys_ready", peer.barrier)
        d_yx, i_yx, part = engine.forward_cols_peers(x, y, peer.sources(), r, tau=tau, partials=part)
        _coll(prof, "peer_barrier_keys_read", peer.barrier)
    elif hasattr(engine, "forward_rows"):
        d_xy, i_xy, keys, part = engine.forward_rows(x, y, q, tau=tau)
        keys = allreduce_colkeys(keys, group, prof)
        d_yx, i_yx, part = engine.forward_cols(x, y, keys, r, tau=tau, partials=part)
    else:
        d_xy, i_xy, d_yx, i_yx, part = engine.forward(x, y, tau=tau, q_slice=q, r_slice=r)
    part = allreduce_partials(part, B, 0, group, prof)
    cd, loss, F, P, R = engine.finalize(part, N, M, w1, w2)
    out = dict(d_xy=d_xy, idx_xy=i_xy, d_yx=d_yx, idx_yx=i_yx, partials=part, cd=cd, loss=loss, fscore=F,
               precision=P, recall=R, q_slice=q, r_slice=r)
    if backward:
        i_xy_full = all_gather_rows(i_xy, N, group, prof)
        i_yx_full = all_gather_rows(i_yx, M, group, prof)
        gx, gy = engine.backward(x, y, i_xy_full, i_yx_full, g_scalar=w1 / (B * N), h_scalar=w2 / (B * M),
                                 q_slice=q, r_slice=r)
        out.update(grad_x=gx, grad_y=gy)
    return out
