"""PyTorch-facing API over libcd (argument marshalling only; every step runs in the CUDA kernels).

PyTorch supplies device memory and the current stream.  Inputs must be CUDA fp32 contiguous
(B, N, 3) / (B, M, 3) tensors on an sm_100 device.  Names follow the paper's notation: X is the
prediction cloud, Y the reference cloud; d_xy / idx_xy are the per-point squared distances and
nearest-neighbour indices of X in Y, d_yx / idx_yx the reverse direction.
"""
from __future__ import annotations

import ctypes
import functools

import numpy as np
import torch

from . import _lib
from ._lib import check

_ws_cache: dict = {}


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _device_guard(fn):
    """Run a wrapper with the CUDA device of its tensor arguments current, so libcd's device checks,
    launches and the current stream all refer to the GPU the data lives on; tensors on two different
    GPUs are rejected before any call."""
    @functools.wraps(fn)
    def wrapped(*args, **kw):
        devs = {a.device for a in (*args, *kw.values()) if isinstance(a, torch.Tensor) and a.is_cuda}
        if len(devs) > 1:
            raise ValueError(f"{fn.__name__}: tensors on several devices {sorted(map(str, devs))}")
        if not devs:
            return fn(*args, **kw)
        with torch.cuda.device(devs.pop()):
            return fn(*args, **kw)
    return wrapped


def _cached_ws(kind: str, op: int, n: int, device) -> torch.Tensor:
    """One workspace per (device, current stream, kind, op), grown to the largest size requested:
    calls on one stream are ordered, so they may share it; calls on different streams never do."""
    device = torch.device(device)
    key = (str(device), torch.cuda.current_stream(device).cuda_stream, kind, op)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < n:
        buf = torch.empty(n, dtype=torch.uint8, device=device)  # caching allocator: >= 512-B aligned
        _ws_cache[key] = buf
    return buf


def workspace(op: int, B: int, N: int, M: int, device) -> torch.Tensor:
    """Workspace bytes from cd_workspace_size (see _cached_ws)."""
    n = int(_lib.load().cd_workspace_size(op, B, N, M))
    if n == 0:
        raise _lib.CdError(1, f"invalid sizes B={B} N={N} M={M}")
    return _cached_ws("cd", op, n, device)


def _check_cloud(t, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.float32 or t.dim() != 3 or t.shape[-1] != 3:
        raise TypeError(f"{name} must be fp32 of shape (B, P, 3), got {t.dtype} {tuple(t.shape)}")
    return t.contiguous()


def set_forward_splits(s: int) -> int:
    """Test hook: force the forward's target-split count (0 = auto).  Returns the previous value."""
    return int(_lib.load().cd_set_forward_splits(int(s)))


@_device_guard
def forward(x: torch.Tensor, y: torch.Tensor, tau: float | None = None, q_slice=None, r_slice=None,
            want_partials: bool = True, algorithm: str = "brute"):
    """cd_forward: both NN directions.  Returns (d_xy, idx_xy, d_yx, idx_yx, partials[B,4] fp64).

    q_slice=(q0,q1) / r_slice=(r0,r1) restrict the query rows (query sharding); outputs are
    slice-sized.  algorithm="pruned" uses cd_forward_pruned (exact, culled; full problems only);
    "auto" picks it for full problems with at least 8192 points per cloud (its results equal the brute
    force's bit for bit, R3'), the brute force otherwise."""
    if algorithm == "auto":
        full = q_slice is None and r_slice is None
        algorithm = "pruned" if full and min(x.shape[1], y.shape[1]) >= 8192 else "brute"
    if algorithm == "pruned":
        if q_slice is not None or r_slice is not None:
            raise ValueError("the pruned forward takes the full problem")
        return forward_pruned(x, y, tau=tau, want_partials=want_partials)
    if algorithm != "brute":
        raise ValueError(f"unknown algorithm {algorithm!r}")
    x = _check_cloud(x, "x")
    y = _check_cloud(y, "y")
    B, N, _ = x.shape
    M = y.shape[1]
    if y.shape[0] != B:
        raise ValueError("batch mismatch")
    q0, q1 = q_slice if q_slice is not None else (0, N)
    r0, r1 = r_slice if r_slice is not None else (0, M)
    dev = x.device
    d_xy = torch.empty((B, q1 - q0), dtype=torch.float32, device=dev)
    i_xy = torch.empty((B, q1 - q0), dtype=torch.int32, device=dev)
    d_yx = torch.empty((B, r1 - r0), dtype=torch.float32, device=dev)
    i_yx = torch.empty((B, r1 - r0), dtype=torch.int32, device=dev)
    part = torch.empty((B, 4), dtype=torch.float64, device=dev) if want_partials else None
    ws = workspace(_lib.CD_OP_FORWARD, B, N, M, dev)
    lib = _lib.load()
    check(lib.cd_forward(_ptr(x), _ptr(y), B, N, M, q0, q1, r0, r1, _ptr(d_xy), _ptr(i_xy), _ptr(d_yx), _ptr(i_yx),
                         _ptr(part), float(-1.0 if tau is None else tau), _ptr(ws), ws.numel(), _stream()))
    return d_xy, i_xy, d_yx, i_yx, part


@_device_guard
def forward_pruned(x: torch.Tensor, y: torch.Tensor, tau: float | None = None, want_partials: bool = True):
    """cd_forward_pruned: exact nearest neighbours with Hilbert-ordered tiles and lower-bound culling (same results as the brute force)."""
    x = _check_cloud(x, "x")
    y = _check_cloud(y, "y")
    B, N, _ = x.shape
    M = y.shape[1]
    dev = x.device
    d_xy = torch.empty((B, N), dtype=torch.float32, device=dev)
    i_xy = torch.empty((B, N), dtype=torch.int32, device=dev)
    d_yx = torch.empty((B, M), dtype=torch.float32, device=dev)
    i_yx = torch.empty((B, M), dtype=torch.int32, device=dev)
    part = torch.empty((B, 4), dtype=torch.float64, device=dev) if want_partials else None
    ws = workspace(_lib.CD_OP_FORWARD_PRUNED, B, N, M, dev)
    check(_lib.load().cd_forward_pruned(_ptr(x), _ptr(y), B, N, M, _ptr(d_xy), _ptr(i_xy), _ptr(d_yx), _ptr(i_yx),
                                        _ptr(part), float(-1.0 if tau is None else tau), _ptr(ws), ws.numel(),
                                        _stream()))
    return d_xy, i_xy, d_yx, i_yx, part


def set_forward_mode(mode: int) -> int:
    """Test hook: 0 = automatic (fused bidirectional kernel for full problems), 1 = per-direction
    kernel always, 2 = fused, 3 = tensor-core filter + exact re-scan (full problems).
    Returns the previous value."""
    return int(_lib.load().cd_set_forward_mode(int(mode)))


COLKEY_EMPTY = (1 << 63) - 1


@_device_guard
def forward_rows(x: torch.Tensor, y: torch.Tensor, q_slice, tau: float | None = None, partials=None, keys=None):
    """cd_forward_rows: X rows q_slice fully + column keys for every Y point (query sharding).

    keys: optional [B,M] int64 output tensor (e.g. a symmetric-memory buffer peers read).
    Returns (d_xy, idx_xy, colkeys[B,M] int64, partials[B,4] fp64 with columns 0 and 2 set)."""
    x = _check_cloud(x, "x")
    y = _check_cloud(y, "y")
    B, N, _ = x.shape
    M = y.shape[1]
    q0, q1 = q_slice
    dev = x.device
    d_xy = torch.empty((B, q1 - q0), dtype=torch.float32, device=dev)
    i_xy = torch.empty((B, q1 - q0), dtype=torch.int32, device=dev)
    if keys is None:
        keys = torch.empty((B, M), dtype=torch.int64, device=dev)
    elif keys.dtype != torch.int64 or tuple(keys.shape) != (B, M) or not keys.is_contiguous() or keys.device != dev:
        raise TypeError(f"keys must be a contiguous int64 ({B}, {M}) tensor on {dev}")
    if partials is None:
        partials = torch.zeros((B, 4), dtype=torch.float64, device=dev)
    ws = workspace(_lib.CD_OP_FORWARD, B, N, M, dev)
    check(_lib.load().cd_forward_rows(_ptr(x), _ptr(y), B, N, M, q0, q1, _ptr(d_xy), _ptr(i_xy), _ptr(keys),
                                      _ptr(partials), float(-1.0 if tau is None else tau), _ptr(ws), ws.numel(),
                                      _stream()))
    return d_xy, i_xy, keys, partials


@_device_guard
def forward_cols(x: torch.Tensor, y: torch.Tensor, colkeys: torch.Tensor, r_slice, tau: float | None = None,
                 partials=None):
    """cd_forward_cols: resolve Y rows r_slice from (reduced) column keys.  Returns (d_yx, idx_yx,
    partials) with partials columns 1 and 3 set."""
    x = _check_cloud(x, "x")
    y = _check_cloud(y, "y")
    B, N, _ = x.shape
    M = y.shape[1]
    r0, r1 = r_slice
    dev = x.device
    d_yx = torch.empty((B, r1 - r0), dtype=torch.float32, device=dev)
    i_yx = torch.empty((B, r1 - r0), dtype=torch.int32, device=dev)
    if partials is None:
        partials = torch.zeros((B, 4), dtype=torch.float64, device=dev)
    ws = workspace(_lib.CD_OP_FORWARD, B, N, M, dev)
    check(_lib.load().cd_forward_cols(_ptr(x), _ptr(y), B, N, M, _ptr(colkeys.contiguous()), r0, r1, _ptr(d_yx),
                                      _ptr(i_yx), _ptr(partials), float(-1.0 if tau is None else tau), _ptr(ws),
                                      ws.numel(), _stream()))
    return d_yx, i_yx, partials


@_device_guard
def forward_cols_peers(x: torch.Tensor, y: torch.Tensor, colkeys, r_slice, tau: float | None = None,
                       partials=None):
    """cd_forward_cols_peers: resolve Y rows r_slice from the element-wise MIN of several [B,M] int64 key
    arrays read directly by the resolve kernel (the all-reduce fused into it).  colkeys: a list of
    tensors on x's device or of raw device pointers (ints, e.g. symmetric-memory peer buffers the
    caller has synchronised).  Returns (d_yx, idx_yx, partials) as forward_cols."""
    x = _check_cloud(x, "x")
    y = _check_cloud(y, "y")
    B, N, _ = x.shape
    M = y.shape[1]
    r0, r1 = r_slice
    dev = x.device
    ptrs = []
    for k in colkeys:
        if isinstance(k, torch.Tensor):
            if k.dtype != torch.int64 or tuple(k.shape) != (B, M) or not k.is_contiguous() or k.device != dev:
                raise TypeError(f"each key array must be a contiguous int64 ({B}, {M}) tensor on {dev}")
            ptrs.append(k.data_ptr())
        else:
            ptrs.append(int(k))
    arr = (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs)
    d_yx = torch.empty((B, r1 - r0), dtype=torch.float32, device=dev)
    i_yx = torch.empty((B, r1 - r0), dtype=torch.int32, device=dev)
    if partials is None:
        partials = torch.zeros((B, 4), dtype=torch.float64, device=dev)
    ws = workspace(_lib.CD_OP_FORWARD, B, N, M, dev)
    check(_lib.load().cd_forward_cols_peers(_ptr(x), _ptr(y), B, N, M, arr, len(ptrs), r0, r1, _ptr(d_yx),
                                            _ptr(i_yx), _ptr(partials), float(-1.0 if tau is None else tau),
                                            _ptr(ws), ws.numel(), _stream()))
    return d_yx, i_yx, partials


@_device_guard
def finalize(partials: torch.Tensor, N: int, M: int, w1: float = 1.0, w2: float = 1.0):
    """cd_finalize: returns (cd_per_batch[B], loss[1], fscore[B], precision[B], recall[B])."""
    B = partials.shape[0]
    dev = partials.device
    cd = torch.empty(B, dtype=torch.float32, device=dev)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    F = torch.empty(B, dtype=torch.float32, device=dev)
    P = torch.empty(B, dtype=torch.float32, device=dev)
    R = torch.empty(B, dtype=torch.float32, device=dev)
    check(_lib.load().cd_finalize(_ptr(partials.contiguous()), B, N, M, float(w1), float(w2), _ptr(cd), _ptr(loss),
                                  _ptr(F), _ptr(P), _ptr(R), _stream()))
    return cd, loss, F, P, R


@_device_guard
def fscore_from_distances(d_xy: torch.Tensor, d_yx: torch.Tensor, tau: float):
    """cd_fscore: (F, P, R) per batch element from per-point squared distances."""
    B, N = d_xy.shape
    M = d_yx.shape[1]
    dev = d_xy.device
    F = torch.empty(B, dtype=torch.float32, device=dev)
    P = torch.empty(B, dtype=torch.float32, device=dev)
    R = torch.empty(B, dtype=torch.float32, device=dev)
    ws = workspace(_lib.CD_OP_FSCORE, B, N, M, dev)
    check(_lib.load().cd_fscore(_ptr(d_xy.contiguous()), _ptr(d_yx.contiguous()), B, N, M, float(tau), _ptr(F),
                                _ptr(P), _ptr(R), _ptr(ws), ws.numel(), _stream()))
    return F, P, R


@_device_guard
def fscore(x: torch.Tensor, y: torch.Tensor, tau: float):
    """F-score at radius tau built on the same NN pass (forward with hit counting + finalize)."""
    _, _, _, _, part = forward(x, y, tau=tau)
    _, _, F, P, R = finalize(part, x.shape[1], y.shape[1])
    return F, P, R


@_device_guard
def backward(x: torch.Tensor, y: torch.Tensor, idx_xy: torch.Tensor, idx_yx: torch.Tensor, g=None, h=None,
             g_scalar: float = 0.0, h_scalar: float = 0.0, q_slice=None, r_slice=None):
    """cd_backward: gradients of sum(g*d_xy) + sum(h*d_yx) wrt x (rows q_slice) and y (rows r_slice)."""
    x = _check_cloud(x, "x")
    y = _check_cloud(y, "y")
    B, N, _ = x.shape
    M = y.shape[1]
    q0, q1 = q_slice if q_slice is not None else (0, N)
    r0, r1 = r_slice if r_slice is not None else (0, M)
    dev = x.device
    gx = torch.empty((B, q1 - q0, 3), dtype=torch.float32, device=dev)
    gy = torch.empty((B, r1 - r0, 3), dtype=torch.float32, device=dev)
    g = g.contiguous().float() if g is not None else None
    h = h.contiguous().float() if h is not None else None
    ws = workspace(_lib.CD_OP_BACKWARD, B, N, M, dev)
    check(_lib.load().cd_backward(_ptr(x), _ptr(y), B, N, M, _ptr(idx_xy.contiguous()), _ptr(idx_yx.contiguous()),
                                  _ptr(g), _ptr(h), float(g_scalar), float(h_scalar), q0, q1, r0, r1, _ptr(gx),
                                  _ptr(gy), _ptr(ws), ws.numel(), _stream()))
    return gx, gy


@_device_guard
def loss_backward(x: torch.Tensor, y: torch.Tensor, idx_xy: torch.Tensor, idx_yx: torch.Tensor,
                  grad_loss: torch.Tensor, w1: float = 1.0, w2: float = 1.0, q_slice=None, r_slice=None):
    """cd_loss_backward: gradients of grad_loss[0] * loss (cd_finalize's loss with weights w1, w2) wrt
    x (rows q_slice) and y (rows r_slice); grad_loss is a 1-element fp32 CUDA tensor read on the device."""
    x = _check_cloud(x, "x")
    y = _check_cloud(y, "y")
    B, N, _ = x.shape
    M = y.shape[1]
    q0, q1 = q_slice if q_slice is not None else (0, N)
    r0, r1 = r_slice if r_slice is not None else (0, M)
    if grad_loss.numel() != 1 or grad_loss.dtype != torch.float32 or not grad_loss.is_cuda:
        raise TypeError("grad_loss must be a 1-element fp32 CUDA tensor")
    dev = x.device
    gx = torch.empty((B, q1 - q0, 3), dtype=torch.float32, device=dev)
    gy = torch.empty((B, r1 - r0, 3), dtype=torch.float32, device=dev)
    ws = workspace(_lib.CD_OP_BACKWARD, B, N, M, dev)
    check(_lib.load().cd_loss_backward(_ptr(x), _ptr(y), B, N, M, _ptr(idx_xy.contiguous()),
                                       _ptr(idx_yx.contiguous()), _ptr(grad_loss.contiguous()), float(w1), float(w2),
                                       q0, q1, r0, r1, _ptr(gx), _ptr(gy), _ptr(ws), ws.numel(), _stream()))
    return gx, gy


def step_host(x_host: np.ndarray, y_host: np.ndarray, tau: float | None = None, w1: float = 1.0, w2: float = 1.0,
              want_grads: bool = True, device=None, out=None):
    """cd_step_host: one whole step through HOST buffers (H2D of the clouds, forward, finalize,
    loss backward, D2H of loss / F-score / gradients).  Host arrays should be pinned (see
    pinned_copy / pinned_empty).  Synchronises the device's current stream before returning
    (loss, fscore, grad_x, grad_y)."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.device(device):
        return _step_host(x_host, y_host, tau, w1, w2, want_grads, device, out)


def _step_host(x_host, y_host, tau, w1, w2, want_grads, device, out):
    B, N, _ = x_host.shape
    M = y_host.shape[1]
    ws = workspace(_lib.CD_OP_STEP, B, N, M, device)
    if out is None:
        out = dict(loss=pinned_empty((1,)), fscore=pinned_empty((B,)),
                   grad_x=pinned_empty((B, N, 3)) if want_grads else None,
                   grad_y=pinned_empty((B, M, 3)) if want_grads else None)
    check(_lib.load().cd_step_host(
        ctypes.c_void_p(x_host.ctypes.data) if isinstance(x_host, np.ndarray) else _ptr(x_host),
        ctypes.c_void_p(y_host.ctypes.data) if isinstance(y_host, np.ndarray) else _ptr(y_host),
        B, N, M, float(-1.0 if tau is None else tau), float(w1), float(w2),
        _host_ptr(out["loss"]), _host_ptr(out["fscore"]) if tau is not None else None,
        _host_ptr(out["grad_x"]), _host_ptr(out["grad_y"]), _ptr(ws), ws.numel(), _stream()))
    torch.cuda.current_stream().synchronize()
    return out


class HostStepper:
    """End-to-end steps from pinned host clouds with the host<->device copies overlapped with the
    compute (cd_step_host_overlapped).  Owns a private workspace, a copy stream, a second compute
    stream (two_streams) and nchunks + 1 events on its device; outputs (loss, F-score, gradients)
    land in pinned host tensors.  step() is asynchronous on the device's current stream: synchronise
    it before reading the outputs.  graph=True captures the call once and replays it."""

    def __init__(self, B: int, N: int, M: int, tau: float | None = None, w1: float = 1.0, w2: float = 1.0,
                 nchunks: int | None = None, device=None, want_grads: bool = True, graph: bool = False,
                 two_streams: bool = True):
        self.B, self.N, self.M, self.tau, self.w1, self.w2 = B, N, M, tau, w1, w2
        # measured (tools/time_e2e.py, gradients copied back, graph replay): c3 1 range 2.48 ms, 2: 2.30, 3: 2.25,
        # 4: 2.20, 8: 2.34; c2 1: 0.153, 2: 0.149, 4: 0.191 (each range's forward then under-fills the GPU)
        # -> up to 4 ranges of at least 2^31 distance evaluations each
        self.nchunks = nchunks or max(1, min(4, B, (B * N * M) >> 31))
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(self.device):
            self._init_device_state(B, N, M, want_grads, two_streams)
        # graph=True: the first step() with given host buffers is captured (the C call forks and joins
        # its copy stream, so it is capturable) and later steps replay it — every replay still copies
        # that step's inputs in and its results out; only the host-side launch work is saved
        self.graph = graph
        self._graph = None
        self._graph_key = None

    def _init_device_state(self, B, N, M, want_grads, two_streams):
        # a private workspace: its staging area is written by this stepper's copy stream
        n = int(_lib.load().cd_workspace_size(_lib.CD_OP_STEP, B, N, M))
        if n == 0:
            raise _lib.CdError(1, f"invalid sizes B={B} N={N} M={M}")
        self.ws = torch.empty(n, dtype=torch.uint8, device=self.device)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        # odd batch ranges compute on a second stream (overlapping the previous range's tail wave)
        self.stream2 = torch.cuda.Stream(device=self.device) if two_streams and self.nchunks > 1 else None
        self.events = [torch.cuda.Event() for _ in range(self.nchunks + 1)]
        for ev in self.events:       # materialise the cudaEvent handles
            ev.record()
        torch.cuda.synchronize(self.device)
        self._evp = (ctypes.c_void_p * (self.nchunks + 1))(*[ev.cuda_event for ev in self.events])
        self.loss = pinned_empty((1,))
        self.fscore = pinned_empty((B,))
        self.grad_x = pinned_empty((B, N, 3)) if want_grads else None
        self.grad_y = pinned_empty((B, M, 3)) if want_grads else None

    def d2h_bytes(self) -> int:
        """Bytes copied device -> host per step (loss, F-score, gradients)."""
        return 4 + (4 * self.B if self.tau is not None else 0) + \
            (12 * self.B * (self.N + self.M) if self.grad_x is not None else 0)

    def step(self, x_host: torch.Tensor, y_host: torch.Tensor):
        with torch.cuda.device(self.device):   # the stepper's workspace, streams and events live there
            return self._step(x_host, y_host)

    def _step(self, x_host, y_host):
        if self.graph:
            key = (x_host.data_ptr(), y_host.data_ptr())
            if self._graph is None or self._graph_key != key:
                self._call(x_host, y_host)                     # warm-up (plans, attributes) outside capture
                torch.cuda.current_stream().synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._call(x_host, y_host)
                self._graph, self._graph_key = g, key
            self._graph.replay()
            return self.loss, self.fscore, self.grad_x, self.grad_y
        self._call(x_host, y_host)
        return self.loss, self.fscore, self.grad_x, self.grad_y

    def _call(self, x_host, y_host):
        check(_lib.load().cd_step_host_overlapped(
            _host_ptr(x_host), _host_ptr(y_host), self.B, self.N, self.M,
            float(-1.0 if self.tau is None else self.tau), float(self.w1), float(self.w2),
            _host_ptr(self.loss), _host_ptr(self.fscore) if self.tau is not None else None,
            _host_ptr(self.grad_x), _host_ptr(self.grad_y), self.nchunks, _ptr(self.ws), self.ws.numel(), _stream(),
            ctypes.c_void_p(self.copy_stream.cuda_stream),
            ctypes.c_void_p(self.stream2.cuda_stream) if self.stream2 is not None else None, self._evp))


def _host_ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def pinned_empty(shape, dtype=torch.float32):
    return torch.empty(shape, dtype=dtype, pin_memory=True)


def pinned_copy(a: np.ndarray) -> torch.Tensor:
    t = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
    t.numpy()[...] = a
    return t


class ChamferFunction(torch.autograd.Function):
    """loss = mean_b [w1 mean_i d_xy + w2 mean_j d_yx] with the argmin held fixed in backward."""

    @staticmethod
    def forward(ctx, x, y, w1, w2, algorithm="brute"):
        d_xy, i_xy, d_yx, i_yx, part = forward(x, y, algorithm=algorithm)
        _, loss, _, _, _ = finalize(part, x.shape[1], y.shape[1], w1, w2)
        ctx.save_for_backward(x, y, i_xy, i_yx)
        ctx.w = (w1, w2)
        return loss[0]

    @staticmethod
    def backward(ctx, grad_out):
        x, y, i_xy, i_yx = ctx.saved_tensors
        w1, w2 = ctx.w
        # g = dL/dd_xy = grad_out * w1 / (B N): the upstream scalar multiplies a uniform fill
        gx, gy = loss_backward(x, y, i_xy, i_yx, grad_out.reshape(1), w1, w2)
        return gx, gy, None, None, None


def chamfer(x: torch.Tensor, y: torch.Tensor, w1: float = 1.0, w2: float = 1.0, algorithm: str = "brute") -> torch.Tensor:
    """Differentiable Chamfer loss (R1)."""
    return ChamferFunction.apply(x, y, w1, w2, algorithm)


def launch_count(op: int, B: int, N: int, M: int) -> int:
    return int(_lib.load().cd_launch_count(op, B, N, M))


def set_profile_events(start=None, stop=None):
    """Record torch.cuda.Events around the nn_fwd_kernel of subsequent forwards (None disables)."""
    _lib.load().cd_set_profile_events(ctypes.c_void_p(start.cuda_event) if start is not None else None,
                                      ctypes.c_void_p(stop.cuda_event) if stop is not None else None)



# ---------------------------------------------------------------------------------------- NEXT-4
def _sample_ws(op, B, Nv, Nf, N, device):
    lib = _lib.load()
    n = int(lib.cd_sample_workspace_size(op, B, Nv, Nf, N))
    if n == 0:
        raise _lib.CdError(1, f"invalid sizes B={B} Nv={Nv} Nf={Nf} N={N}")
    return _cached_ws("sample", op, n, device)


@_device_guard
def sample_mesh(verts: torch.Tensor, faces: torch.Tensor, r_face: torch.Tensor, r_bary: torch.Tensor):
    """cd_sample_mesh: (points [B,N,3], face_idx [B,N], bary [B,N,3]) for B meshes sharing `faces`."""
    if not verts.is_cuda or verts.dtype != torch.float32 or verts.dim() != 3:
        raise TypeError("verts must be CUDA fp32 (B, Nv, 3)")
    verts = verts.contiguous()
    faces = faces.to(torch.int32).contiguous()
    B, Nv, _ = verts.shape
    Nf = faces.shape[0]
    N = r_face.shape[1]
    dev = verts.device
    pts = torch.empty((B, N, 3), dtype=torch.float32, device=dev)
    fi = torch.empty((B, N), dtype=torch.int32, device=dev)
    ba = torch.empty((B, N, 3), dtype=torch.float32, device=dev)
    ws = _sample_ws(_lib.CD_OP_SAMPLE, B, Nv, Nf, N, dev)
    check(_lib.load().cd_sample_mesh(_ptr(verts), _ptr(faces), B, Nv, Nf, N, _ptr(r_face.contiguous()),
                                     _ptr(r_bary.contiguous()), _ptr(pts), _ptr(fi), _ptr(ba), _ptr(ws), ws.numel(),
                                     _stream()))
    return pts, fi, ba


@_device_guard
def sample_mesh_backward(faces: torch.Tensor, face_idx: torch.Tensor, bary: torch.Tensor, Nv: int,
                         grad_points: torch.Tensor):
    """cd_sample_mesh_backward: gradient w.r.t. the vertices (choices fixed)."""
    faces = faces.to(torch.int32).contiguous()
    B, N = face_idx.shape
    Nf = faces.shape[0]
    dev = bary.device
    gv = torch.empty((B, Nv, 3), dtype=torch.float32, device=dev)
    ws = _sample_ws(_lib.CD_OP_SAMPLE_BACKWARD, B, Nv, Nf, N, dev)
    check(_lib.load().cd_sample_mesh_backward(_ptr(faces), _ptr(face_idx.contiguous()), _ptr(bary.contiguous()), B,
                                              Nv, Nf, N, _ptr(grad_points.contiguous().float()), _ptr(gv), _ptr(ws),
                                              ws.numel(), _stream()))
    return gv


class SampleMeshFunction(torch.autograd.Function):
    """points = sample(verts; faces, randoms) with the reparameterisation gradient."""

    @staticmethod
    def forward(ctx, verts, faces, r_face, r_bary):
        pts, fi, ba = sample_mesh(verts, faces, r_face, r_bary)
        ctx.save_for_backward(faces, fi, ba)
        ctx.Nv = verts.shape[1]
        ctx.mark_non_differentiable(fi)
        return pts, fi

    @staticmethod
    def backward(ctx, grad_points, _grad_fi):
        faces, fi, ba = ctx.saved_tensors
        return sample_mesh_backward(faces, fi, ba, ctx.Nv, grad_points), None, None, None


def sample_points(verts, faces, r_face, r_bary):
    """Differentiable surface sampling: returns (points, face_idx); points carry gradients to verts."""
    return SampleMeshFunction.apply(verts, faces, r_face, r_bary)



# ---------------------------------------------------------------------------------------- NEXT-3
def _p2s_ws(op, B, N, Nv, Nf, device):
    n = int(_lib.load().cd_p2s_workspace_size(op, B, N, Nv, Nf))
    if n == 0:
        raise _lib.CdError(1, f"invalid sizes B={B} N={N} Nv={Nv} Nf={Nf}")
    return _cached_ws("p2s", op, n, device)


@_device_guard
def p2s_forward(points: torch.Tensor, verts: torch.Tensor, faces: torch.Tensor, algorithm: str = "brute"):
    """cd_p2s_forward (algorithm="brute") or cd_p2s_forward_pruned (algorithm="pruned", R26):
    (d [B,N], face [B,N], closest [B,N,3], bary [B,N,3], per_batch [B], loss [1])."""
    if algorithm not in ("brute", "pruned"):
        raise ValueError(f"algorithm must be 'brute' or 'pruned', got {algorithm!r}")
    points = _check_cloud(points, "points")
    verts = _check_cloud(verts, "verts")
    faces = faces.to(torch.int32).contiguous()
    B, N, _ = points.shape
    Nv = verts.shape[1]
    Nf = faces.shape[0]
    dev = points.device
    d = torch.empty((B, N), dtype=torch.float32, device=dev)
    fi = torch.empty((B, N), dtype=torch.int32, device=dev)
    cl = torch.empty((B, N, 3), dtype=torch.float32, device=dev)
    ba = torch.empty((B, N, 3), dtype=torch.float32, device=dev)
    pb = torch.empty(B, dtype=torch.float32, device=dev)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    op = _lib.CD_OP_P2S if algorithm == "brute" else _lib.CD_OP_P2S_PRUNED
    fn = _lib.load().cd_p2s_forward if algorithm == "brute" else _lib.load().cd_p2s_forward_pruned
    ws = _p2s_ws(op, B, N, Nv, Nf, dev)
    check(fn(_ptr(points), _ptr(verts), _ptr(faces), B, N, Nv, Nf, _ptr(d), _ptr(fi), _ptr(cl),
             _ptr(ba), _ptr(pb), _ptr(loss), _ptr(ws), ws.numel(), _stream()))
    return d, fi, cl, ba, pb, loss


@_device_guard
def p2s_backward(points, closest, face, bary, faces, Nv: int, g=None, g_scalar: float = 0.0,
                 want_points: bool = True, want_verts: bool = True):
    """cd_p2s_backward: (grad_points or None, grad_verts or None)."""
    faces = faces.to(torch.int32).contiguous()
    B, N, _ = points.shape
    Nf = faces.shape[0]
    dev = points.device
    gp = torch.empty((B, N, 3), dtype=torch.float32, device=dev) if want_points else None
    gv = torch.empty((B, Nv, 3), dtype=torch.float32, device=dev) if want_verts else None
    ws = _p2s_ws(_lib.CD_OP_P2S_BACKWARD, B, N, Nv, Nf, dev)
    check(_lib.load().cd_p2s_backward(_ptr(points.contiguous()), _ptr(closest.contiguous()), _ptr(face.contiguous()),
                                      _ptr(bary.contiguous()), _ptr(faces), B, N, Nv, Nf,
                                      _ptr(g.contiguous().float()) if g is not None else None, float(g_scalar),
                                      _ptr(gp), _ptr(gv), _ptr(ws), ws.numel(), _stream()))
    return gp, gv


@_device_guard
def p2s_loss_backward(points, closest, face, bary, faces, Nv: int, grad_loss: torch.Tensor,
                      want_points: bool = True, want_verts: bool = True):
    """cd_p2s_loss_backward: gradients of grad_loss[0] * (mean point-to-surface loss)."""
    faces = faces.to(torch.int32).contiguous()
    B, N, _ = points.shape
    Nf = faces.shape[0]
    if grad_loss.numel() != 1 or grad_loss.dtype != torch.float32 or not grad_loss.is_cuda:
        raise TypeError("grad_loss must be a 1-element fp32 CUDA tensor")
    dev = points.device
    gp = torch.empty((B, N, 3), dtype=torch.float32, device=dev) if want_points else None
    gv = torch.empty((B, Nv, 3), dtype=torch.float32, device=dev) if want_verts else None
    ws = _p2s_ws(_lib.CD_OP_P2S_BACKWARD, B, N, Nv, Nf, dev)
    check(_lib.load().cd_p2s_loss_backward(_ptr(points.contiguous()), _ptr(closest.contiguous()),
                                           _ptr(face.contiguous()), _ptr(bary.contiguous()), _ptr(faces), B, N, Nv,
                                           Nf, _ptr(grad_loss.contiguous()), _ptr(gp), _ptr(gv), _ptr(ws),
                                           ws.numel(), _stream()))
    return gp, gv


class PointToSurfaceFunction(torch.autograd.Function):
    """loss = mean_b mean_i min_f dist^2(p_i, face f); gradients to points and mesh vertices."""

    @staticmethod
    def forward(ctx, points, verts, faces, algorithm="brute"):
        d, fi, cl, ba, pb, loss = p2s_forward(points, verts, faces, algorithm=algorithm)
        ctx.save_for_backward(points, cl, fi, ba, faces)
        ctx.Nv = verts.shape[1]
        return loss[0]

    @staticmethod
    def backward(ctx, grad_out):
        points, cl, fi, ba, faces = ctx.saved_tensors
        gp, gv = p2s_loss_backward(points, cl, fi, ba, faces, ctx.Nv, grad_out.reshape(1),
                                   want_points=ctx.needs_input_grad[0], want_verts=ctx.needs_input_grad[1])
        return gp, gv, None, None


def point_to_surface(points, verts, faces, algorithm: str = "brute"):
    """Differentiable point-to-surface loss (GEOMetrics); algorithm "pruned" culls
    faces (R26) with the same minimum."""
    return PointToSurfaceFunction.apply(points, verts, faces, algorithm)
