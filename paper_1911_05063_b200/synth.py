"""Seeded synthetic point clouds shaped like the paper's workloads.

This module holds NONE of the method's arithmetic (no distances, no nearest neighbours, no
losses): it only draws inputs.  It is the one module both the oracle side (tests, bench
cpu_baseline) and the CUDA side consume, so both see the same bytes.

Recipe:
* "ShapeNet-like" shape per batch element b: an icosphere (subdivision 5, 20,480 faces) with a
  smooth radial deformation r(n) = 0.35 * (1 + sum_{k<8} a_k sin(w_k <n, e_k> + phi_k)),
  a_k ~ U(0, 0.1), w_k ~ U(1, 4) * pi, phi_k ~ U(0, 2 pi), e_k random unit axes; normalised
  to the unit cube [-0.5, 0.5]^3 (ShapeNet-style normalisation).
* Points sampled area-uniformly: face with probability proportional to area, square-root
  barycentrics u = 1 - sqrt(r1), v = sqrt(r1)(1 - r2), w = sqrt(r1) r2.
* X = N surface samples ("prediction"); Y = M surface samples + N(0, 0.005^2) jitter
  ("reference"), so F@0.01 is mid-range.  Points come out in random order (unordered sets).
* Seeds: np.random.SeedSequence([1911050630, config_index, b]).spawn(3) -> (shape, X, Y) PCG64
  streams per batch element, so Y_b and X_{b+1} never share a stream.
"""
from __future__ import annotations

import functools

import numpy as np

ROOT_SEED = 1911050630

# The five BASELINE.json configs (index = configs[k]).
CONFIGS = {
    "c1": dict(index=0, B=1, N=1024, M=1024, tau=None, backward=False,
               desc="B=1, N=M=1,024 fp32 3D clouds, Chamfer forward + indices"),
    "c2": dict(index=1, B=32, N=2048, M=2048, tau=None, backward=True,
               desc="B=32, N=M=2,048 (PointNet/ShapeNet sampling) Chamfer forward+backward"),
    "c3": dict(index=2, B=32, N=16384, M=16384, tau=0.01, backward=True,
               desc="B=32, N=M=16,384 Chamfer forward+backward plus F-score at tau=0.01"),
    "c4": dict(index=3, B=8, N=100000, M=100000, tau=0.01, backward=True,
               desc="B=8, N=M=100,000 mesh-surface samples, batch-sharded"),
    "c5": dict(index=4, B=4, N=1048576, M=1048576, tau=0.01, backward=True,
               desc="B=4, N=M=1,048,576 clouds, query-sharded"),
}


@functools.lru_cache(maxsize=2)
def icosphere(subdiv: int = 5):
    """Unit icosphere: (V, 3) float64 vertices, (F, 3) int64 faces."""
    t = (1.0 + 5.0 ** 0.5) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t),
             (0, -1, -t), (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    v = np.array(verts, np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array(faces, np.int64)
    for _ in range(subdiv):
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]], axis=0)
        e_sorted = np.sort(e, axis=1)
        uniq, inv = np.unique(e_sorted, axis=0, return_inverse=True)
        mid = v[uniq[:, 0]] + v[uniq[:, 1]]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        base = v.shape[0]
        v = np.concatenate([v, mid], axis=0)
        nf = f.shape[0]
        m01 = base + inv[:nf]
        m12 = base + inv[nf:2 * nf]
        m20 = base + inv[2 * nf:]
        f = np.concatenate([
            np.stack([f[:, 0], m01, m20], 1),
            np.stack([f[:, 1], m12, m01], 1),
            np.stack([f[:, 2], m20, m12], 1),
            np.stack([m01, m12, m20], 1)], axis=0)
    return v, f


def random_shape(rng: np.random.Generator, subdiv: int = 5):
    """Deformed icosphere normalised to [-0.5, 0.5]^3: (V,3) vertices, (F,3) faces."""
    v, f = icosphere(subdiv)
    K = 8
    axes = rng.normal(size=(K, 3))
    axes /= np.linalg.norm(axes, axis=1, keepdims=True)
    amp = rng.uniform(0.0, 0.1, size=K)
    freq = rng.uniform(1.0, 4.0, size=K) * np.pi
    phase = rng.uniform(0.0, 2 * np.pi, size=K)
    u = v @ axes.T  # (V, K)
    r = 0.35 * (1.0 + (amp * np.sin(freq * u + phase)).sum(axis=1))
    p = v * r[:, None]
    lo, hi = p.min(axis=0), p.max(axis=0)
    p = (p - (lo + hi) / 2) / (hi - lo).max()
    return p, f


def sample_surface(rng: np.random.Generator, verts, faces, n: int):
    """Area-uniform surface samples with square-root barycentrics."""
    a, b, c = verts[faces[:, 0]], verts[faces[:, 1]], verts[faces[:, 2]]
    area = 0.5 * np.linalg.norm(np.cross(b - a, c - a), axis=1)
    cdf = np.cumsum(area)
    cdf /= cdf[-1]
    fi = np.searchsorted(cdf, rng.random(n), side="right").clip(0, faces.shape[0] - 1)
    r1 = np.sqrt(rng.random(n))
    r2 = rng.random(n)
    wa, wb, wc = 1.0 - r1, r1 * (1.0 - r2), r1 * r2
    return wa[:, None] * a[fi] + wb[:, None] * b[fi] + wc[:, None] * c[fi]


def _streams(config_index: int, b: int):
    ss = np.random.SeedSequence([ROOT_SEED, int(config_index), int(b)])
    return [np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(3)]


def shape_pair(B: int, N: int, M: int, config_index: int = 0, jitter: float = 0.005,
               b0: int = 0):
    """X (B,N,3), Y (B,M,3) fp32 "prediction vs reference" clouds for batch elements b0..b0+B-1."""
    X = np.empty((B, N, 3), np.float32)
    Y = np.empty((B, M, 3), np.float32)
    for k in range(B):
        rs, rx, ry = _streams(config_index, b0 + k)
        v, f = random_shape(rs)
        X[k] = sample_surface(rx, v, f, N)
        Y[k] = sample_surface(ry, v, f, M) + ry.normal(scale=jitter, size=(M, 3))
    return X, Y


def uniform_pair(B: int, N: int, M: int, seed: int = 0):
    """X, Y uniform in [-0.5, 0.5]^3 (fp32)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([ROOT_SEED, 1000 + seed])))
    X = rng.uniform(-0.5, 0.5, size=(B, N, 3)).astype(np.float32)
    Y = rng.uniform(-0.5, 0.5, size=(B, M, 3)).astype(np.float32)
    return X, Y


def config_inputs(name: str, b0: int = 0, B: int | None = None):
    """Inputs for a BASELINE.json config (optionally a batch sub-range, for batch sharding)."""
    c = CONFIGS[name]
    B = c["B"] if B is None else B
    return shape_pair(B, c["N"], c["M"], config_index=c["index"], b0=b0)


def mesh_batch(B: int, config_index: int = 100, subdiv: int = 5):
    """Deformed-icosphere meshes sharing one topology: verts (B,V,3) fp32, faces (F,3) int32."""
    _, faces = icosphere(subdiv)
    verts = []
    for b in range(B):
        rs, _, _ = _streams(config_index, b)
        v, _ = random_shape(rs, subdiv)
        verts.append(v)
    return np.stack(verts).astype(np.float32), faces.astype(np.int32)


def sampling_randoms(B: int, N: int, seed: int = 0):
    """Random numbers the sampling step draws (passed to both sides as inputs): r_face (B,N) uint32,
    r_bary (B,N,2) fp32 uniforms in [0, 1)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([ROOT_SEED, 2000 + seed])))
    r_face = rng.integers(0, 2 ** 32, size=(B, N), dtype=np.uint64).astype(np.uint32)
    r_bary = rng.random(size=(B, N, 2), dtype=np.float32)
    return r_face, r_bary
