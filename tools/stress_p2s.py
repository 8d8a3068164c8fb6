#!/usr/bin/env python
"""Randomised cross-check of the culled point-to-surface forward against the brute-force kernel:
the same face for every point (lowest original index among exact fp32 ties, R3') and bit-identical
d / closest / bary.  python tools/stress_p2s.py [draws] [seed]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1911_05063_b200 import api as cd, synth
import oracle

draws = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
bad = 0
for k in range(draws):
    B = int(rng.integers(1, 4))
    sub = int(rng.integers(0, 5))
    N = int(rng.choice([1, 5, 100, 1000, 4097, 10000]))
    V, F = synth.mesh_batch(B, subdiv=sub, config_index=3000 + k)
    if rng.random() < 0.3:   # some degenerate faces: a repeated vertex (zero area) or collinear corners
        F = F.copy()
        bad_f = rng.choice(len(F), size=max(1, len(F) // 10), replace=False)
        F[bad_f, 2] = F[bad_f, 1]
    kind = rng.choice(["near", "on", "far", "shape", "scaled"])
    if kind in ("near", "on"):
        rf, rb = synth.sampling_randoms(B, N, seed=4000 + k)
        P, _, _, _ = oracle.sample_mesh(V, F, rf, rb)
        if kind == "near":
            P = P + rng.normal(scale=10 ** rng.uniform(-4, -1), size=P.shape)
    elif kind == "far":
        P = rng.uniform(-3, 3, size=(B, N, 3))
    else:
        P = synth.shape_pair(B, N, 8, config_index=5000 + k)[0]
    P = P.astype(np.float32)
    if kind == "scaled":
        s = float(2.0 ** rng.integers(-6, 7))
        P, V = (P * s + 7.0).astype(np.float32), (V * s + 7.0).astype(np.float32)
    p, v, f = torch.from_numpy(np.ascontiguousarray(P)).cuda(), torch.from_numpy(V).cuda(), torch.from_numpy(F).cuda()
    ob = [t.cpu().numpy() for t in cd.p2s_forward(p, v, f)]
    op = [t.cpu().numpy() for t in cd.p2s_forward(p, v, f, algorithm="pruned")]
    ok = all(np.array_equal(a, b) for a, b in zip(op[:4], ob[:4]))
    if not ok:
        bad += 1
        print(f"MISMATCH draw {k} {kind} B={B} sub={sub} N={N}", flush=True)
print(f"stress_p2s: {draws} draws, {bad} failures")
