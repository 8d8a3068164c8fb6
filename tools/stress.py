#!/usr/bin/env python
"""Randomised cross-check of every forward path on one GPU: fused (default), per-direction, pruned,
tensor-core and query-sharded (rows / MIN of column keys / columns, emulated) forwards must agree bit
for bit (d, idx, hit counts) on random shapes / distributions, and the backward must be
deterministic.  python tools/stress.py [draws] [seed]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1911_05063_b200 import api as cd, synth

draws = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
bad = 0
for k in range(draws):
    B = int(rng.integers(1, 6))
    N = int(rng.choice([1, 2, 7, 31, 33, 511, 513, 1000, 2048, 3001, 8191, 12000, 20000]))
    M = int(rng.choice([1, 3, 32, 100, 512, 1025, 2047, 4096, 9000, 17000]))
    kind = rng.choice(["shape", "uniform", "dup", "cluster", "lattice", "scaled"])
    if kind == "shape":
        X, Y = synth.shape_pair(B, N, M, config_index=1000 + k)
    elif kind == "uniform":
        X, Y = synth.uniform_pair(B, N, M, seed=k)
    elif kind == "dup":
        Y = rng.uniform(-0.5, 0.5, size=(B, M, 3)).astype(np.float32)
        X = Y[:, rng.integers(0, M, size=N)].copy()
        Y = np.concatenate([Y, Y], axis=1)[:, :M].copy()
    elif kind == "cluster":
        Y = rng.uniform(-0.5, 0.5, size=(B, M, 3)).astype(np.float32)
        X = (Y[:, :1] + 5.0 + rng.normal(scale=1e-3, size=(B, N, 3))).astype(np.float32)
    elif kind == "lattice":
        g = (rng.integers(0, 16, size=(B, N + M, 3)) * 2.0 ** -5).astype(np.float32)
        X, Y = g[:, :N].copy(), (g[:, N:] + 2.0 ** -7).astype(np.float32)
    else:
        X, Y = synth.shape_pair(B, N, M, config_index=2000 + k)
        s = float(2.0 ** rng.integers(-8, 9))
        X, Y = (X * s + 100.0).astype(np.float32), (Y * s + 100.0).astype(np.float32)
    x, y = torch.from_numpy(np.ascontiguousarray(X)).cuda(), torch.from_numpy(np.ascontiguousarray(Y)).cuda()
    tau = float(rng.choice([0.0, 0.01, 0.05]))
    outs = {}
    for name, mode, algo in (("fused", 2, "brute"), ("unfused", 1, "brute"), ("tc", 3, "brute"), ("pruned", 0, "pruned")):
        old = cd.set_forward_mode(mode)
        try:
            outs[name] = [t.cpu().numpy() for t in cd.forward(x, y, tau=tau, algorithm=algo)]
        finally:
            cd.set_forward_mode(old)
    ref = outs["fused"]
    for name in ("unfused", "tc", "pruned"):
        o = outs[name]
        ok = all(np.array_equal(a.view(np.uint32) if a.dtype == np.float32 else a, b.view(np.uint32) if b.dtype == np.float32 else b)
                 for a, b in zip(o[:4], ref[:4])) and np.array_equal(o[4][:, 2:], ref[4][:, 2:])
        if not ok:
            bad += 1
            print(f"MISMATCH draw {k} {kind} B={B} N={N} M={M} tau={tau} path={name}", flush=True)
    # query sharding emulated on one GPU: rows per "rank", element-wise MIN of the column keys,
    # columns per "rank" -> the 1-GPU per-point results
    world = int(rng.integers(2, 9))
    keys = None
    drs, irs, dcs, ics = [], [], [], []
    for r in range(world):
        q = ((N * r) // world, (N * (r + 1)) // world)
        d_, i_, kk, _ = cd.forward_rows(x, y, q, tau=tau)
        drs.append(d_)
        irs.append(i_)
        keys = kk if keys is None else torch.minimum(keys, kk)
    for r in range(world):
        rr = ((M * r) // world, (M * (r + 1)) // world)
        d_, i_, _ = cd.forward_cols(x, y, keys, rr, tau=tau)
        dcs.append(d_)
        ics.append(i_)
    sh = [torch.cat(t, 1).cpu().numpy() for t in (drs, irs, dcs, ics)]
    if not all(np.array_equal(a.view(np.uint32) if a.dtype == np.float32 else a,
                              b.view(np.uint32) if b.dtype == np.float32 else b) for a, b in zip(sh, ref[:4])):
        bad += 1
        print(f"MISMATCH draw {k} query-sharded x{world}", flush=True)
    g1 = cd.backward(x, y, torch.from_numpy(ref[1]).cuda(), torch.from_numpy(ref[3]).cuda(), g_scalar=0.5, h_scalar=0.25)
    g2 = cd.backward(x, y, torch.from_numpy(ref[1]).cuda(), torch.from_numpy(ref[3]).cuda(), g_scalar=0.5, h_scalar=0.25)
    if not all(torch.equal(a, b) for a, b in zip(g1, g2)):
        bad += 1
        print(f"NONDETERMINISTIC backward draw {k}", flush=True)
print(f"stress: {draws} draws, {bad} failures")
