#!/usr/bin/env python
"""Randomised backward check against the oracle (bitwise, fp32 results of the same fp64 order), with
random index maps that include skewed and degenerate in-degree (one target taking every edge), random
query slices and tensor / scalar cotangents.  python tools/bwd_check.py [draws] [seed]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from paper_1911_05063_b200 import api as cd

draws = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
bad = 0
for k in range(draws):
    B = int(rng.integers(1, 5))
    N = int(rng.choice([1, 5, 300, 511, 512, 513, 1500, 4097, 20000, 70000]))
    M = int(rng.choice([1, 2, 100, 512, 1024, 2049, 9000, 33000]))
    if rng.random() < 0.1:   # c3-sized (2^20 keys: one 11-bit global pass) and beyond
        B, N, M = int(rng.choice([32, 40])), 16384, int(rng.choice([16384, 20000]))
    X = rng.normal(size=(B, N, 3)).astype(np.float32)
    Y = rng.normal(size=(B, M, 3)).astype(np.float32)
    kind = rng.choice(["uniform", "skew", "one", "few"])
    if kind == "uniform":
        ixy = rng.integers(0, M, size=(B, N))
        iyx = rng.integers(0, N, size=(B, M))
    elif kind == "skew":
        ixy = (M * rng.random(size=(B, N)) ** 6).astype(np.int64)
        iyx = (N * rng.random(size=(B, M)) ** 6).astype(np.int64)
    elif kind == "one":
        ixy = np.full((B, N), M - 1)
        iyx = np.zeros((B, M), np.int64)
    else:
        ixy = rng.integers(0, min(M, 3), size=(B, N))
        iyx = rng.integers(max(N - 3, 0), N, size=(B, M))
    ixy = ixy.astype(np.int32)
    iyx = iyx.astype(np.int32)
    tensor = bool(rng.integers(0, 2))
    g = rng.normal(size=(B, N)).astype(np.float32) if tensor else None
    h = rng.normal(size=(B, M)).astype(np.float32) if tensor else None
    q0 = int(rng.integers(0, N)); q1 = int(rng.integers(q0, N + 1))
    r0 = int(rng.integers(0, M)); r1 = int(rng.integers(r0, M + 1))
    sl = bool(rng.integers(0, 2))
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    kw = dict(g_scalar=0.5, h_scalar=0.25) if not tensor else {}
    args = (x, y, torch.from_numpy(ixy).cuda(), torch.from_numpy(iyx).cuda())
    if tensor:
        args = args + (torch.from_numpy(g).cuda(), torch.from_numpy(h).cuda())
    if sl:
        gx, gy = cd.backward(*args, q_slice=(q0, q1), r_slice=(r0, r1), **kw)
    else:
        gx, gy = cd.backward(*args, **kw)
    torch.cuda.synchronize()
    if tensor:
        gxr, gyr, _, _ = oracle.backward(X, Y, ixy, iyx, g, h)
    else:
        gxr, gyr, _, _ = oracle.backward(X, Y, ixy, iyx, g_scalar=np.float32(0.5), h_scalar=np.float32(0.25))
    if sl:
        gxr, gyr = gxr[:, q0:q1], gyr[:, r0:r1]
    ok = np.array_equal(gx.cpu().numpy(), gxr.astype(np.float32)) and np.array_equal(gy.cpu().numpy(), gyr.astype(np.float32))
    if not ok:
        bad += 1
        print("MISMATCH", k, B, N, M, kind, tensor, sl, (q0, q1, r0, r1), flush=True)
print(f"bwd_check draws={draws} bad={bad}", flush=True)
sys.exit(1 if bad else 0)
