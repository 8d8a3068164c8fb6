#!/usr/bin/env python
"""Culled vs brute point-to-surface: fraction of rows with the same face / bit-identical outputs on
the test workloads (near, far, on-surface, bench config)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from paper_1911_05063_b200 import api as cd, synth


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


cases = []
V, F = synth.mesh_batch(2, subdiv=3, config_index=132)
cases.append(("far", (synth.shape_pair(2, 3000, 8, config_index=133)[0] * 5.0 + 3.0).astype(np.float32), V, F))
rf, rb = synth.sampling_randoms(2, 3000, seed=12)
cases.append(("on", oracle.sample_mesh(V, F, rf, rb)[0].astype(np.float32), V, F))
V5, F5 = synth.mesh_batch(8, subdiv=5, config_index=134)
rf, rb = synth.sampling_randoms(8, 16384, seed=13)
P5 = oracle.sample_mesh(V5, F5, rf, rb)[0]
cases.append(("bench", (P5 + np.random.default_rng(6).normal(scale=1e-2, size=P5.shape)).astype(np.float32), V5, F5))
bad = 0
for name, P, V, F in cases:
    op = cd.p2s_forward(t(P), t(V), t(F), algorithm="pruned")
    ob = cd.p2s_forward(t(P), t(V), t(F))
    torch.cuda.synchronize()
    same = (op[1] == ob[1]).float().mean().item()
    ident = all(torch.equal(a, b) for a, b in zip(op[:4], ob[:4]))
    bad += not ident
    print(f"{name}: same face {same:.6f} identical {ident}", flush=True)
sys.exit(1 if bad else 0)
