#!/usr/bin/env python
"""Brute-force point-to-surface forward time per forced split count (bench NEXT-3 workload): design
data for plan_p2s.  python tools/sweep_p2s_splits.py [s1,s2,...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

splits = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 64]
B, N = 8, 16384
V, F = synth.mesh_batch(B, subdiv=5, config_index=200)
P = synth.shape_pair(B, N, 8, config_index=201)[0]
v, f, p = torch.from_numpy(V).cuda(), torch.from_numpy(F).cuda(), torch.from_numpy(P).cuda()
ref = None
for s in splits:
    cd.set_forward_splits(s)
    for _ in range(2):
        out = cd.p2s_forward(p, v, f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        out = cd.p2s_forward(p, v, f)
    e1.record()
    torch.cuda.synchronize()
    ref = ref or [t.clone() for t in out[:4]]
    same = all(torch.equal(a, b) for a, b in zip(ref, out[:4]))
    print(f"p2s splits={s:3d} forward_ms={e0.elapsed_time(e1) / 5:.4f} same={same}", flush=True)
cd.set_forward_splits(0)
