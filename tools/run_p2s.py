#!/usr/bin/env python
"""Run the point-to-surface forward (bench NEXT-3 workload) a few times (for ncu captures) and time
both algorithms with CUDA events: python tools/run_p2s.py [brute|pruned|both]."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

algos = ["brute", "pruned"] if len(sys.argv) < 2 or sys.argv[1] == "both" else [sys.argv[1]]
B, N = 8, 16384
V, F = synth.mesh_batch(B, subdiv=5, config_index=200)
P = synth.shape_pair(B, N, 8, config_index=201)[0]
v, f, p = torch.from_numpy(V).cuda(), torch.from_numpy(F).cuda(), torch.from_numpy(P).cuda()
for algo in algos:
    for _ in range(2):
        cd.p2s_forward(p, v, f, algorithm=algo)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        cd.p2s_forward(p, v, f, algorithm=algo)
    e1.record()
    torch.cuda.synchronize()
    print(algo, "ms", e0.elapsed_time(e1) / 10)
print("ok")
