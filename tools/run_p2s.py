#!/usr/bin/env python
"""Run the point-to-surface forward (bench NEXT-3 workload) a few times (for ncu captures)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

B, N = 8, 16384
V, F = synth.mesh_batch(B, subdiv=5, config_index=200)
P = synth.shape_pair(B, N, 8, config_index=201)[0]
v, f, p = torch.from_numpy(V).cuda(), torch.from_numpy(F).cuda(), torch.from_numpy(P).cuda()
for _ in range(2):
    cd.p2s_forward(p, v, f)
torch.cuda.synchronize()
print("ok")
