#!/usr/bin/env python
"""Forward once, then the backward a few times on a config (for ncu launch lists of the backward)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
X, Y = synth.config_inputs(cfg)
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
B, N, M = X.shape[0], X.shape[1], Y.shape[1]
d_xy, i_xy, d_yx, i_yx, _ = cd.forward(x, y, tau=0.01, algorithm="pruned" if cfg in ("c4", "c5") else "brute")
torch.cuda.synchronize()
for _ in range(reps):
    cd.backward(x, y, i_xy, i_yx, g_scalar=1.0 / (B * N), h_scalar=1.0 / (B * M))
torch.cuda.synchronize()
print("ok")
