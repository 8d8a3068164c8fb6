#!/usr/bin/env python
"""Run the forward a few times (for ncu launch lists): run_forward.py <config> <brute|pruned> [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

cfg, algo = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
X, Y = synth.config_inputs(cfg)
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
for _ in range(reps):
    cd.forward(x, y, tau=synth.CONFIGS[cfg]["tau"], algorithm=algo)
torch.cuda.synchronize()
print("ok")
