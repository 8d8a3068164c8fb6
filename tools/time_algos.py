#!/usr/bin/env python
"""Device time of the full forward (cd_forward brute vs cd_forward_pruned) per config."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

for cfg in sys.argv[1:] or ["c2", "c3", "c4", "c5"]:
    X, Y = synth.config_inputs(cfg)
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    tau = synth.CONFIGS[cfg]["tau"]
    reps = {"c1": 50, "c2": 50, "c3": 20, "c4": 5, "c5": 2}[cfg]
    for algo in ("brute", "pruned"):
        for _ in range(2):
            cd.forward(x, y, tau=tau, algorithm=algo)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            cd.forward(x, y, tau=tau, algorithm=algo)
        b.record()
        torch.cuda.synchronize()
        print(f"{cfg} {algo:6s} forward_ms={a.elapsed_time(b) / reps:.4f}", flush=True)
