#!/usr/bin/env python
"""Per-direction (unfused) forward time per forced split count on c3/c4 (design data for choose_splits)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1911_05063_b200 import api as cd, synth, _lib
for cfg in ["c3", "c4"]:
    X, Y = synth.config_inputs(cfg)
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    _lib.load().cd_set_forward_mode(1)
    for s in [0, 2, 4, 6, 8, 12, 16, 24, 32]:
        cd.set_forward_splits(s)
        for _ in range(2):
            cd.forward(x, y, tau=0.01)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5 if cfg == "c3" else 2
        a.record()
        for _ in range(reps):
            cd.forward(x, y, tau=0.01)
        b.record(); torch.cuda.synchronize()
        print(cfg, "unfused splits", s, "forward ms %.4f" % (a.elapsed_time(b) / reps), flush=True)
    cd.set_forward_splits(0)
    _lib.load().cd_set_forward_mode(0)
