#!/usr/bin/env python
"""Tensor-core forward (mode 3) device time per forced target-split count on c3 (design data for plan_tc)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1911_05063_b200 import api as cd, synth, _lib
X, Y = synth.config_inputs("c3")
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
_lib.load().cd_set_forward_mode(3)
for s in [0, 1, 2, 3, 4, 5, 6, 8, 12, 16]:
    cd.set_forward_splits(s)
    for _ in range(3):
        cd.forward(x, y, tau=0.01)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        cd.forward(x, y, tau=0.01)
    b.record(); torch.cuda.synchronize()
    print("tc splits", s, "forward ms %.4f" % (a.elapsed_time(b) / 10), flush=True)
cd.set_forward_splits(0)
