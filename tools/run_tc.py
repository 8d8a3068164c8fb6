#!/usr/bin/env python
"""Run the tensor-core forward on a config a few times (for ncu captures): python tools/run_tc.py [cfg] [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1911_05063_b200 import api as cd, synth, _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
X, Y = synth.config_inputs(cfg)
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
_lib.load().cd_set_forward_mode(3)
for _ in range(reps):
    cd.forward(x, y, tau=0.01)
torch.cuda.synchronize()
print("ok")
