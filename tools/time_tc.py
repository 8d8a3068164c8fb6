#!/usr/bin/env python
"""CUDA-event time of the tensor-core forward's main kernel (cd_set_profile_events) on a config."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth, _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
X, Y = synth.config_inputs(cfg)
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
_lib.load().cd_set_forward_mode(3)
for _ in range(2):
    cd.forward(x, y, tau=0.01)
fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
fa.record(); fb.record(); torch.cuda.synchronize()
cd.set_profile_events(fa, fb)
ts = []
for _ in range(5):
    cd.forward(x, y, tau=0.01)
    torch.cuda.synchronize()
    ts.append(fa.elapsed_time(fb))
cd.set_profile_events(None, None)
print(os.environ.get("CD_LIB_VARIANT", "default"), "main kernel ms", min(ts))
