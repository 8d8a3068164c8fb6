#!/usr/bin/env python
"""CUDA-event time of the fused forward kernel (cd_set_profile_events) on a config, clocks ramped."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
X, Y = synth.config_inputs(cfg)
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
ref = cd.forward(x, y, tau=0.01)
for _ in range(30):
    cd.forward(x, y, tau=0.01)
fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
fa.record(); fb.record(); torch.cuda.synchronize()
cd.set_profile_events(fa, fb)
ts = []
for _ in range(10):
    out = cd.forward(x, y, tau=0.01)
    torch.cuda.synchronize()
    ts.append(fa.elapsed_time(fb))
cd.set_profile_events(None, None)
same = all(torch.equal(p, q) for p, q in zip(ref, out))
print(os.environ.get("CD_LIB_VARIANT", "default"), cfg, "fused kernel ms min %.4f median %.4f" % (min(ts), sorted(ts)[5]), "same", same)
