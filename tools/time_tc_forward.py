#!/usr/bin/env python
"""Whole tensor-core forward (mode 3) device time vs the FP32 fused forward, and bit-equality of the
outputs: python tools/time_tc_forward.py [config]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth, _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
X, Y = synth.config_inputs(cfg)
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
res = {}
for mode in (0, 3):
    _lib.load().cd_set_forward_mode(mode)
    for _ in range(3):
        out = cd.forward(x, y, tau=0.01)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            out = cd.forward(x, y, tau=0.01)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 10)
    res[mode] = (best, [t.clone() for t in out])
_lib.load().cd_set_forward_mode(0)
same = all(torch.equal(p, q) for p, q in zip(res[0][1], res[3][1]))
print(os.environ.get("CD_LIB_VARIANT", "default"), cfg, "forward ms fused %.4f tensor %.4f identical %s" % (res[0][0], res[3][0], same))
