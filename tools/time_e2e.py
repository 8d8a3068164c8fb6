#!/usr/bin/env python
"""e2e step time (HostStepper, pinned host clouds, gradients copied back) for several nchunks, eager
and CUDA-graph replayed: python tools/time_e2e.py c3 1 2 4 8"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
X, Y = synth.config_inputs(cfg)
B, N, M = X.shape[0], X.shape[1], Y.shape[1]
xh, yh = cd.pinned_copy(X), cd.pinned_copy(Y)
for graph, two in ((False, False), (True, False), (True, True)):
    for nc in [int(v) for v in sys.argv[2:]]:
        st = cd.HostStepper(B, N, M, tau=synth.CONFIGS[cfg]["tau"], nchunks=min(nc, B), graph=graph, two_streams=two)
        for _ in range(20):
            st.step(xh, yh)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                st.step(xh, yh)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 20)
        print(cfg, "graph" if graph else "eager", "2 streams" if two else "1 stream", "nchunks", nc, "e2e ms/step", best,
              flush=True)
