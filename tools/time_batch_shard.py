#!/usr/bin/env python
"""Per-rank work of batch sharding on one GPU: device time of the forward (brute) + loss backward for
a config's first B_local batch elements, B_local = B / G for G = 1, 2, 4, 8 (what one rank of a
G-GPU batch-sharded run computes), and the efficiency t(B) / (G t(B/G)).
python tools/time_batch_shard.py [c4] [G ...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
gs = [int(g) for g in sys.argv[2:]] or [1, 2, 4, 8]
Bfull = synth.CONFIGS[cfg]["B"]
tau = synth.CONFIGS[cfg]["tau"]
t1 = None
for G in gs:
    B = Bfull // G
    X, Y = synth.config_inputs(cfg, B=B)
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()

    def step():
        d_xy, i_xy, d_yx, i_yx, part = cd.forward(x, y, tau=tau)
        cd.backward(x, y, i_xy, i_yx, g_scalar=1.0 / (B * X.shape[1]), h_scalar=1.0 / (B * Y.shape[1]))

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    reps = max(2, 40 // (Bfull // G))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    if G == 1:
        t1 = ms
    eff = (t1 / (G * ms)) if t1 else float("nan")
    print(f"{cfg} G={G} B_local={B} step_ms={ms:.4f} efficiency_vs_G1={eff:.4f}", flush=True)
